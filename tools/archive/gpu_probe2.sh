mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe tools/mma_probe.cu && timeout 120 /tmp/mma_probe > gpurun_out/mma_probe.log 2>&1
