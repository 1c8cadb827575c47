mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu -lcuda && timeout 300 /tmp/tma_probe > gpurun_out/tma_probe.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe tools/pipe_probe.cu -lcuda && timeout 120 /tmp/pipe_probe > gpurun_out/pipe_probe.log 2>&1
