# round 2: skinny epilogue with 16-byte stores
for D in 0 4; do timeout 120 python tools/gemm_bench.py --rows 100,410,1530 --dbg $D --which qkv,o,gu,down | grep -v "^\s*$"; done
echo "qkv dbg=3 $(timeout 120 python tools/skinny_trace.py --which qkv --rows 410 --dbg 3 | grep -E 'tfull0|published' | tr -s ' ' | tr '\n' ' ')"
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x 2>&1 | tail -3
