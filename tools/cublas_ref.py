"""cuBLAS (torch.matmul) time for the DyLLM GEMM shapes: the library reference point for the
hand-written tcgen05 kernels (tools/gemm_bench.py). Not used on the product path."""
import torch

shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (24576, 4096), "down": (4096, 12288)}
for name, (N, K) in shapes.items():
    W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    for M in (100, 205, 410, 1530, 15296):
        A = torch.randn(M, K, device="cuda").bfloat16()
        for _ in range(3):
            torch.matmul(A, W.T)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            torch.matmul(A, W.T)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        print(f"cublas {name:5s} M={M:6d}: {us:8.2f} us  {2.0 * M * N * K / us / 1e6:7.1f} TFLOP/s")
