"""B200-native DyLLM salient-token denoising step (arxiv 2603.08026).

The compute path lives in libdyllm.so (include/dyllm.h); `dyllm` is its ctypes binding.
Import `paper_2603_08026_b200.dyllm` explicitly — it raises if the library is not built.
"""
__all__ = ["dyllm"]
