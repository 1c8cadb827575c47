"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds ONLY configuration shapes and counter-based random number
generators. It contains none of DyLLM's arithmetic (no norm, projection,
attention, similarity, selection or unmasking). Both `oracle/` and the tests /
bench of the CUDA path import it; the CUDA library (csrc/init.cu) carries its
own independent implementation of the same generator.
"""
from .configs import ModelCfg, RunCfg, PRESETS, preset  # noqa: F401
from .gen import (  # noqa: F401
    ih4_normal, ih4_normal_bf16_bits, bf16_bits_to_f32, f32_to_bf16_bits,
    model_weights, layer_weights, global_weights, prompt_tokens, stream_id,
    TENSOR_CODES,
)
