"""Counter-based synthetic generators ("IH4"): bit-reproducible on CPU and GPU.

Every element of every tensor is a pure function of (seed, stream, element
index), so any element can be regenerated independently (used for sampled
parity at full size). The CUDA library implements the same generator in
csrc/kernels.cu:ih4_fill_kernel ("input recipe"); nothing here is DyLLM
arithmetic.

Definition (all integer arithmetic mod 2**64):
    mix64(x):  z = x + 0x9E3779B97F4A7C15
               z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
               z = (z ^ (z >> 27)) * 0x94D049BB133111EB
               return z ^ (z >> 31)
    key(seed, stream) = mix64(seed ^ mix64(stream))
    h_i               = mix64(key + i)
    S_i = sum of the four 16-bit fields of h_i            (0 .. 262140)
    c_i = S_i - 131070                                     (int, exact in fp32)
    v_i = bf16_rne( fp32(c_i) * fp32(std / SD_IH4) )       (one IEEE fp32 multiply)
with SD_IH4 = sqrt((65536**2 - 1) / 3), the standard deviation of a sum of four
uniform 16-bit integers. The result is Irwin-Hall(4): mean 0, std `std`,
support ±3.46 std — a bounded stand-in for the normal init std 0.02 of S:146-154.
Token ids: t_i = h_i mod mask_id (prompt ids never equal the mask id).
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)
SD_IH4 = math.sqrt((65536.0 ** 2 - 1.0) / 3.0)

# tensor codes for stream ids (layer-local tensors use layer * 64 + code)
TENSOR_CODES = {
    "wq": 1, "wk": 2, "wv": 3, "bq": 4, "bk": 5, "bv": 6, "wo": 7,
    "w_gate": 8, "w_up": 9, "w_down": 10, "g_attn": 11, "g_ffn": 12,
    "emb": 20, "g_final": 21, "lm_head": 22, "tokens": 30,
    # synthetic cache/activation contents for teacher-forced parity at full size
    "cK": 40, "cV": 41, "cQ": 42, "cC": 43, "cH": 44, "cX": 45, "cX2": 46,
}
GLOBAL_LAYER = 65535


def stream_id(layer: int, name: str) -> int:
    return layer * 64 + TENSOR_CODES[name]


def _mix64_py(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _mix64_np(x: np.ndarray) -> np.ndarray:
    z = x + GOLDEN
    z = (z ^ (z >> np.uint64(30))) * C1
    z = (z ^ (z >> np.uint64(27))) * C2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> int:
    return _mix64_py((seed & M64) ^ _mix64_py(stream & M64))


def _hashes(seed: int, stream: int, start: int, n: int) -> np.ndarray:
    key = np.uint64(stream_key(seed, stream))
    idx = np.arange(start, start + n, dtype=np.uint64)
    return _mix64_np(idx + key)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    return ((u + r) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def ih4_scale(std: float) -> np.float32:
    return np.float32(std / SD_IH4)


def ih4_normal_bf16_bits(seed: int, stream: int, n: int, std: float, start: int = 0,
                         chunk: int = 1 << 24) -> np.ndarray:
    """n IH4 values (elements start..start+n of the stream) as bf16 bit patterns."""
    out = np.empty(n, dtype=np.uint16)
    scale = ih4_scale(std)
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        h = _hashes(seed, stream, start + s, m)
        f = np.uint64(0xFFFF)
        tot = (h & f) + ((h >> np.uint64(16)) & f) + ((h >> np.uint64(32)) & f) + (h >> np.uint64(48))
        c = tot.astype(np.int64) - 131070
        v = c.astype(np.float32) * scale          # one fp32 multiply, IEEE RN
        out[s:s + m] = f32_to_bf16_bits(v)
    return out


def ih4_normal(seed: int, stream: int, shape, std: float, dtype=np.float64) -> np.ndarray:
    n = int(np.prod(shape))
    return bf16_bits_to_f32(ih4_normal_bf16_bits(seed, stream, n, std)).astype(dtype).reshape(shape)


def prompt_tokens(seed: int, batch: int, L_P: int, mask_id: int) -> np.ndarray:
    out = np.empty((batch, L_P), dtype=np.int32)
    for b in range(batch):
        h = _hashes(seed, stream_id(b, "tokens") + (1 << 40), 0, L_P)
        out[b] = (h % np.uint64(mask_id)).astype(np.int32)
    return out


def layer_weights(cfg, seed: int, layer: int, dtype=np.float64) -> dict:
    """One layer's weights in torch-Linear layout W[out][in] (y = x @ W.T)."""
    d, qw, kw, F = cfg.d_model, cfg.q_width, cfg.kv_width, cfg.d_ff
    s = cfg.w_std
    sqk = cfg.qk_std or cfg.w_std
    w = {
        "wq": ih4_normal(seed, stream_id(layer, "wq"), (qw, d), sqk, dtype),
        "wk": ih4_normal(seed, stream_id(layer, "wk"), (kw, d), sqk, dtype),
        "wv": ih4_normal(seed, stream_id(layer, "wv"), (kw, d), s, dtype),
        "wo": ih4_normal(seed, stream_id(layer, "wo"), (d, qw), s, dtype),
        "w_gate": ih4_normal(seed, stream_id(layer, "w_gate"), (F, d), s, dtype),
        "w_up": ih4_normal(seed, stream_id(layer, "w_up"), (F, d), s, dtype),
        "w_down": ih4_normal(seed, stream_id(layer, "w_down"), (d, F), s, dtype),
        "g_attn": np.ones(d, dtype=dtype),
        "g_ffn": np.ones(d, dtype=dtype),
    }
    if cfg.qkv_bias:
        w["bq"] = ih4_normal(seed, stream_id(layer, "bq"), (qw,), s, dtype)
        w["bk"] = ih4_normal(seed, stream_id(layer, "bk"), (kw,), s, dtype)
        w["bv"] = ih4_normal(seed, stream_id(layer, "bv"), (kw,), s, dtype)
    return w


def global_weights(cfg, seed: int, dtype=np.float64) -> dict:
    d = cfg.d_model
    s = cfg.w_std
    return {
        "emb": ih4_normal(seed, stream_id(GLOBAL_LAYER, "emb"), (cfg.vocab, d), s, dtype),
        "g_final": np.ones(d, dtype=dtype),
        "lm_head": ih4_normal(seed, stream_id(GLOBAL_LAYER, "lm_head"), (cfg.vocab, d),
                              getattr(cfg, "lm_std", 0.0) or s, dtype),
    }


def model_weights(cfg, seed: int, dtype=np.float64) -> dict:
    g = global_weights(cfg, seed, dtype)
    g["layers"] = [layer_weights(cfg, seed, l, dtype) for l in range(cfg.n_layers)]
    return g


def cache_tensor(seed: int, layer: int, name: str, batch: int, N: int, width: int, std: float,
                 dtype=np.float32) -> np.ndarray:
    """Synthetic [batch][N][width] cache/activation contents (IH4, one stream per sequence), for
    teacher-forced parity at full size: the oracle and the GPU receive the same bf16 values."""
    out = np.empty((batch, N, width), dtype=dtype)
    for b in range(batch):
        out[b] = ih4_normal(seed, stream_id(layer, name) + ((b + 1) << 32), (N, width), std, dtype)
    return out
