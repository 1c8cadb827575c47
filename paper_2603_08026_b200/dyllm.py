"""Thin ctypes binding of libdyllm.so (include/dyllm.h): argument marshalling only.

Every step of the DyLLM path runs in the CUDA library; torch supplies device memory, streams
and process groups. There is no CPU fallback: importing this module fails loudly when
libdyllm.so is missing, and every call raises DyllmError on a non-zero status.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdyllm.so")

OK, DONE = 0, 1
INPUT_FULL, INPUT_RESPONSE = 0, 1
K, V, Q, CTX, H, STATS = 0, 1, 2, 3, 4, 5
_CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


class DyllmError(RuntimeError):
    pass


class ModelCfg(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("d_ff", C.c_int32),
                ("vocab", C.c_int32), ("mask_id", C.c_int32), ("rope_theta", C.c_float),
                ("rms_eps", C.c_float), ("qkv_bias", C.c_int32), ("residual_mode", C.c_int32),
                ("dtype", C.c_int32)]

    @classmethod
    def from_py(cls, m):
        return cls(m.n_layers, m.d_model, m.n_heads, m.n_kv_heads, m.head_dim, m.d_ff, m.vocab,
                   m.mask_id, m.rope_theta, m.rms_eps, int(m.qkv_bias), m.residual_mode,
                   int(getattr(m, "dtype", 0)))


class RunCfg(C.Structure):
    _fields_ = [("batch", C.c_int32), ("L_P", C.c_int32), ("L_R", C.c_int32), ("block", C.c_int32),
                ("n_u", C.c_int32), ("T_full", C.c_int32), ("full_period", C.c_int32),
                ("layer1_policy", C.c_int32), ("cmp", C.c_int32), ("select_mode", C.c_int32)]

    @classmethod
    def from_py(cls, r):
        return cls(r.batch, r.L_P, r.L_R, r.block, r.n_u, r.T_full, r.full_period, r.layer1_policy, r.cmp,
                   getattr(r, "select_mode", 0))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built — run __graft_entry__.build() "
                          "(the DyLLM path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I, I64, F, D, U64 = C.c_void_p, C.c_int, C.c_int64, C.c_float, C.c_double, C.c_uint64
    PP = C.POINTER(C.c_void_p)
    sig = {
        "dyllm_last_error": (C.c_char_p, []),
        "dyllm_version": (I, []),
        "dyllm_ctx_create": (I, [I, P, PP]),
        "dyllm_ctx_sync": (I, [P]),
        "dyllm_ctx_destroy": (None, [P]),
        "dyllm_weights_blob_elems": (I64, [C.POINTER(ModelCfg)]),
        "dyllm_weights_load": (I, [P, C.POINTER(ModelCfg), P, I64, PP]),
        "dyllm_weights_init_random": (I, [P, C.POINTER(ModelCfg), U64, D, PP]),
        "dyllm_weights_destroy": (None, [P]),
        "dyllm_cache_create": (I, [P, P, C.POINTER(RunCfg), PP]),
        "dyllm_cache_destroy": (None, [P]),
        "dyllm_cache_init": (I, [P, P, P, P]),
        "dyllm_layer_step": (I, [P, P, P, I, I, P, P, F, P, P, P]),
        "dyllm_denoise_step": (I, [P, P, P, I, P, P, P, P, P]),
        "dyllm_full_step": (I, [P, P, P, P, P, P]),
        "dyllm_cache_tensor": (I, [P, I, I, PP, C.POINTER(C.c_int64)]),
        "dyllm_cache_copy": (I, [P, P, I, I, P, I, I]),
        "dyllm_cache_set_carried": (I, [P, P, P, P]),
        "dyllm_cache_refresh_stats": (I, [P, P, I]),
        "dyllm_cache_set_decoded": (I, [P, P, P]),
        "dyllm_cache_set_trace": (I, [P, P, P, P, P]),
        "dyllm_select_salient": (I, [P, I, I, I, I, P, P, F, I, P, P, P]),
        "dyllm_gemm_bf16": (I, [P, P, I, I, I, P, P, P, P, P]),
        "dyllm_unmask": (I, [P, P, P, P, P, P]),
        "dyllm_ctx_profile": (I, [P, I]),
        "dyllm_ctx_profile_read": (I, [P, I, P, I]),
        "dyllm_launch_count": (U64, []),
        "dyllm_set_option": (I, [I, I]),
        "dyllm_debug_trace_buffer": (I, [I, P]),
        "dyllm_tp_unique_id": (I, [P, I]),
        "dyllm_tp_create": (I, [P, I, I, P, PP]),
        "dyllm_tp_attach": (I, [P, I, P]),
        "dyllm_tp_cache_init": (I, [P, P, P]),
        "dyllm_tp_denoise_step": (I, [P, P, I, P, P, P, P, P]),
        "dyllm_tp_destroy": (None, [P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()
EXPORTED = [n for n in dir(_lib) if n.startswith("dyllm_")]


def lib():
    return _lib


OPT_SKINNY_GEMM, OPT_SKINNY_SPLIT, OPT_ATTN_FUSED, OPT_SKINNY_ONE_CHUNK, OPT_PDL, OPT_ATTN_INC, OPT_ATTN_T4 = 1, 2, 3, 4, 5, 6, 7
OPT_ATTN_PINC, OPT_ATTN_COS, OPT_SKINNY_CHUNK, OPT_SKINNY_KROT, OPT_SKINNY_DEBUG, OPT_SKINNY_KB = 8, 9, 10, 11, 12, 13
OPT_QKV_FUSED = 14


def set_option(option: int, value: int) -> int:
    """Process-wide kernel-path option; returns the previous value."""
    return _check(_lib.dyllm_set_option(option, value))


def _check(rc):
    if rc < 0:
        raise DyllmError(f"libdyllm status {rc}: {_lib.dyllm_last_error().decode()}")
    return rc


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_cuda:
            raise DyllmError("expected a CUDA tensor")
        return C.c_void_p(t.data_ptr())
    return t


class _CudaArray:
    """__cuda_array_interface__ wrapper: zero-copy torch view of a library-owned buffer."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 2, "strides": None}


def blob_from_weights(cfg, W) -> np.ndarray:
    """Pack synth/oracle-layout weights (bf16-representable floats) into the dyllm_weights_load blob."""
    from synth.gen import f32_to_bf16_bits
    parts = [W["emb"], W["g_final"], W["lm_head"]]
    for lw in W["layers"]:
        parts += [lw["g_attn"], lw["wq"], lw["wk"], lw["wv"]]
        if cfg.qkv_bias:
            parts += [lw["bq"], lw["bk"], lw["bv"]]
        parts += [lw["wo"], lw["g_ffn"], lw["w_gate"], lw["w_up"], lw["w_down"]]
    flat = np.concatenate([np.asarray(p, dtype=np.float32).ravel() for p in parts])
    return f32_to_bf16_bits(flat)


class Context:
    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        torch.cuda.set_device(device)
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = C.c_void_p()
        # The library launches on the caller's stream so its kernels are ordered with torch's
        # copies and events. torch's default stream has handle 0, which the ABI reads as "create
        # a private stream"; pass cudaStreamLegacy (0x1), the same legacy default stream, instead.
        handle = self.stream.cuda_stream or _CUDA_STREAM_LEGACY
        _check(_lib.dyllm_ctx_create(device, C.c_void_p(handle), C.byref(h)))
        self.h = h

    def sync(self):
        _check(_lib.dyllm_ctx_sync(self.h))

    def close(self):
        if self.h:
            _lib.dyllm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # instrumentation --------------------------------------------------------------------
    def profile(self, enable: bool):
        _check(_lib.dyllm_ctx_profile(self.h, int(enable)))

    def profile_read(self, kclass: int) -> np.ndarray:
        n = _check(_lib.dyllm_ctx_profile_read(self.h, kclass, None, 0))
        out = np.zeros(max(n, 1), dtype=np.float32)
        _check(_lib.dyllm_ctx_profile_read(self.h, kclass, out.ctypes.data_as(C.c_void_p), n))
        return out[:n]

    # kernel-level calls -----------------------------------------------------------------
    def select_salient(self, c_new, c_cache, row_lo, tau, cmp, idx_out, off_out, sim_out=None):
        b, N, w = c_new.shape
        _check(_lib.dyllm_select_salient(self.h, b, N, row_lo, w, _ptr(c_new), _ptr(c_cache),
                                         float(tau), cmp, _ptr(idx_out), _ptr(off_out), _ptr(sim_out)))

    def gemm_bf16(self, A, W, D, M_dev=None, resid=None, bias=None):
        M_cap, Kd = A.shape
        Nn = W.shape[0]
        _check(_lib.dyllm_gemm_bf16(self.h, _ptr(M_dev), M_cap, Nn, Kd, _ptr(A), _ptr(W), _ptr(D),
                                    _ptr(resid), _ptr(bias)))


class Weights:
    def __init__(self, ctx: Context, cfg, h):
        self.ctx, self.cfg, self.h = ctx, cfg, h

    @classmethod
    def from_blob(cls, ctx, cfg, blob: np.ndarray):
        mc = ModelCfg.from_py(cfg)
        blob = np.ascontiguousarray(blob, dtype=np.uint16)
        h = C.c_void_p()
        _check(_lib.dyllm_weights_load(ctx.h, C.byref(mc), blob.ctypes.data_as(C.c_void_p),
                                       blob.size, C.byref(h)))
        return cls(ctx, cfg, h)

    @classmethod
    def random(cls, ctx, cfg, seed: int, std: float | None = None):
        mc = ModelCfg.from_py(cfg)
        h = C.c_void_p()
        _check(_lib.dyllm_weights_init_random(ctx.h, C.byref(mc), seed,
                                              float(cfg.w_std if std is None else std), C.byref(h)))
        return cls(ctx, cfg, h)

    @staticmethod
    def blob_elems(cfg) -> int:
        return _lib.dyllm_weights_blob_elems(C.byref(ModelCfg.from_py(cfg)))

    def close(self):
        if self.h:
            _lib.dyllm_weights_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Cache:
    """Per-session activation caches (K, V, Q, C, H per layer + H_0) and step scratch."""

    def __init__(self, ctx: Context, w: Weights, run):
        self.ctx, self.w, self.run, self.cfg = ctx, w, run, w.cfg
        self.N = run.L_P + run.L_R
        rc = RunCfg.from_py(run)
        h = C.c_void_p()
        _check(_lib.dyllm_cache_create(ctx.h, w.h, C.byref(rc), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            _lib.dyllm_cache_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def init(self, tokens: torch.Tensor):
        _check(_lib.dyllm_cache_init(self.ctx.h, self.w.h, self.h, _ptr(tokens)))

    def layer_step(self, layer, input_mode, idx_in, off_in, tau, idx_out, off_out, sim_out=None):
        _check(_lib.dyllm_layer_step(self.ctx.h, self.w.h, self.h, layer, input_mode, _ptr(idx_in),
                                     _ptr(off_in), float(tau), _ptr(idx_out), _ptr(off_out),
                                     _ptr(sim_out)))

    def denoise_step(self, t, tau, tokens, dec_pos, dec_tok, sal_counts=None):
        taus = np.broadcast_to(np.asarray(tau, dtype=np.float32), (self.cfg.n_layers,)).copy()
        return _check(_lib.dyllm_denoise_step(self.ctx.h, self.w.h, self.h, t,
                                              taus.ctypes.data_as(C.c_void_p), _ptr(tokens),
                                              _ptr(dec_pos), _ptr(dec_tok), _ptr(sal_counts)))

    def full_step(self, tokens, dec_pos, dec_tok):
        _check(_lib.dyllm_full_step(self.ctx.h, self.w.h, self.h, _ptr(tokens), _ptr(dec_pos),
                                    _ptr(dec_tok)))

    def unmask(self, tokens, dec_pos, dec_tok):
        _check(_lib.dyllm_unmask(self.ctx.h, self.w.h, self.h, _ptr(tokens), _ptr(dec_pos), _ptr(dec_tok)))

    def refresh_stats(self, layer):
        _check(_lib.dyllm_cache_refresh_stats(self.ctx.h, self.h, layer))

    def set_carried(self, idx=None, off=None):
        _check(_lib.dyllm_cache_set_carried(self.ctx.h, self.h, _ptr(idx), _ptr(off)))

    def set_decoded(self, dec=None):
        _check(_lib.dyllm_cache_set_decoded(self.ctx.h, self.h, _ptr(dec)))

    def set_trace(self, lists=None, offs=None, sims=None):
        _check(_lib.dyllm_cache_set_trace(self.ctx.h, self.h, _ptr(lists), _ptr(offs), _ptr(sims)))

    def tensor(self, layer, which) -> torch.Tensor:
        """Zero-copy torch view of one cache tensor (bf16, fp32 in the fp32-parity mode; H: layer 0 =
        embeddings; STATS: float32
        [b][N][H][2]). A writable view: K / Q / STATS views invalidate the incremental statistics."""
        p = C.c_void_p()
        n = C.c_int64()
        _check(_lib.dyllm_cache_tensor(self.h, layer, which, C.byref(p), C.byref(n)))
        width = n.value // (self.run.batch * self.N)
        dev = f"cuda:{self.ctx.device}"
        if which == STATS:
            arr = _CudaArray(p.value, (self.run.batch, self.N, width, 2), "<f4")
            return torch.as_tensor(arr, device=dev)
        if getattr(self.cfg, "dtype", 0) == 1:      # fp32-parity mode
            return torch.as_tensor(_CudaArray(p.value, (self.run.batch, self.N, width), "<f4"), device=dev)
        arr = _CudaArray(p.value, (self.run.batch, self.N, width), "<i2")
        return torch.as_tensor(arr, device=dev).view(torch.bfloat16)

    def export(self, layer, which) -> torch.Tensor:
        """Read-only copy of one cache tensor (does not invalidate the statistics)."""
        b, N = self.run.batch, self.N
        dev = f"cuda:{self.ctx.device}"
        if which == STATS:
            out = torch.empty((b, N, self.cfg.n_heads, 2), dtype=torch.float32, device=dev)
        else:
            w = {K: self.cfg.kv_width, V: self.cfg.kv_width, Q: self.cfg.q_width, CTX: self.cfg.q_width,
                 H: self.cfg.d_model}[which]
            dt = torch.float32 if getattr(self.cfg, "dtype", 0) == 1 else torch.bfloat16
            out = torch.empty((b, N, w), dtype=dt, device=dev)
        _check(_lib.dyllm_cache_copy(self.ctx.h, self.h, layer, which, _ptr(out), 1, 1))
        return out

    def import_(self, layer, which, src: torch.Tensor):
        _check(_lib.dyllm_cache_copy(self.ctx.h, self.h, layer, which, _ptr(src.contiguous()), 1, 0))


from .dist import shard_weights  # noqa: E402,F401  (tensor-parallel shard slicing, host logic)


class TensorParallel:
    """A tensor-parallel group (dyllm_tp_*): loopback (every shard in this process, nccl_id None)
    or NCCL (this process is `rank` of `world`)."""

    def __init__(self, ctx: Context, world: int, rank: int = 0, nccl_id: bytes | None = None):
        self.ctx, self.world = ctx, world
        h = C.c_void_p()
        buf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _check(_lib.dyllm_tp_create(ctx.h, world, rank, buf, C.byref(h)))
        self.h = h
        self.caches = []

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_lib.dyllm_tp_unique_id(buf, 128))
        return buf.raw

    def attach(self, shard: int, cache: "Cache"):
        _check(_lib.dyllm_tp_attach(self.h, shard, cache.h))
        self.caches.append(cache)

    @staticmethod
    def _warr(weights):
        arr = (C.c_void_p * len(weights))(*[w.h.value for w in weights])
        return arr

    def init(self, weights, tokens):
        _check(_lib.dyllm_tp_cache_init(self.h, self._warr(weights), _ptr(tokens)))

    def denoise_step(self, weights, t, tau, tokens, dec_pos, dec_tok, sal_counts=None):
        n_layers = weights[0].cfg.n_layers
        taus = np.broadcast_to(np.asarray(tau, dtype=np.float32), (n_layers,)).copy()
        return _check(_lib.dyllm_tp_denoise_step(self.h, self._warr(weights), t, taus.ctypes.data_as(C.c_void_p),
                                                 _ptr(tokens), _ptr(dec_pos), _ptr(dec_tok), _ptr(sal_counts)))

    def close(self):
        if self.h:
            _lib.dyllm_tp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Engine:
    """Public generation API (Alg. 1): prompts in host memory -> generated tokens in host memory."""

    def __init__(self, ctx: Context, w: Weights, run):
        self.ctx, self.w, self.run, self.cfg = ctx, w, run, w.cfg
        self.cache = Cache(ctx, w, run)
        dev = f"cuda:{ctx.device}"
        b, N = run.batch, run.L_P + run.L_R
        self.tokens = torch.empty((b, N), dtype=torch.int32, device=dev)
        self.dec_pos = torch.empty((b, run.n_u), dtype=torch.int32, device=dev)
        self.dec_tok = torch.empty((b, run.n_u), dtype=torch.int32, device=dev)
        self.sal_counts = torch.zeros((run.T_total, self.cfg.n_layers, b), dtype=torch.int32, device=dev)

    def load_prompts(self, prompts_host: torch.Tensor):
        """prompts_host: [b][L_P] int32 (pinned for async copy). Builds Concat(P, [mask] * L_R)."""
        run = self.run
        self.tokens[:, run.L_P:].fill_(self.cfg.mask_id)
        self.tokens[:, :run.L_P].copy_(prompts_host, non_blocking=True)

    def run_steps(self, tau, full_recompute=False, record_counts=True):
        for t in range(self.run.T_total):
            if full_recompute:
                self.cache.full_step(self.tokens, self.dec_pos, self.dec_tok)
            else:
                self.cache.denoise_step(t, tau, self.tokens, self.dec_pos, self.dec_tok,
                                        self.sal_counts[t] if record_counts else None)

    def generate(self, prompts_host: torch.Tensor, tau, out_host: torch.Tensor | None = None,
                 full_recompute=False):
        self.load_prompts(prompts_host)
        self.run_steps(tau, full_recompute)
        if out_host is None:
            return self.tokens.cpu()
        out_host.copy_(self.tokens, non_blocking=True)
        return out_host
