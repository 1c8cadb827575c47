"""Model / run shapes for the BASELINE.json configs (SURVEY.md §8 "Config symbols").

Values the paper does not give (vocab, mask id, rope theta, eps, tiny-config
schedule) are the builder's readings, listed in DESIGN.md §2.
"""
from __future__ import annotations

from dataclasses import dataclass, replace, asdict


@dataclass(frozen=True)
class ModelCfg:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int
    mask_id: int
    rope_theta: float
    rms_eps: float
    qkv_bias: bool = False
    residual_mode: int = 0      # 0 = pre-norm residual block (LLaDA/Dream), 1 = paper_literal Alg.2/3
    w_std: float = 0.02         # std of every projection / embedding / lm-head weight
    qk_std: float = 0.0         # std of W_q / W_k (0 -> w_std); the sigma_qk sharpness knob
    lm_std: float = 0.0         # std of the LM head (0 -> w_std); > w_std gives distinct confidences (tests)
    dtype: int = 0              # 0 = bf16 storage (the product path); 1 = fp32-parity mode (DESIGN D12)
    name: str = ""

    @property
    def kv_width(self) -> int:
        return self.n_kv_heads * self.head_dim

    @property
    def q_width(self) -> int:
        return self.n_heads * self.head_dim

    def as_dict(self):
        return asdict(self)


@dataclass(frozen=True)
class RunCfg:
    batch: int
    L_P: int
    L_R: int
    block: int = 32             # semi-AR block size B
    n_u: int = 1                # tokens unmasked per step
    T_full: int = 4             # warm-up FullSteps
    full_period: int = 4        # full-input sparse step when t % period == 0
    layer1_policy: int = 1      # 0 = carried (Alg.1 literal), 1 = carried ∪ decoded (DESIGN D5)
    cmp: int = 0                # 0 = strict '<' (Alg.3), 1 = '<=' (§3.2)
    select_mode: int = 0        # 0 = fixed threshold tau (paper); 1 = per-sequence fraction f (D19)

    @property
    def N(self) -> int:
        return self.L_P + self.L_R

    @property
    def T_total(self) -> int:
        return -(-self.L_R // self.n_u)

    def as_dict(self):
        return asdict(self)


TINY = ModelCfg(n_layers=2, d_model=64, n_heads=4, n_kv_heads=4, head_dim=16, d_ff=256,
                vocab=512, mask_id=511, rope_theta=1e4, rms_eps=1e-6, name="tiny")
TINY_RUN = RunCfg(batch=1, L_P=16, L_R=16, block=8, n_u=4, T_full=1, full_period=2)

SMALL128 = ModelCfg(n_layers=2, d_model=256, n_heads=2, n_kv_heads=2, head_dim=128, d_ff=768,
                    vocab=512, mask_id=511, rope_theta=5e5, rms_eps=1e-5, name="small128")
SMALL128_GQA = replace(SMALL128, n_kv_heads=1, qkv_bias=True, rope_theta=1e6, rms_eps=1e-6,
                       name="small128_gqa")
SMALL64 = ModelCfg(n_layers=2, d_model=256, n_heads=4, n_kv_heads=2, head_dim=64, d_ff=768,
                   vocab=512, mask_id=511, rope_theta=1e4, rms_eps=1e-6, name="small64")
SMALL128_RUN = RunCfg(batch=2, L_P=96, L_R=64, block=32, n_u=1, T_full=4, full_period=4)

LLADA8B = ModelCfg(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=32, head_dim=128,
                   d_ff=12288, vocab=126464, mask_id=126336, rope_theta=5e5, rms_eps=1e-5,
                   name="llada8b")
LLADA8B_RUN = RunCfg(batch=16, L_P=700, L_R=256, block=32, n_u=1, T_full=4, full_period=4)

DREAM7B = ModelCfg(n_layers=28, d_model=3584, n_heads=28, n_kv_heads=4, head_dim=128,
                   d_ff=18944, vocab=152064, mask_id=151666, rope_theta=1e6, rms_eps=1e-6,
                   qkv_bias=True, name="dream7b")
DREAM7B_RUN = RunCfg(batch=16, L_P=160, L_R=512, block=32, n_u=1, T_full=4, full_period=4)

PRESETS = {
    "tiny": (TINY, TINY_RUN),
    "small128": (SMALL128, SMALL128_RUN),
    "small128_gqa": (SMALL128_GQA, SMALL128_RUN),
    "small64": (SMALL64, SMALL128_RUN),
    "llada8b": (LLADA8B, LLADA8B_RUN),
    "dream7b": (DREAM7B, DREAM7B_RUN),
}


def preset(name: str):
    return PRESETS[name]
