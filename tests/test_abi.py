"""CPU checks of the C-ABI boundary: the library builds/loads, exports every symbol that
include/dyllm.h declares, and validates host-side arguments without touching a GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dyllm.h")
LIB = os.path.join(ROOT, "paper_2603_08026_b200", "libdyllm.so")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dyllm_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2603_08026_b200 import build
        build.build()
    return C.CDLL(LIB)


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("dyllm_cache_init", "dyllm_layer_step", "dyllm_denoise_step", "dyllm_full_step",
              "dyllm_select_salient", "dyllm_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_loads_and_covers_the_abi():
    from paper_2603_08026_b200 import dyllm
    assert dyllm.lib().dyllm_version() == 100
    assert set(_declared()) <= set(dir(dyllm.lib())) | set(dyllm.EXPORTED)


def test_blob_size_and_shape_validation_on_host():
    from paper_2603_08026_b200 import dyllm
    from synth import configs
    for name in ("tiny", "small128", "small128_gqa", "llada8b", "dream7b"):
        cfg, _ = configs.preset(name)
        n = dyllm.Weights.blob_elems(cfg)
        d, qw, kw, F, V = cfg.d_model, cfg.q_width, cfg.kv_width, cfg.d_ff, cfg.vocab
        per = d + qw * d + 2 * kw * d + (qw + 2 * kw if cfg.qkv_bias else 0) + d * qw + d + 3 * F * d
        assert n == 2 * V * d + d + per * cfg.n_layers
    from dataclasses import replace
    bad = replace(configs.TINY, head_dim=24, n_heads=2)     # head_dim not in {16,32,64,128}
    assert dyllm.Weights.blob_elems(bad) == -1
    assert b"head_dim" in dyllm.lib().dyllm_last_error()


def test_blob_layout_matches_header_order():
    from paper_2603_08026_b200 import dyllm
    from synth import configs, gen
    cfg, _ = configs.preset("tiny")
    W = gen.model_weights(cfg, 0)
    blob = dyllm.blob_from_weights(cfg, W)
    assert blob.size == dyllm.Weights.blob_elems(cfg)
    d, V = cfg.d_model, cfg.vocab
    assert (gen.bf16_bits_to_f32(blob[:V * d]).reshape(V, d) == W["emb"]).all()
    off = 2 * V * d + d + d                      # emb, g_final, lm_head, layer0.g_attn
    wq = gen.bf16_bits_to_f32(blob[off:off + cfg.q_width * d]).reshape(cfg.q_width, d)
    assert (wq == W["layers"][0]["wq"]).all()


def test_no_gpu_calls_fail_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_08026_b200 import dyllm
    h = C.c_void_p()
    rc = dyllm.lib().dyllm_ctx_create(0, None, C.byref(h))
    assert rc == -5 and dyllm.lib().dyllm_last_error()
