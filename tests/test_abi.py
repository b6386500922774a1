"""C-ABI library: loads, exports every symbol include/specformer.h declares, host-only queries
(weight table, byte counts, config validation). No compute calls (CPU-only box)."""
import ctypes as C
import os
import re

import pytest

from paper_2511_20340_b200 import _native as N
from paper_2511_20340_b200 import build as B
from paper_2511_20340_b200.engine import EngineConfig, weight_table
from synth import get_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return N.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "specformer.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:sf|specformer)_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert {s for s, _, _ in N.SIGNATURES} == set(syms)
    assert b"sm_100a" in lib.specformer_build_info()


def _c(name, **kw):
    return EngineConfig.from_model(get_config(name), **kw).to_c()


@pytest.mark.parametrize("name", ["tiny", "small", "7b"])
def test_weight_table_layout(lib, name):
    m = get_config(name)
    cfg = EngineConfig.from_model(m)
    tab = weight_table(cfg)
    c = cfg.to_c()
    total = lib.sf_weights_bytes(C.byref(c))
    esz = 2 if m.dtype == "bf16" else 4
    prev_end = 0
    n_params = 0
    for nm, shape, off, dt, layout in tab:
        assert layout == (1 if (dt == N.SF_BF16 and nm != 'embed') else 0)
        assert off % 256 == 0 and off >= prev_end
        n = 1
        for s in shape:
            n *= s
        n_params += n
        prev_end = off + n * (esz if dt == N.SF_BF16 else 4)
    assert prev_end <= total
    names = [t[0] for t in tab]
    assert names[0] == "embed" and "lm_head" in names and "sf.w_p" in names
    # parameter count == base + SpecFormer head (qkv fused, gate/up interleaved: same counts)
    d, F, V, L, k = m.d_model, m.d_ff, m.vocab, m.n_layers, m.draft_len
    qkv = (m.n_heads + 2 * m.n_kv_heads) * m.head_dim
    attn = qkv * d + d * m.n_heads * m.head_dim
    base = 2 * V * d + L * (2 * d + attn + 3 * F * d) + d
    head = 4 * d + 4 * d * d + d + attn + d + k * d * d + k * d + d + attn + d + 3 * F * d
    assert n_params == base + head
    assert lib.sf_workspace_bytes(C.byref(c)) > 0


def test_draft_len_zero_table_has_no_head(lib):
    names = [t[0] for t in weight_table(EngineConfig.from_model(get_config("tiny"), draft_len=0))]
    assert not any(n.startswith("sf.") for n in names)


@pytest.mark.parametrize("field,value", [("rms_eps", 0.0), ("n_kv_heads", 3), ("kv_block", 8), ("max_seq", 100),
                                         ("tp_size", 2), ("head_dim", 48), ("dtype", 7), ("max_batch", 0)])
def test_invalid_configs_rejected(lib, field, value):
    c = _c("tiny")
    setattr(c, field, value)
    assert lib.sf_weights_bytes(C.byref(c)) == -1
    assert lib.sf_workspace_bytes(C.byref(c)) == -1
    h = C.c_void_p()
    assert lib.specformer_init(C.byref(c), C.c_void_p(256), C.c_void_p(256), None, C.byref(h)) == N.SF_ERR_ARG


def test_bf16_shape_constraints(lib):
    c = _c("small")
    c.vocab = 32001
    assert lib.sf_weights_bytes(C.byref(c)) == -1
    # bf16 head_dim 128: the flash-decoding attention folds at most 64 key segments of 2048 keys
    c = _c("7b")
    c.max_seq = 64 * 2048
    assert lib.sf_workspace_bytes(C.byref(c)) > 0
    c.max_seq = 64 * 2048 + 16
    assert lib.sf_workspace_bytes(C.byref(c)) == -1


def test_null_handle_calls(lib):
    assert lib.specformer_draft_step(None, None, None) == N.SF_ERR_ARG
    assert lib.specformer_sync(None) == N.SF_ERR_ARG
    assert lib.specformer_kernel_launches(None) == -1
    lib.specformer_destroy(None)


def test_draft_blocks_table(lib):
    """NEXT-2 "+Larger": extra draft blocks appear as sf.blk<i>_* with the block's shapes."""
    m = get_config("small").replace(draft_blocks=3)
    tab = {n: s for n, s, *_ in weight_table(EngineConfig.from_model(m))}
    for i in (1, 2):
        b = f"sf.blk{i}_"
        assert tab[b + "wqkv"] == tab["sf.blk_wqkv"] and tab[b + "w_down"] == tab["sf.blk_w_down"]
        assert tab[b + "attn_norm"] == (m.d_model,)
    assert not any(n.startswith("sf.blk3_") for n in tab)
    c = EngineConfig.from_model(m).to_c()
    c.draft_blocks = 5
    assert lib.sf_weights_bytes(C.byref(c)) == -1
