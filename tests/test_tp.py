"""Tensor-parallel host logic (no GPU): the per-rank weight tables the library reports, the
vocabulary split, and the weight slicing of engine.pack_weights -- checked against the algebra the
split must preserve (column-parallel QKV / gate-up, row-parallel O / down / W_D,
vocabulary-parallel LM head)."""
import ctypes as C

import pytest
import torch

from paper_2511_20340_b200 import _native as N
from paper_2511_20340_b200 import build as B
from paper_2511_20340_b200.engine import EngineConfig, _source_tensor, weight_table
from synth import get_config, make_weights

GQA = get_config("70b").replace(name="70b-narrow", n_layers=2, d_model=512, n_heads=8, n_kv_heads=4,
                                d_ff=1024, vocab=4096, batch=2, prompt_len=32, gen_len=8)


@pytest.fixture(scope="module")
def lib():
    B.build()
    return N.load()


def _cfg(tp, r, m=GQA):
    return EngineConfig.from_model(m, max_batch=2, max_seq=128, tp_size=tp, tp_rank=r)


@pytest.mark.parametrize("tp", [2, 4])
def test_rank_tables_and_vocab_split(lib, tp):
    full = {n: s for n, s, *_ in weight_table(_cfg(1, 0))}
    covered = []
    for r in range(tp):
        cfg = _cfg(tp, r)
        tab = {n: s for n, s, *_ in weight_table(cfg)}
        assert set(tab) == set(full)
        hq, hkv, hd, F, d = GQA.n_heads // tp, GQA.n_kv_heads // tp, GQA.head_dim, GQA.d_ff // tp, GQA.d_model
        assert tab["layers.0.wqkv"] == ((hq + 2 * hkv) * hd, d)
        assert tab["layers.0.wo"] == (d, hq * hd)
        assert tab["layers.1.w_gu"] == (2 * F, d) and tab["layers.1.w_down"] == (d, F)
        assert tab["sf.w_d"] == (d, 4 * d // tp)
        for n in ("embed", "sf.w_p", "sf.b_p", "final_norm", "layers.0.attn_norm"):
            assert tab[n] == full[n]
        v0, v1 = cfg.vocab_shard()
        assert tab["lm_head"] == (v1 - v0, d) and v0 % 128 == 0 and v1 % 128 == 0
        covered.append((v0, v1))
        c = cfg.to_c()
        assert lib.sf_weights_bytes(C.byref(c)) > 0 and lib.sf_workspace_bytes(C.byref(c)) > 0
    assert covered[0][0] == 0 and covered[-1][1] == GQA.vocab
    assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))


@pytest.mark.parametrize("field,value", [("tp_size", 3), ("tp_rank", 2), ("tp_rank", -1)])
def test_invalid_tp_configs(lib, field, value):
    c = _cfg(2, 0).to_c()
    setattr(c, field, value)
    assert lib.sf_weights_bytes(C.byref(c)) == -1


def test_tp_needs_bf16(lib):
    c = EngineConfig.from_model(get_config("tiny"), tp_size=2, tp_rank=0).to_c()
    assert lib.sf_weights_bytes(C.byref(c)) == -1


def test_slices_preserve_the_layer_algebra():
    """Column-parallel pieces concatenate to the full projection; row-parallel pieces sum to it."""
    torch.manual_seed(0)
    w = {k: v.double() for k, v in make_weights(GQA.replace(dtype="fp32"), seed=3).items()}
    tp, d, hd = 2, GQA.d_model, GQA.head_dim
    x = torch.randn(5, d, dtype=torch.float64)
    # column-parallel q|k|v: rank r's rows = its q heads, then its kv heads (rope_pairs off)
    q = x @ w["layers.0.wq"].T
    k = x @ w["layers.0.wk"].T
    outs = [x @ _source_tensor("layers.0.wqkv", w, 0, _cfg(tp, r)).T for r in range(tp)]
    hq, hkv = GQA.n_heads // tp * hd, GQA.n_kv_heads // tp * hd
    assert torch.allclose(torch.cat([o[:, :hq] for o in outs], 1), q)
    assert torch.allclose(torch.cat([o[:, hq:hq + hkv] for o in outs], 1), k)
    # row-parallel O: sum over ranks of (rank's heads of the attention output) @ (rank's O columns)
    a = torch.randn(5, GQA.n_heads * hd, dtype=torch.float64)
    full = a @ w["layers.0.wo"].T
    part = sum(a[:, r * hq:(r + 1) * hq] @ _source_tensor("layers.0.wo", w, 0, _cfg(tp, r)).T for r in range(tp))
    assert torch.allclose(part, full)
    # gate/up: rank r's interleaved rows are (gate_i, up_i) for its FFN rows; down columns match them
    F = GQA.d_ff // tp
    for r in range(tp):
        gu = _source_tensor("layers.1.w_gu", w, 0, _cfg(tp, r))
        assert torch.equal(gu[0::2], w["layers.1.w_gate"][r * F:(r + 1) * F])
        assert torch.equal(gu[1::2], w["layers.1.w_up"][r * F:(r + 1) * F])
    h = torch.randn(5, GQA.d_ff, dtype=torch.float64)
    full = h @ w["layers.1.w_down"].T
    part = sum(h[:, r * F:(r + 1) * F] @ _source_tensor("layers.1.w_down", w, 0, _cfg(tp, r)).T for r in range(tp))
    assert torch.allclose(part, full)
    # W_D over I_Cat's column blocks; LM head over vocabulary rows
    icat = torch.randn(5, 4 * d, dtype=torch.float64)
    part = sum(icat[:, r * 4 * d // tp:(r + 1) * 4 * d // tp] @ _source_tensor("sf.w_d", w, 0, _cfg(tp, r)).T
               for r in range(tp))
    assert torch.allclose(part, icat @ w["sf.w_d"].T)
    logits = torch.cat([x @ _source_tensor("lm_head", w, 0, _cfg(tp, r)).T for r in range(tp)], 1)
    assert torch.allclose(logits, x @ w["lm_head"].T)
