"""Pins of the fp64 oracle against things other than itself (CPU only).

Each pin cites what fixes the expected value: a closed form, a SPEC.md / PAPER.md
worked example (tests/golden/paper_values.json), a brute-force scalar loop, or an
invariant of the method (causality, residual identities, losslessness).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from oracle import analytics as A
from synth import get_config, make_weights, make_prompts

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))

# micro config: GQA (Hq=2, Hkv=1) and Hq*hd != d so a transposed operand fails on shape
MICRO = get_config("tiny").replace(name="micro", n_layers=2, d_model=12, n_heads=2, n_kv_heads=1,
                                   head_dim=4, d_ff=20, vocab=37, draft_len=3, prompt_len=5, gen_len=12)


def W_of(cfg, seed=0, jitter=0.0, **kw):
    return O.Weights(cfg, make_weights(cfg, seed=seed, norm_jitter=jitter, **kw))


# ------------------------------------------------------------------ primitives
def test_rms_norm_spec_example():
    g = GOLD["rms_norm_example"]
    y = O.rms_norm(np.array(g["x"]), np.ones(2), g["eps"])
    np.testing.assert_allclose(y, g["y"], atol=g["tol"])


def test_rms_norm_zero_and_unit_rms():
    assert np.all(O.rms_norm(np.zeros(8), np.full(8, 3.0), 1e-6) == 0)
    x = np.random.default_rng(0).normal(size=(5, 33))
    y = O.rms_norm(x, np.ones(33), 1e-12)
    np.testing.assert_allclose(np.sqrt(np.mean(y * y, axis=-1)), 1.0, atol=1e-9)
    # scale applies elementwise after normalisation
    g = np.arange(1, 34, dtype=float)
    np.testing.assert_allclose(O.rms_norm(x, g, 1e-12), y * g, rtol=1e-12)


def test_group_rms_norm_reduces_to_rms_and_zero_slice():
    rng = np.random.default_rng(1)
    taps = rng.normal(size=(4, 3, 8))
    taps[2] = 0.0
    s = rng.normal(size=(4, 8))
    out = O.group_rms_norm(taps, s, 1e-6)
    assert out.shape == (3, 32)
    for g in range(4):
        sl = out[:, 8 * g: 8 * (g + 1)]
        if g == 2:
            assert np.all(sl == 0)
        else:  # closed form per slice: x * s / sqrt(mean x^2 + eps), written with explicit loops
            for t in range(3):
                ms = sum(v * v for v in taps[g, t]) / 8
                exp = [taps[g, t, i] * s[g, i] / math.sqrt(ms + 1e-6) for i in range(8)]
                np.testing.assert_allclose(sl[t], exp, rtol=1e-13)


def test_softmax_stability_and_attention_brute_force():
    # SPEC S75: softmax [1000, 0] -> [1, 0] without overflow, via scores q.k/sqrt(hd)
    q = np.array([[1000.0]])
    k = np.array([[1.0], [0.0]])
    v = np.array([[7.0], [-3.0]])
    out = O.attention_dense_masked(q, k, v, np.ones((1, 2), bool))
    assert abs(out[0, 0] - 7.0) < 1e-12
    # brute force scalar loops on a random masked problem
    rng = np.random.default_rng(2)
    q, k, v = rng.normal(size=(3, 4)), rng.normal(size=(6, 4)), rng.normal(size=(6, 5))
    mask = rng.random((3, 6)) < 0.6
    mask[:, 0] = True
    out = O.attention_dense_masked(q, k, v, mask)
    for i in range(3):
        w = [math.exp(sum(q[i, t] * k[j, t] for t in range(4)) / 2.0) if mask[i, j] else 0.0 for j in range(6)]
        z = sum(w)
        for c in range(5):
            assert abs(out[i, c] - sum(w[j] * v[j, c] for j in range(6)) / z) < 1e-12


def test_attention_singleton_uniform_and_full_mask():
    # S83: single query == single key -> v; S85: uniform q,k -> mean of unmasked v
    assert O.attention_dense_masked(np.ones((1, 3)), np.ones((1, 3)), np.array([[7.0, 1, 2]]),
                                    np.ones((1, 1), bool))[0, 0] == 7.0
    v = np.arange(12.0).reshape(4, 3)
    mask = np.array([[True, True, False, True]])
    out = O.attention_dense_masked(np.ones((1, 3)), np.ones((4, 3)), v, mask)
    np.testing.assert_allclose(out[0], v[[0, 1, 3]].mean(axis=0), rtol=1e-14)
    with pytest.raises(ValueError):
        O.attention_dense_masked(np.ones((1, 3)), np.ones((2, 3)), np.ones((2, 3)), np.zeros((1, 2), bool))


def test_rope_closed_forms():
    rng = np.random.default_rng(3)
    x = rng.normal(size=(5, 2, 8))
    pos = np.array([0, 1, 2, 7, 100])
    y = O.rope(x, pos, 10000.0)
    np.testing.assert_allclose(y[0], x[0], rtol=0, atol=0)                      # position 0: identity
    np.testing.assert_allclose(np.linalg.norm(y, axis=-1), np.linalg.norm(x, axis=-1), rtol=1e-13)
    # explicit 2-D rotation of pair (i, i+4) by pos * theta^(-2i/8)
    for t in range(5):
        for i in range(4):
            a = pos[t] * 10000.0 ** (-2 * i / 8)
            assert abs(y[t, 0, i] - (x[t, 0, i] * math.cos(a) - x[t, 0, i + 4] * math.sin(a))) < 1e-12
            assert abs(y[t, 0, i + 4] - (x[t, 0, i + 4] * math.cos(a) + x[t, 0, i] * math.sin(a))) < 1e-12
    # relative-position property: <R_m q, R_n k> depends on m - n only
    q, k = rng.normal(size=(1, 1, 8)), rng.normal(size=(1, 1, 8))
    d1 = (O.rope(q, [9], 1e4) * O.rope(k, [4], 1e4)).sum()
    d2 = (O.rope(q, [105], 1e4) * O.rope(k, [100], 1e4)).sum()
    assert abs(d1 - d2) < 1e-12


def test_swiglu_closed_form():
    assert np.all(O.swiglu(np.zeros((1, 3)), np.ones((4, 3)), np.ones((4, 3)), np.ones((3, 4))) == 0)
    # scalar case: w_down * silu(a x) * (b x)
    a, b, c, x = 0.7, -1.3, 2.0, 1.1
    exp = c * (a * x / (1 + math.exp(-a * x))) * (b * x)
    got = O.swiglu(np.array([[x]]), np.array([[a]]), np.array([[b]]), np.array([[c]]))[0, 0]
    assert abs(got - exp) < 1e-14


def test_argmax_ties_and_nonfinite():
    assert O.argmax_lowest([0.3, 0.7]) == 1
    assert O.argmax_lowest([0.5, 0.5]) == 0
    assert O.argmax_lowest([-1e300, -1e300, 4.0, 4.0]) == 2
    with pytest.raises(FloatingPointError):
        O.argmax_lowest([0.0, float("nan")])


def test_taps_index():
    assert O.taps_index(2) == (0, 1, 1, 2)     # Tiny: duplicated tap (reading C1)
    assert O.taps_index(32) == (0, 16, 31, 32)
    assert O.taps_index(5) == (0, 2, 4, 5)


@pytest.mark.parametrize("ex", GOLD["accept_examples"])
def test_accept_spec_examples(ex):
    m, em = O.accept(ex["draft"], ex["greedy"])
    assert m == ex["m"] and em == ex["emitted"]


# ------------------------------------------------------------------ base model
def test_base_forward_single_token_closed_form():
    """T=1 at position 0: softmax over one key is 1, so the attention sub-block is
    W_o W_v RMS(h) (GQA: every q head reads kv head 0), RoPE does not touch v."""
    cfg = MICRO.replace(n_layers=1)
    W = W_of(cfg, jitter=0.1)
    cache = O.KVCache(2, cfg.n_kv_heads, cfg.head_dim)
    tok = 5
    logits, taps = O.base_forward(W, [tok], 0, cache)
    h0 = W["embed"][tok]
    x = h0 / math.sqrt(np.mean(h0 ** 2) + cfg.rms_eps) * W["layers.0.attn_norm"]
    v = [sum(W["layers.0.wv"][j, i] * x[i] for i in range(cfg.d_model)) for j in range(cfg.head_dim)]
    att = np.concatenate([v, v])  # Hq=2 heads share kv head 0
    h1 = h0 + np.array([sum(W["layers.0.wo"][r, j] * att[j] for j in range(8)) for r in range(cfg.d_model)])
    x2 = h1 / math.sqrt(np.mean(h1 ** 2) + cfg.rms_eps) * W["layers.0.ffn_norm"]
    gate = W["layers.0.w_gate"] @ x2
    up = W["layers.0.w_up"] @ x2
    h2 = h1 + W["layers.0.w_down"] @ (gate / (1 + np.exp(-gate)) * up)
    np.testing.assert_allclose(taps[0, 0], h0, rtol=1e-14)
    np.testing.assert_allclose(taps[3, 0], h2, rtol=1e-12, atol=1e-15)
    hf = h2 / math.sqrt(np.mean(h2 ** 2) + cfg.rms_eps) * W["final_norm"]
    np.testing.assert_allclose(logits[0], W["lm_head"] @ hf, rtol=1e-11, atol=1e-15)


def test_base_incremental_equals_full_and_causality():
    cfg = MICRO
    W = W_of(cfg, seed=3)
    toks = [3, 9, 1, 30, 7, 2]
    c1 = O.KVCache(3, 1, 4)
    full, taps_full = O.base_forward(W, toks, 0, c1)
    c2 = O.KVCache(3, 1, 4)
    a, _ = O.base_forward(W, toks[:4], 0, c2)
    b, taps_b = O.base_forward(W, toks[4:], 4, c2)
    np.testing.assert_allclose(np.vstack([a, b]), full, rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(taps_b, taps_full[:, 4:], rtol=1e-11, atol=1e-14)
    # causality probe (S179): changing token 4 leaves logits < 4 unchanged
    c3 = O.KVCache(3, 1, 4)
    pert, _ = O.base_forward(W, toks[:4] + [11, 2], 0, c3)
    np.testing.assert_array_equal(pert[:4], full[:4])
    assert not np.allclose(pert[4:], full[4:])


def test_truncate_then_extend_equals_fresh_prefill():
    cfg = MICRO
    W = W_of(cfg, seed=4)
    c = O.KVCache(3, 1, 4)
    O.base_forward(W, [1, 2, 3, 4, 5, 6, 7], 0, c)
    c.truncate(range(2), 4)
    x, _ = O.base_forward(W, [8, 9], 4, c)
    c2 = O.KVCache(3, 1, 4)
    y, _ = O.base_forward(W, [1, 2, 3, 4, 8, 9], 0, c2)
    np.testing.assert_allclose(x, y[4:], rtol=1e-11, atol=1e-14)


def test_residual_identity_zero_outputs():
    """All W_o and W_down zero => every HS equals the embedding (Eq.7 residual)."""
    cfg = MICRO
    w = make_weights(cfg, seed=5)
    for l in range(cfg.n_layers):
        w[f"layers.{l}.wo"].zero_()
        w[f"layers.{l}.w_down"].zero_()
    W = O.Weights(cfg, w)
    logits, taps = O.base_forward(W, [4, 5, 6], 0, O.KVCache(3, 1, 4))
    for g in range(4):
        np.testing.assert_array_equal(taps[g], W["embed"][[4, 5, 6]])


# ------------------------------------------------------------------ SpecFormer pieces
def test_context_layer_zero_wo_and_causality():
    cfg = MICRO
    w = make_weights(cfg, seed=6, norm_jitter=0.1)
    W = O.Weights(cfg, w)
    rng = np.random.default_rng(6)
    taps = rng.normal(size=(4, 5, cfg.d_model))
    c = O.KVCache(3, 1, 4)
    i_d = O.context_layer(W, taps, 0, c)
    # causality (S266): perturbing row 4 leaves rows 0..3 unchanged
    taps2 = taps.copy()
    taps2[:, 4] += 1.0
    i_d2 = O.context_layer(W, taps2, 0, O.KVCache(3, 1, 4))
    np.testing.assert_array_equal(i_d[:4], i_d2[:4])
    # S265: zero MSA output projection => I_D = W_D I_Cat (explicit loops)
    w["sf.ctx_wo"].zero_()
    W0 = O.Weights(cfg, w)
    i_d0 = O.context_layer(W0, taps, 0, O.KVCache(3, 1, 4))
    icat = O.group_rms_norm(taps, W0["sf.group_scale"], cfg.rms_eps)
    for t in range(5):
        for r in range(cfg.d_model):
            assert abs(i_d0[t, r] - sum(W0["sf.w_d"][r, j] * icat[t, j] for j in range(4 * cfg.d_model))) < 1e-13


def test_positional_ffn_zero_weight_and_slices():
    cfg = MICRO
    w = make_weights(cfg, seed=7)
    W = O.Weights(cfg, w)
    i_d = np.random.default_rng(7).normal(size=cfg.d_model)
    D = O.positional_ffn(W, i_d)
    assert D.shape == (cfg.draft_len, cfg.d_model)
    x = O.rms_norm(i_d, W["sf.pos_norm"], cfg.rms_eps)
    d = cfg.d_model
    for j in range(cfg.draft_len):   # slot j = rows [j d, (j+1) d) of W_P (S276)
        np.testing.assert_allclose(D[j], W["sf.w_p"][j * d:(j + 1) * d] @ x + W["sf.b_p"][j * d:(j + 1) * d],
                                   rtol=1e-13)
    w["sf.w_p"].zero_()
    D0 = O.positional_ffn(O.Weights(cfg, w), i_d)
    np.testing.assert_array_equal(D0, W["sf.b_p"].reshape(cfg.draft_len, d))   # S274


def test_draft_block_identity_and_permutation_equivariance():
    cfg = MICRO
    w = make_weights(cfg, seed=8, norm_jitter=0.1)
    W = O.Weights(cfg, w)
    D = np.random.default_rng(8).normal(size=(cfg.draft_len, cfg.d_model))
    E = O.draft_block(W, D)
    perm = [2, 0, 1]
    np.testing.assert_allclose(O.draft_block(W, D[perm]), E[perm], rtol=1e-12, atol=1e-14)  # S284
    w["sf.blk_wo"].zero_()
    w["sf.blk_w_down"].zero_()
    np.testing.assert_array_equal(O.draft_block(O.Weights(cfg, w), D), D)          # S283


def test_draft_block_slot_causal_ablation():
    """"+Att Mask" (T4, P497-514): with the slot-causal mask, slot j ignores later slots (perturbing
    the last slot leaves the others unchanged), slot 0 is the block applied to slot 0 alone (a k = 1
    block, where causal and bidirectional coincide), and the last slot sees the same keys as the
    unmasked block (so its output equals the bidirectional block's last row)."""
    cfg = MICRO
    W = O.Weights(cfg, make_weights(cfg, seed=8, norm_jitter=0.1))
    D = np.random.default_rng(11).normal(size=(cfg.draft_len, cfg.d_model))
    Ec = O.draft_block(W, D, slot_causal=True)
    D2 = D.copy()
    D2[-1] += 1.0
    Ec2 = O.draft_block(W, D2, slot_causal=True)
    np.testing.assert_array_equal(Ec2[:-1], Ec[:-1])
    assert not np.allclose(Ec2[-1], Ec[-1])
    np.testing.assert_allclose(Ec[:1], O.draft_block(W, D[:1]), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(Ec[-1], O.draft_block(W, D)[-1], rtol=1e-12, atol=1e-14)
    assert not np.allclose(Ec[0], O.draft_block(W, D)[0])


def test_draft_blocks_larger_ablation():
    """"+Larger" (T4, P497-514) read as stacked draft blocks: a second block whose output projections
    are zero is the identity (so two blocks reduce to one), and a second block equals applying the
    one-block function with that block's weights to the first block's output."""
    cfg2 = MICRO.replace(draft_blocks=2)
    w = make_weights(cfg2, seed=8, norm_jitter=0.1)
    D = np.random.default_rng(12).normal(size=(cfg2.draft_len, cfg2.d_model))
    E1 = O.draft_block(O.Weights(MICRO, w), D)
    E2 = O.draft_block(O.Weights(cfg2, w), D)
    assert not np.allclose(E1, E2)
    moved = {k.replace("sf.blk1_", "sf.blk_"): v for k, v in w.items() if k.startswith("sf.blk1_")}
    np.testing.assert_allclose(E2, O.draft_block(O.Weights(MICRO, {**w, **moved}), E1), rtol=1e-12, atol=1e-14)
    w["sf.blk1_wo"].zero_()
    w["sf.blk1_w_down"].zero_()
    np.testing.assert_array_equal(O.draft_block(O.Weights(cfg2, w), D), E1)


def test_draft_logits_shape_and_constant_case():
    cfg = MICRO
    W = W_of(cfg, seed=9)
    dl = O.draft_logits(W, np.random.default_rng(9).normal(size=cfg.d_model))
    assert dl.shape == (cfg.draft_len, cfg.vocab)
    assert len(O.draft_tokens(W, np.ones(cfg.d_model))) == cfg.draft_len


# ------------------------------------------------------------------ losslessness
def _regime_fn(regime, W, prompt, N, k, V):
    if regime == "specformer":
        return None
    ar = O.decode_greedy(W, prompt, N + k + 2)
    if regime == "perfect":
        # the token at position n+1+j (j=1..k) is AR token index (n - P) + 1 + j
        return lambda s, n, out: [ar[n - len(prompt) + j] for j in range(1, k + 1)]
    # adversarial: always wrong at slot 1
    return lambda s, n, out: [(ar[n - len(prompt) + 1] + 1) % V] + [0] * (k - 1)


@pytest.mark.parametrize("cfgname", ["tiny", "micro"])
@pytest.mark.parametrize("regime", ["specformer", "perfect", "adversarial"])
def test_sd_equals_ar_many_seeds(cfgname, regime):
    """P25-26 losslessness: SD output == AR greedy output exactly, for any drafts
    (S380, S394). 17 weight seeds per regime (SPEC acceptance #1)."""
    cfg = get_config("tiny") if cfgname == "tiny" else MICRO
    N = 32 if cfgname == "tiny" else 12
    k = cfg.draft_len
    for seed in range(17):
        W = W_of(cfg, seed=seed, jitter=0.1 if seed % 2 else 0.0)
        prompt = make_prompts(1, cfg.prompt_len, cfg.vocab, seed=100 + seed)[0].tolist()
        ar = O.decode_greedy(W, prompt, N)
        fn = _regime_fn(regime, W, prompt, N, k, cfg.vocab)
        sd, steps = O.sd_decode(W, prompt, N, draft_fn=fn)
        assert sd == ar, (seed, regime)
        if regime == "perfect":   # reading C11: ceil((N-1)/(k+1)) steps
            assert len(steps) == math.ceil((N - 1) / (k + 1))
            assert all(s["m"] == k for s in steps)
        if regime == "adversarial":
            assert len(steps) == N - 1 and all(s["m"] == 0 for s in steps)


def test_replay_matches_free_run_and_a_definition():
    cfg = get_config("tiny")
    W = W_of(cfg, seed=1)
    prompt = make_prompts(1, cfg.prompt_len, cfg.vocab)[0].tolist()
    toks, steps = O.sd_decode(W, prompt, cfg.gen_len, record=True)
    traj = []
    last = None
    g0 = O.decode_greedy(W, prompt, 1)[0]
    last = g0
    for s in steps:
        traj.append(dict(draft=s["draft"], m=s["m"], last=last))
        last = s["greedy"][s["m"]]
    _, rep = O.replay(W, prompt, traj)
    for s, r in zip(steps, rep):
        assert s["greedy"] == r["greedy"]
        np.testing.assert_allclose(s["logits"], r["logits"], rtol=0, atol=0)
    # a = 1 + mean(m) (S397) and kappa = a when k = l_d (Eq.5)
    a = sum(s["m"] + 1 for s in steps) / len(steps)
    assert A.kappa(a, cfg.draft_len, cfg.draft_len) == pytest.approx(a)
