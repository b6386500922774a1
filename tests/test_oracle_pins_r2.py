"""More pins of the fp64 oracle (CPU only): the top-1/top-2 margin rule, the GQA q -> kv head
grouping at Hq = 4 / Hkv = 2, and reading C14 (the next draft's context row after a commit of
m > 0 tokens equals the last row of a fresh prefill over the committed sequence)."""
import math

import numpy as np
import pytest

import oracle as O
import oracle.model as OM
from synth import get_config, make_prompts, make_weights


# ------------------------------------------------------------------ top2_margin (reading C21)
def test_top2_margin_closed_forms():
    # the margin is top-1 minus top-2 of the row, wherever they sit
    assert O.top2_margin([1.0, 3.0, 2.0]) == 1.0
    assert O.top2_margin([3.0, -5.0, 2.5, 0.0]) == 0.5
    assert O.top2_margin([-1.0, -4.0]) == 3.0
    # an exact tie at the top is margin 0 (whatever the third value)
    assert O.top2_margin([0.25, 7.0, 7.0, 6.0]) == 0.0
    # a duplicated runner-up does not count twice: [5, 4, 4] -> 1
    assert O.top2_margin([4.0, 5.0, 4.0]) == 1.0
    # brute force over random rows: max over i of (x_i - max_{j != i} x_j), clipped at 0
    rng = np.random.default_rng(3)
    for _ in range(50):
        x = rng.normal(size=9)
        i = int(np.argmax(x))
        exp = x[i] - max(x[j] for j in range(9) if j != i)
        assert abs(O.top2_margin(x) - exp) < 1e-15


# ------------------------------------------------------------------ GQA grouping
GQA = get_config("tiny").replace(name="gqa42", n_layers=1, d_model=16, n_heads=4, n_kv_heads=2, head_dim=4,
                                 d_ff=24, vocab=29, draft_len=2, prompt_len=4, gen_len=6)


def _gqa_weights(seed):
    w = {k: v.double().numpy() for k, v in make_weights(GQA, seed=seed).items()}
    w["layers.0.wo"] = np.eye(16)  # Hq * hd == d: the attention output passes through unchanged
    return O.Weights(GQA, w)


def test_gqa_single_token_reads_its_group_kv_head():
    """One token attends only itself, so query head h outputs exactly the value vector of its kv
    head. Grouping (base_forward): q head h reads kv head floor(h Hkv / Hq) -- q heads
    {0, 1} share kv head 0 and {2, 3} kv head 1 (contiguous groups). An interleaved grouping
    (h mod Hkv) would give q head 1 kv head 1 instead."""
    W = _gqa_weights(1)
    x = np.random.default_rng(4).normal(size=(1, 16))
    cache = O.KVCache(2, 2, 4)
    out = OM._attn(W, "layers.0.", x, np.array([0]), cache, 0)
    v = (x @ W["layers.0.wv"].T).reshape(2, 4)
    for h, g in enumerate((0, 0, 1, 1)):
        np.testing.assert_allclose(out[0, 4 * h:4 * h + 4], v[g], rtol=1e-13, atol=1e-15)
    assert not np.allclose(v[0], v[1])


def test_gqa_causal_block_brute_force():
    """Several tokens with RoPE and causal masking, against scalar loops written from the
    definitions (softmax(q k / sqrt(hd)) v per head, head h on kv head h // 2)."""
    W = _gqa_weights(2)
    rng = np.random.default_rng(5)
    T = 5
    x = rng.normal(size=(T, 16))
    pos = np.arange(T) + 3
    cache = O.KVCache(2, 2, 4)
    cache.K[0] = np.zeros((2, 3, 4))
    cache.V[0] = np.zeros((2, 3, 4))  # three earlier (zero) keys / values at positions 0..2
    out = OM._attn(W, "layers.0.", x, pos, cache, 0)
    q = O.rope((x @ W["layers.0.wq"].T).reshape(T, 4, 4), pos, GQA.rope_theta)
    k = O.rope((x @ W["layers.0.wk"].T).reshape(T, 2, 4), pos, GQA.rope_theta)
    v = (x @ W["layers.0.wv"].T).reshape(T, 2, 4)
    for h in range(4):
        g = h // 2
        keys = [np.zeros(4)] * 3 + [k[j, g] for j in range(T)]
        vals = [np.zeros(4)] * 3 + [v[j, g] for j in range(T)]
        for i in range(T):
            n_vis = 3 + i + 1  # keys at positions <= pos[i]
            s = [sum(q[i, h, c] * keys[j][c] for c in range(4)) / 2.0 for j in range(n_vis)]
            mx = max(s)
            e = [math.exp(t - mx) for t in s]
            z = sum(e)
            exp = [sum(e[j] * vals[j][c] for j in range(n_vis)) / z for c in range(4)]
            np.testing.assert_allclose(out[i, 4 * h:4 * h + 4], exp, rtol=1e-12, atol=1e-14)


# ------------------------------------------------------------------ reading C14
MICRO = get_config("tiny").replace(name="micro-c14", n_layers=2, d_model=12, n_heads=2, n_kv_heads=1,
                                   head_dim=4, d_ff=20, vocab=37, draft_len=3, prompt_len=5, gen_len=14)


@pytest.mark.parametrize("corrupt", [[1, 2, 3, 4], [4, 2, 1, 3], [3, 3, 4, 2]])
def test_next_draft_row_is_fresh_prefill_last_row(corrupt):
    """C14: the next draft reads I_D at the verify row m_b (the context layer ran over the step's
    k+1 verify rows in the GPU path; over the m+1 committed rows here). After a commit of m > 0
    tokens that row must equal the last row of a FRESH prefill (base forward + context layer)
    over the committed sequence prompt + emitted[:-1] -- whichever m the step accepted. Drafts are
    the true greedy continuation corrupted at a per-step slot, so the steps see m = 0 .. k."""
    W = O.Weights(MICRO, make_weights(MICRO, seed=3, norm_jitter=0.1))
    prompt = make_prompts(1, MICRO.prompt_len, MICRO.vocab, seed=4)[0].tolist()
    k = MICRO.draft_len
    ar = O.decode_greedy(W, prompt, MICRO.gen_len + 2 * (k + 1))

    def draft_fn(step, n, out):
        g = len(out)  # the next draft continues after the bonus token out[-1]
        d = list(ar[g:g + k])
        j = corrupt[step % len(corrupt)]
        if j <= k:
            d[j - 1] = (d[j - 1] + 1) % MICRO.vocab
        return d

    toks, steps = O.sd_decode(W, prompt, MICRO.gen_len, draft_fn=draft_fn, record=True)
    assert toks == ar[:MICRO.gen_len]
    ms = [s["m"] for s in steps]
    assert any(0 < m < k for m in ms) and k in ms  # ragged commits, including a full accept
    out = []
    for s in steps:
        out += s["greedy"][: s["m"] + 1]
        committed = prompt + ([ar[0]] + out)[:-1]
        assert len(committed) == s["n"] + s["m"] + 1
        cache = OM._new_cache(MICRO)
        g0, i_d_fresh, _ = O.prefill(W, committed, cache)
        np.testing.assert_allclose(s["i_d"], i_d_fresh, rtol=1e-10, atol=1e-12)
        assert g0 == ([ar[0]] + out)[-1]  # and its greedy token is the committed last token


# ------------------------------------------------------------------ NEXT-2 variants: "-Pos", BIDIR_PREFIX
VAR = get_config("tiny").replace(name="var", n_layers=2, d_model=16, n_heads=4, n_kv_heads=2, head_dim=4,
                                 d_ff=20, vocab=41, draft_len=3, prompt_len=6, gen_len=12)


def _w64(cfg, seed, **kw):
    return {k: v.double().numpy() for k, v in make_weights(cfg, seed=seed, norm_jitter=0.1, **kw).items()}


def test_no_pos_ffn_is_identity_stack_plus_bias():
    """"-Pos" (T4 P499; reading: W_P removed, D_j = RMS(I_D) + b_P[j]) equals Eq.9 with W_P replaced by k
    stacked identities -- and with b_P = 0 every slot is the same row, so the (permutation-equivariant)
    bidirectional block gives k identical draft-logit rows."""
    cfg = VAR.replace(no_pos_ffn=True)
    w = _w64(cfg, 5)
    i_d = np.random.default_rng(6).normal(size=cfg.d_model)
    D = O.positional_ffn(O.Weights(cfg, w), i_d)
    w_id = dict(w)
    w_id["sf.w_p"] = np.tile(np.eye(cfg.d_model), (cfg.draft_len, 1))
    np.testing.assert_allclose(D, O.positional_ffn(O.Weights(VAR, w_id), i_d), rtol=1e-13, atol=1e-15)
    w0 = dict(w)
    w0["sf.b_p"] = np.zeros_like(w["sf.b_p"])
    dl = O.draft_logits(O.Weights(cfg, w0), i_d)
    for j in range(1, cfg.draft_len):
        np.testing.assert_allclose(dl[j], dl[0], rtol=1e-12, atol=1e-13)
    assert not np.allclose(O.draft_logits(O.Weights(cfg, w), i_d)[1], O.draft_logits(O.Weights(cfg, w), i_d)[0])


def test_draft_prefix_attention_brute_force_and_zero_prefix_closed_form():
    """BIDIR_PREFIX (reading: the draft slots sit at positions n..n+k-1, rotated there, and
    every slot sees the context layer's n cached keys and all k slots): one head against scalar loops;
    with a zero prefix (K = V = 0) the output is the closed form sum_j e^s_j v_j / (n + sum_j e^s_j)."""
    cfg = VAR.replace(draft_prefix=True)
    W = O.Weights(cfg, _w64(cfg, 7))
    rng = np.random.default_rng(8)
    k, n, hd = cfg.draft_len, 5, cfg.head_dim
    x = rng.normal(size=(k, cfg.d_model))
    PK, PV = rng.normal(size=(2, n, hd)), rng.normal(size=(2, n, hd))  # [Hkv, n, hd] each
    out = OM._attn(W, "sf.blk_", x, None, None, None, ctx_prefix=(PK, PV, n)) @ np.linalg.pinv(W["sf.blk_wo"].T)
    q = O.rope((x @ W["sf.blk_wq"].T).reshape(k, 4, hd), n + np.arange(k), cfg.rope_theta)
    kk = O.rope((x @ W["sf.blk_wk"].T).reshape(k, 2, hd), n + np.arange(k), cfg.rope_theta)
    v = (x @ W["sf.blk_wv"].T).reshape(k, 2, hd)
    for h in range(4):
        g = h // 2
        keys = [PK[g, j] for j in range(n)] + [kk[j, g] for j in range(k)]
        vals = [PV[g, j] for j in range(n)] + [v[j, g] for j in range(k)]
        for i in range(k):
            sc = [sum(q[i, h, c] * kv[c] for c in range(hd)) / math.sqrt(hd) for kv in keys]
            mx = max(sc)
            e = [math.exp(t - mx) for t in sc]
            exp = [sum(e[j] * vals[j][c] for j in range(n + k)) / sum(e) for c in range(hd)]
            np.testing.assert_allclose(out[i, h * hd:(h + 1) * hd], exp, rtol=1e-9, atol=1e-11)
    Z = np.zeros((2, n, hd))
    out0 = OM._attn(W, "sf.blk_", x, None, None, None, ctx_prefix=(Z, Z, n)) @ np.linalg.pinv(W["sf.blk_wo"].T)
    for h in range(4):
        g = h // 2
        for i in range(k):
            sc = [float(q[i, h] @ kk[j, g]) / math.sqrt(hd) for j in range(k)]
            num = sum(math.exp(s) * v[j, g] for j, s in enumerate(sc))
            np.testing.assert_allclose(out0[i, h * hd:(h + 1) * hd], num / (n + sum(math.exp(s) for s in sc)),
                                       rtol=1e-9, atol=1e-11)


@pytest.mark.parametrize("variant", [dict(no_pos_ffn=True), dict(draft_prefix=True),
                                     dict(no_pos_ffn=True, draft_prefix=True)], ids=["nopos", "prefix", "both"])
def test_variants_stay_lossless(variant):
    """The variants change the drafts only: SD output == AR output exactly (P25), and with the prefix
    variant the draft depends on the committed context (different drafts than the paper's block)."""
    cfg = VAR.replace(**variant)
    w = _w64(cfg, 9)
    prompt = make_prompts(1, cfg.prompt_len, cfg.vocab, seed=10)[0].tolist()
    W = O.Weights(cfg, w)
    toks, steps = O.sd_decode(W, prompt, cfg.gen_len, record=True)
    assert toks == O.decode_greedy(W, prompt, cfg.gen_len)
    base = O.sd_decode(O.Weights(VAR, w), prompt, cfg.gen_len, record=True)[1]
    assert not np.allclose(steps[0]["draft_logits"], base[0]["draft_logits"])
