"""GPU parity, round 2: ragged acceptance, the bench-size blocks, batch invariance at full width and
teacher-forced checks (reading C21 (ii) and (iv) of SURVEY 8c), all through the C ABI against the
fp64 oracle.

* Ragged acceptance (PAPER P22-23 "accordingly updates the contextual information", lossless rule
  P25): drafts are the GPU's own greedy continuation corrupted at a per-(step, sequence) slot, fed
  through verify_step(draft_in), so one batch holds m = 0, 0 < m < k and m = k. Every step is
  compared with oracle.replay: logits, the NEXT step's draft logits (the draft reads I_D at the
  verify row r_b = m and the context layer's positions after an (m+1)-token commit), accept
  lengths, emitted tokens, seq_len and last_token.
* The bench's verify block sizes at full width (T = 320 at 7B B = 64; T = 576 at 13B k = 8, two
  GEMM chunks) against the oracle; B = 64 vs B = 1 bit-exact at full width.
* Teacher-forced taps (C21 iv): the oracle's SpecFormer head fed the GPU's own hook taps, so the
  draft head is bounded on its own, at full depth; teacher-forced single layers (C21 ii).
"""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_helpers import make_engine, max_seq_for, oracle_replay, rel_l2, run_gpu, setup
from paper_2511_20340_b200 import Engine, EngineConfig
from paper_2511_20340_b200 import _native as N
from synth import get_config, make_prompts, make_weights

pytestmark = pytest.mark.gpu

TINY = get_config("tiny")
SMALL = get_config("small")
MID = SMALL.replace(name="mid", n_layers=2, d_model=512, n_heads=4, n_kv_heads=4, head_dim=128, d_ff=1408,
                    vocab=4096, batch=4, prompt_len=300, gen_len=24)
GQA = MID.replace(name="gqa", d_model=1024, n_heads=8, n_kv_heads=2, prompt_len=200, batch=3)
W7D2 = get_config("7b").replace(name="7b-d2", n_layers=2, batch=3, prompt_len=200, gen_len=10)


def corrupt_slots(n_steps, B, k, seed):
    """Per-(step, sequence) corruption slot in 1..k+1 (k+1 = no corruption): uniform, so every
    accept length 0..k occurs; slot j gives m = j - 1 when the continuation is the base's greedy."""
    g = np.random.default_rng(seed)
    return g.integers(1, k + 2, size=(n_steps, B)).astype(np.int32)


def forced_run(cfg, w, prompts, n_steps, slots, ar, eng=None, want_logits=True, flags=0):
    """Eager draft -> verify(draft_in) -> accept with drafts = AR continuation corrupted at slots[s, b].
    Records per step: last, draft (forced), draft_logits (of the REAL draft forward), greedy, logits,
    m, emitted, seq_len, last_token (after the commit)."""
    B, k, V = prompts.shape[0], cfg.draft_len, cfg.vocab
    if eng is None:
        eng = make_engine(cfg, w, B, n_steps * (k + 1) + 2, flags=flags)
    g0 = eng.prefill(prompts.cuda())
    eng.sync()
    out = [[int(t)] for t in g0.cpu()]
    last = g0.cpu().numpy().copy()
    steps = []
    for s in range(n_steps):
        rec = {"last": last.copy()}
        if want_logits:
            _, dl = eng.draft_step(want_logits=True)
            rec["draft_logits"] = dl.cpu().numpy()
        else:
            eng.draft_step()
        forced = np.zeros((B, k), np.int32)
        for b in range(B):
            gidx = len(out[b])  # the drafts continue after the bonus token out[b][-1]
            forced[b] = ar[b][gidx:gidx + k]
            j = int(slots[s, b])
            if j <= k:
                forced[b, j - 1] = (forced[b, j - 1] + 1) % V
        res = eng.verify_step(torch.from_numpy(forced).cuda(), want_logits=want_logits)
        g, lg = res if want_logits else (res, None)
        m, em, sl = eng.accept_commit()
        lt = eng.capture(4, (B,), torch.int32)
        eng.sync()
        rec.update(draft=forced, greedy=g.cpu().numpy(), m=m.cpu().numpy(), emitted=em.cpu().numpy(),
                   seq_len=sl.cpu().numpy(), last_token=lt.cpu().numpy())
        if lg is not None:
            rec["logits"] = lg.cpu().numpy()
        for b in range(B):
            out[b] += [int(t) for t in rec["emitted"][b] if t >= 0]
            last[b] = rec["greedy"][b, rec["m"][b]]
        steps.append(rec)
    return {"tokens": out, "steps": steps, "engine": eng}


def check_commit_integers(cfg, prompts, res):
    """Reading a8 / P23 / P25 as integer logic (bit-exact): m = oracle accept(draft, greedy);
    emitted = greedy[0..m] then -1; seq_len += m + 1; last_token = greedy[m]."""
    k, B = cfg.draft_len, prompts.shape[0]
    n = np.full(B, prompts.shape[1])
    ms = []
    for s in res["steps"]:
        for b in range(B):
            m, em = O.accept(s["draft"][b].tolist(), s["greedy"][b].tolist())
            assert s["m"][b] == m
            assert s["emitted"][b].tolist() == em + [-1] * (k - m)
            n[b] += m + 1
            assert s["seq_len"][b] == n[b]
            assert s["last_token"][b] == s["greedy"][b][m]
            ms.append(m)
    return ms


def check_against_oracle(cfg, w, prompts, res, seqs, fp32, rel_tol=1.5e-2, draft_tol=None):
    """Per step: logits and (next-step) draft logits vs oracle.replay along the GPU's trajectory."""
    draft_tol = rel_tol if draft_tol is None else draft_tol
    checked = 0
    for b in seqs:
        _, rep = oracle_replay(cfg, w, prompts[b].tolist(), res["steps"], b)
        for s, r in zip(res["steps"], rep):
            gl, ol = s["logits"][b].astype(np.float64), r["logits"]
            dl, odl = s["draft_logits"][b].astype(np.float64), r["draft_logits"]
            if fp32:
                assert np.all(np.abs(gl - ol) <= 1e-5 + 1e-5 * np.abs(ol)), np.abs(gl - ol).max()
                assert np.all(np.abs(dl - odl) <= 1e-5 + 1e-5 * np.abs(odl)), np.abs(dl - odl).max()
                assert list(s["greedy"][b]) == r["greedy"]
                checked += cfg.draft_len + 1
            else:
                assert rel_l2(gl, ol) <= rel_tol, rel_l2(gl, ol)
                assert rel_l2(dl, odl) <= draft_tol, rel_l2(dl, odl)
                for i in range(cfg.draft_len + 1):
                    if O.top2_margin(ol[i]) > 5e-2:
                        checked += 1
                        assert s["greedy"][b][i] == r["greedy"][i]
                for j in range(cfg.draft_len):
                    if O.top2_margin(odl[j]) > 5e-2:
                        assert O.argmax_lowest(dl[j]) == O.argmax_lowest(odl[j])
    return checked


RAGGED = [
    (TINY.replace(batch=3), True, (0, 1, 2), 9, {}),
    (MID, False, (0, 3), 8, {}),
    (GQA, False, (0, 2), 8, {}),
    (W7D2, False, (0,), 6, dict(rel_tol=2.2e-2, draft_tol=2.6e-2)),
]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("cfg,fp32,seqs,n_steps,tol", RAGGED, ids=["tiny_fp32", "mha128", "gqa4", "7b_width_depth2"])
def test_ragged_acceptance_matches_oracle(cfg, fp32, seqs, n_steps, tol):
    jitter = 0.0 if fp32 else 0.1
    w, prompts = setup(cfg, seed=21, jitter=jitter)
    k = cfg.draft_len
    n_ar = n_steps * (k + 1) + k + 2
    ar = run_gpu(cfg, w, prompts, n_ar, k=0)["tokens"]  # the GPU's own greedy continuation
    slots = corrupt_slots(n_steps, cfg.batch, k, seed=5)
    res = forced_run(cfg, w, prompts, n_steps, slots, ar)
    ms = check_commit_integers(cfg, prompts, res)
    assert 0 in ms and k in ms and any(0 < m < k for m in ms), ms
    # losslessness on the device: what was emitted is the AR continuation
    for b in range(cfg.batch):
        assert res["tokens"][b] == ar[b][:len(res["tokens"][b])]
    assert check_against_oracle(cfg, w, prompts, res, seqs, fp32, **tol) > 10


@pytest.mark.timeout(900)
@pytest.mark.parametrize("cfg", [MID, W7D2], ids=["mha128", "7b_width_depth2"])
def test_ragged_acceptance_graph_matches_eager(cfg):
    """decode_steps (one CUDA graph per step) with sf_set_forced_drafts -- the bench's forced-acceptance
    mode -- emits the eager path's tokens and accept lengths step by step under the same per-sequence
    corruption slots (ragged m), with and without stored logits."""
    w, prompts = setup(cfg, seed=22, jitter=0.1)
    k, B, n_steps = cfg.draft_len, cfg.batch, 6
    ar = run_gpu(cfg, w, prompts, n_steps * (k + 1) + k + 2, k=0)["tokens"]
    slots = corrupt_slots(n_steps, B, k, seed=6)
    eager = forced_run(cfg, w, prompts, n_steps, slots, ar, want_logits=False)
    ms = check_commit_integers(cfg, prompts, eager)
    assert 0 in ms and k in ms and any(0 < m < k for m in ms), ms
    width = max(len(a) for a in ar)
    cont = torch.tensor([a + [a[-1]] * (width - len(a)) for a in ar], dtype=torch.int32).cuda()
    for flags in (N.SF_FLAG_CUDA_GRAPH, N.SF_FLAG_CUDA_GRAPH | N.SF_FLAG_NO_LOGITS):
        eng = make_engine(cfg, w, B, n_steps * (k + 1) + 2, flags=flags)
        eng.prefill(prompts.cuda())
        eng.set_forced_drafts(cont, torch.from_numpy(slots).cuda())
        em_log = torch.zeros(n_steps, B, k + 1, dtype=torch.int32, device="cuda")
        acc_log = torch.zeros(n_steps, B, dtype=torch.int32, device="cuda")
        eng.decode_steps(n_steps, em_log, acc_log)
        eng.sync()
        assert np.array_equal(acc_log.cpu().numpy(), np.stack([s["m"] for s in eager["steps"]]))
        assert np.array_equal(em_log.cpu().numpy(), np.stack([s["emitted"] for s in eager["steps"]]))
        sl = eng.capture(3, (B,), torch.int32).cpu().numpy()
        lt = eng.capture(4, (B,), torch.int32).cpu().numpy()
        assert np.array_equal(sl, eager["steps"][-1]["seq_len"])
        assert np.array_equal(lt, eager["steps"][-1]["last_token"])
        eng.close()


def test_graph_cache_follows_batch_size():
    """A handle whose step graph was captured at one batch size, re-prefilled at another, replays a
    graph of the new size: lengths and last tokens equal a fresh handle's, both ways."""
    cfg = MID.replace(batch=8)
    w, prompts = setup(cfg, seed=23, jitter=0.1)
    k = cfg.draft_len
    eng = make_engine(cfg, w, 8, 64, flags=N.SF_FLAG_CUDA_GRAPH)

    def fresh(B):
        e = make_engine(cfg, w, 8, 64, flags=N.SF_FLAG_CUDA_GRAPH)
        e.prefill(prompts[:B].cuda())
        e.decode_steps(4)
        return e.capture(3, (B,), torch.int32).cpu(), e.capture(4, (B,), torch.int32).cpu()

    for B in (2, 8, 3):
        eng.prefill(prompts[:B].cuda())
        eng.decode_steps(4)
        sl, lt = eng.capture(3, (B,), torch.int32).cpu(), eng.capture(4, (B,), torch.int32).cpu()
        fsl, flt = fresh(B)
        assert torch.equal(sl, fsl) and torch.equal(lt, flt), B
        assert (sl >= cfg.prompt_len + 4).all()


# ------------------------------------------------------------------ bench-size blocks at full width
BIG = [
    (get_config("7b").replace(name="7b-d2-b64", n_layers=2, batch=64, prompt_len=40, gen_len=4), (0, 37, 63)),
    (get_config("13b").replace(name="13b-d2-k8", n_layers=2, batch=64, draft_len=8, prompt_len=40, gen_len=4),
     (0, 63)),
]


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("cfg,seqs", BIG, ids=["7b_width_T320", "13b_width_k8_T576"])
def test_full_width_depth2_bench_blocks(cfg, seqs):
    """Full width, depth 2, at the bench's block sizes: T = B(k+1) = 320 (7B, B = 64: the PARTIAL /
    SwiGLU / QKV-partial epilogues, rope_partial and resid_norm at T = 320) and T = 576 (13B, k = 8:
    two GEMM chunks of 288) against the oracle, with ragged forced acceptance; GPU SD == GPU AR."""
    w, prompts = setup(cfg, seed=24, jitter=0.1)
    k, n_steps = cfg.draft_len, 3
    ar = run_gpu(cfg, w, prompts, n_steps * (k + 1) + k + 2, k=0)["tokens"]
    slots = corrupt_slots(n_steps, cfg.batch, k, seed=7)
    res = forced_run(cfg, w, prompts, n_steps, slots, ar)
    ms = check_commit_integers(cfg, prompts, res)
    assert 0 in ms and k in ms, ms
    for b in range(cfg.batch):
        assert res["tokens"][b] == ar[b][:len(res["tokens"][b])]
    assert check_against_oracle(cfg, w, prompts, res, seqs, False, rel_tol=2.2e-2, draft_tol=2.6e-2) > 10


@pytest.mark.timeout(900)
def test_full_width_batch_invariance_b64_vs_b1():
    """Reading C23 at full width (d = 4096, depth 2): sequence 17 of a B = 64 batch (T = 320 verify
    rows: QKV partials + rope_partial, 2-accumulator-free GEMM tiling, multi-tile attention) and the
    same sequence alone (T = 5: fused RoPE epilogue, small-T fixups) give bit-identical logits, draft
    logits and tokens at every step."""
    cfg = get_config("7b").replace(name="7b-d2-inv", n_layers=2, batch=64, prompt_len=48, gen_len=10)
    w, prompts = setup(cfg, seed=25, jitter=0.1)
    big = run_gpu(cfg, w, prompts, 10, want_logits=True)
    solo = run_gpu(cfg.replace(batch=1), w, prompts[17:18], 10, want_logits=True)
    assert solo["tokens"][0] == big["tokens"][17]
    for s1, s2 in zip(big["steps"], solo["steps"]):
        assert np.array_equal(s1["logits"][17], s2["logits"][0])
        assert np.array_equal(s1["draft_logits"][17], s2["draft_logits"][0])


# ------------------------------------------------------------------ teacher-forced (C21 ii / iv)
def setup_cuda(cfg, seed, jitter):
    """Weights drawn on the GPU (full-depth shapes: fast); the oracle upcasts only what it reads."""
    return make_weights(cfg, seed=seed, norm_jitter=jitter, device="cuda"), make_prompts(1, cfg.prompt_len, cfg.vocab)


def _prefill_taps(cfg, w, prompt):
    """B = 1 prefill of one chunk (P <= 512): the GPU's hook taps of every prompt row, its I_D rows,
    and the first draft step's logits (which read I_D[P - 1])."""
    P = prompt.shape[1]
    assert P <= 512
    eng = make_engine(cfg, w, 1, 8)
    eng.prefill(prompt.cuda())
    taps = eng.capture(6, (4, P, cfg.d_model)).cpu().numpy().astype(np.float64)
    i_d = eng.capture(7, (P, cfg.d_model)).cpu().numpy().astype(np.float64)
    d, dl = eng.draft_step(want_logits=True)
    eng.sync()
    out = dict(taps=taps, i_d=i_d, draft=d[0].cpu().numpy(), draft_logits=dl[0].cpu().numpy().astype(np.float64))
    eng.close()
    return out


TF = [
    get_config("7b").replace(name="7b-full-tf", batch=1, prompt_len=64),
    get_config("13b").replace(name="13b-full-tf", batch=1, prompt_len=48),
    get_config("70b").replace(name="70b-shape-d4-tf", n_layers=4, batch=1, prompt_len=48),
]


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("cfg", TF, ids=["7b_full_depth", "13b_full_depth", "70b_gqa_width"])
def test_teacher_forced_draft_head(cfg):
    """C21 (iv): the oracle's SpecFormer head (grouped RMSNorm, W_D, context layer L+1 over all prompt
    rows, positional FFN, draft block, frozen final norm + LM head) fed the GPU's OWN taps of every
    prompt row: this bounds the draft head alone, independent of the base model's depth. Asserted at
    the depth-2 bound (rel-L2 <= 2.2e-2; the head has about as many rounded GEMMs as two base
    layers), draft tokens exact where the oracle's margin > 5e-2. A second check feeds the
    GPU's own I_D row to the oracle's positional FFN + block + head (Eq.9-10 alone)."""
    w, prompts = setup_cuda(cfg, seed=26, jitter=0.1)
    g = _prefill_taps(cfg, w, prompts[:1])
    W = O.Weights(cfg, w)
    cache = O.model._new_cache(cfg)
    P = prompts.shape[1]
    i_d = O.context_layer(W, g["taps"], 0, cache)
    assert rel_l2(g["i_d"], i_d) <= 2.2e-2, rel_l2(g["i_d"], i_d)
    odl = O.draft_logits(W, i_d[P - 1])
    r = rel_l2(g["draft_logits"], odl)
    assert r <= 2.2e-2, r
    strict = 0
    for j in range(cfg.draft_len):
        if O.top2_margin(odl[j]) > 5e-2:
            strict += 1
            assert int(g["draft"][j]) == O.argmax_lowest(odl[j])
    odl2 = O.draft_logits(W, g["i_d"][P - 1])
    r2 = rel_l2(g["draft_logits"], odl2)
    assert r2 <= 1.5e-2, r2
    print(f"{cfg.name}: teacher-forced I_D rel-L2 {rel_l2(g['i_d'], i_d):.2e}, draft logits {r:.2e} "
          f"(from the GPU's I_D: {r2:.2e}), {strict} strict-margin draft tokens")


LAYER_TF = [
    (get_config("7b").replace(name="7b-d4-tf", n_layers=4, batch=1, prompt_len=96), "d4"),
    (get_config("7b").replace(name="7b-full-tf", batch=1, prompt_len=64), "full"),
    (get_config("70b").replace(name="70b-d4-tf", n_layers=4, batch=1, prompt_len=48), "d4"),
]


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("cfg,kind", LAYER_TF, ids=["7b_width_depth4", "7b_full_depth", "70b_gqa_width_depth4"])
def test_teacher_forced_layers(cfg, kind):
    """C21 (ii): single base layers fed the GPU's own residual stream (rel-L2 <= 1e-2 in bf16; the
    ideal pipeline gives 6.5e-3). Taps are HS[0, L/2, L-1, L]: layer L runs on the GPU's HS[L-1]
    over every prompt row (fresh KV cache) and is compared with the GPU's HS[L]; at depth 4 also
    layers 1..2 from HS[0] (the embedding, exact) against HS[2]."""
    w, prompts = setup_cuda(cfg, seed=27, jitter=0.1)
    g = _prefill_taps(cfg, w, prompts[:1])
    W = O.Weights(cfg, w)
    L, P = cfg.n_layers, prompts.shape[1]
    pos = np.arange(P)
    cache = O.model._new_cache(cfg)
    h = O.decoder_layer(W, L - 1, g["taps"][2], pos, cache)  # HS[L-1] -> HS[L]
    r_last = rel_l2(g["taps"][3], h)
    assert r_last <= 1e-2, r_last
    emb = W["embed"][prompts[0].numpy()]
    assert np.array_equal(g["taps"][0], emb)  # HS[0] = embedding rows, exact
    msg = f"{cfg.name}: layer {L} teacher-forced rel-L2 {r_last:.2e}"
    if kind == "d4":
        cache = O.model._new_cache(cfg)
        h = O.decoder_layer(W, 0, emb, pos, cache)
        h = O.decoder_layer(W, 1, h, pos, cache)
        r12 = rel_l2(g["taps"][1], h)
        assert r12 <= 1e-2 * np.sqrt(2), r12
        msg += f", layers 1-2 from HS[0] {r12:.2e}"
    print(msg)


# ------------------------------------------------------------------ layer-sequence kernel (small T)
SEQ_CFGS = [MID, GQA, W7D2.replace(name="7b-d3-b16", n_layers=3, batch=16, prompt_len=64),
            W7D2.replace(name="7b-d3-b12", n_layers=3, batch=12, prompt_len=64)]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("cfg", SEQ_CFGS, ids=["mha128_T20", "gqa4_T15", "7b_width_T80", "7b_width_T60"])
def test_layer_seq_bit_exact(cfg, monkeypatch):
    """The persistent layer-sequence launch (T <= 80: O-proj -> residual/RMSNorm -> gate/up -> down ->
    residual/RMSNorm -> next QKV with RoPE / KV append in one kernel; csrc/gemm_seq.cuh) keeps the
    standalone launches' partition and arithmetic: logits, draft logits, tokens and accept lengths are
    bit-identical with it off (SF_SEQ_T=0), across the fused-RoPE (T < 64) and RoPE-consumer (T >= 64)
    forms of the QKV phase, with ragged forced acceptance."""
    w, prompts = setup(cfg, seed=28, jitter=0.1)
    k, n_steps = cfg.draft_len, 5
    ar = run_gpu(cfg, w, prompts, n_steps * (k + 1) + k + 2, k=0)["tokens"]
    slots = corrupt_slots(n_steps, cfg.batch, k, seed=8)
    monkeypatch.setenv("SF_SEQ_T", "0")
    off = forced_run(cfg, w, prompts, n_steps, slots, ar)
    monkeypatch.setenv("SF_SEQ_T", "80")
    on = forced_run(cfg, w, prompts, n_steps, slots, ar)
    for s1, s2 in zip(off["steps"], on["steps"]):
        for key in ("logits", "draft_logits", "greedy", "m", "emitted", "seq_len", "last_token"):
            assert np.array_equal(s1[key], s2[key]), key
    check_commit_integers(cfg, prompts, on)


# ------------------------------------------------------------------ NEXT-2 draft variants
VARIANTS = [dict(no_pos_ffn=True), dict(draft_prefix=True), dict(no_pos_ffn=True, draft_prefix=True)]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("base,fp32,seqs", [(TINY.replace(batch=2), True, (0, 1)), (MID, False, (0, 3)),
                                            (GQA, False, (0, 2))], ids=["tiny_fp32", "mha128", "gqa4"])
@pytest.mark.parametrize("variant", VARIANTS, ids=["nopos", "prefix", "both"])
def test_draft_variants_match_oracle(base, fp32, seqs, variant):
    """NEXT-2 "-Pos" (SF_FLAG_NO_POS_FFN) and BIDIR_PREFIX (SF_FLAG_DRAFT_PREFIX; the slots also attend the
    context layer's committed keys, at a different n every step under ragged forced acceptance) against
    the oracle's variant head (DESIGN.md §3 readings), step by step; the verify and accept are unchanged
    (tokens == the GPU's AR continuation)."""
    cfg = base.replace(**variant)
    w, prompts = setup(cfg, seed=29, jitter=0.0 if fp32 else 0.1)
    k, n_steps = cfg.draft_len, 6
    ar = run_gpu(cfg, w, prompts, n_steps * (k + 1) + k + 2, k=0)["tokens"]
    slots = corrupt_slots(n_steps, cfg.batch, k, seed=9)
    res = forced_run(cfg, w, prompts, n_steps, slots, ar)
    check_commit_integers(cfg, prompts, res)
    for b in range(cfg.batch):
        assert res["tokens"][b] == ar[b][:len(res["tokens"][b])]
    assert check_against_oracle(cfg, w, prompts, res, seqs, fp32) > 10
    # free-running SD with the variant's own drafts is still lossless on the device
    sd = run_gpu(cfg, w, prompts, 16)
    assert sd["tokens"] == [a[:16] for a in ar]


# ------------------------------------------------------------------ NEXT-4: device-side KV page pool
def _steps(eng, n, B):
    """n eager draft -> verify -> accept steps; per step (emitted [B, k+1], logits [B, k+1, V])."""
    out = []
    for _ in range(n):
        eng.draft_step()
        g, lg = eng.verify_step(want_logits=True)
        _, em, _ = eng.accept_commit()
        eng.sync()
        out.append((em.cpu().numpy(), lg.cpu().numpy()))
    return out


def test_page_pool_matches_static_pages_and_reports_exhaustion():
    """SF_FLAG_PAGE_POOL (NEXT-4): pages taken from the device-side pool as sequences grow (prefill, then
    fused into the accept kernel) give bit-identical logits / tokens to the static per-sequence ranges,
    with the pool sized to what the run needs (oversubscribed vs max_batch x max_seq); a pool too small
    for the run is a sticky SF_ERR_CAPACITY."""
    cfg = MID
    w, prompts = setup(cfg, seed=30, jitter=0.1)
    B, k, n = cfg.batch, cfg.draft_len, 6
    ms = max_seq_for(cfg, n * (k + 1), k)
    stat = Engine(EngineConfig.from_model(cfg, max_batch=B, max_seq=ms), w)
    stat.prefill(prompts.cuda())
    ref = _steps(stat, n, B)
    need = B * ((cfg.prompt_len + n + k + 1 + 15) // 16)  # a = 1 with random weights: one token per step
    assert need < B * (ms // 16)
    ec = EngineConfig.from_model(cfg, max_batch=B, max_seq=ms, flags=N.SF_FLAG_PAGE_POOL)
    ec.pool_pages = need
    pool = Engine(ec, w)
    pool.prefill(prompts.cuda())
    got = _steps(pool, n, B)
    for (e1, l1), (e2, l2) in zip(ref, got):
        assert np.array_equal(e1, e2) and np.array_equal(l1, l2)
    ec_small = EngineConfig.from_model(cfg, max_batch=B, max_seq=ms, flags=N.SF_FLAG_PAGE_POOL)
    ec_small.pool_pages = B * (cfg.prompt_len // 16)
    small = Engine(ec_small, w)
    small.prefill(prompts.cuda())
    with pytest.raises(N.SpecFormerError) as e:
        small.sync()
    assert e.value.status == N.SF_ERR_CAPACITY


def test_continuous_batching_prefill_slot():
    """Continuous batching (PAPER P18; NEXT-4): after 3 steps, slot 1's sequence is released and a new
    prompt is prefilled into it while slots 0 and 2 keep decoding. Slots 0 / 2 emit exactly the tokens
    of an uninterrupted run; the new sequence emits the tokens and logits of a fresh one-sequence run
    (bit-exact: batch-invariant kernels)."""
    cfg = MID.replace(batch=3)
    w, prompts = setup(cfg, seed=31, jitter=0.1)
    newp = make_prompts(1, cfg.prompt_len - 37, cfg.vocab, seed=77)
    B, k = 3, cfg.draft_len
    ms = max_seq_for(cfg, 12 * (k + 1), k)
    mk = lambda Bm: Engine(EngineConfig.from_model(cfg, max_batch=Bm, max_seq=ms, flags=N.SF_FLAG_PAGE_POOL), w)
    full = mk(B)
    full.prefill(prompts.cuda())
    ref = _steps(full, 7, B)
    eng = mk(B)
    eng.prefill(prompts.cuda())
    first = _steps(eng, 3, B)
    eng.release(1)
    with pytest.raises(N.SpecFormerError) as e:
        eng.draft_step()
    assert e.value.status == N.SF_ERR_STATE
    g0 = eng.prefill_slot(1, newp[0].cuda())
    after = _steps(eng, 4, B)
    for s, (em, lg) in enumerate(first + after):
        for b in (0, 2):
            assert np.array_equal(em[b], ref[s][0][b]) and np.array_equal(lg[b], ref[s][1][b]), (s, b)
    solo = mk(1)
    sg0 = solo.prefill(newp.cuda())
    sref = _steps(solo, 4, 1)
    assert int(g0.cpu()[0]) == int(sg0.cpu()[0])
    for (em, lg), (se, sl) in zip(after, sref):
        assert np.array_equal(em[1], se[0]) and np.array_equal(lg[1], sl[0])


# ------------------------------------------------------------------ tensor parallelism: all-reduce precision
GQA2K = get_config("70b").replace(name="70b-w2k", n_layers=2, d_model=2048, n_heads=16, n_kv_heads=4, d_ff=5632,
                                  batch=2, prompt_len=150, gen_len=8)


def _tp_run(cfg, w, prompts, tp, flags, fused=False):
    import threading

    from paper_2511_20340_b200.engine import LocalGroup
    group = LocalGroup(tp)
    engines, res, errs = [], [None] * tp, []
    for r in range(tp):
        ec = EngineConfig.from_model(cfg, max_batch=cfg.batch, max_seq=max_seq_for(cfg, cfg.gen_len, cfg.draft_len),
                                     tp_size=tp, tp_rank=r, flags=flags)
        eng = Engine(ec, w)
        eng.attach_local_group(group, r)
        engines.append(eng)

    def run(r):
        try:
            if fused:
                engines[r].attach_local_xch()  # (blocks until every rank's thread has attached)
            res[r] = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True, eng=engines[r])
        except Exception as ex:  # pragma: no cover - reported below
            errs.append(ex)

    th = [threading.Thread(target=run, args=(r,)) for r in range(tp)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for r in range(1, tp):
        assert res[r]["tokens"] == res[0]["tokens"]  # every rank emits the same tokens
    merged = {"tokens": res[0]["tokens"], "steps": []}
    for steps in zip(*[x["steps"] for x in res]):
        s = dict(steps[0])
        s["logits"] = np.concatenate([x["logits"] for x in steps], axis=-1)
        s["draft_logits"] = np.concatenate([x["draft_logits"] for x in steps], axis=-1)
        merged["steps"].append(s)
    for e in engines:
        e.close()
    group.close()
    return merged


@pytest.mark.timeout(900)
@pytest.mark.parametrize("tp", [2, 4])
def test_tp_bf16_reduce_parity(tp):
    """SURVEY 8e specifies the row-parallel all-reduce in bf16, the default (fp32 GEMM output rounded RNE,
    summed, widened back); SF_FLAG_TP_F32_REDUCE keeps fp32. Both stay within the bf16
    tolerance of the fp64 oracle (reading C21, depth 2: rel-L2 <= 2.2e-2, tokens exact where the oracle
    margin > 5e-2); the measured rel-L2 of each is printed for DESIGN.md §8 (the local group rounds the
    bf16 sum once; a ring all-reduce rounds at every hop)."""
    cfg = GQA2K
    w, prompts = setup(cfg, seed=32, jitter=0.1)
    errs = {}
    for name, flags in (("fp32", N.SF_FLAG_TP_F32_REDUCE), ("bf16", 0)):
        merged = _tp_run(cfg, w, prompts, tp, flags)
        _, rep = oracle_replay(cfg, w, prompts[0].tolist(), merged["steps"], 0)
        errs[name] = max(rel_l2(s["logits"][0].astype(np.float64), r["logits"]) for s, r in zip(merged["steps"], rep))
        assert errs[name] <= 2.2e-2, (name, errs[name])
        for s, r in zip(merged["steps"], rep):
            for i in range(cfg.draft_len + 1):
                if O.top2_margin(r["logits"][i]) > 5e-2:
                    assert s["greedy"][0][i] == r["greedy"][i]
    print(f"TP={tp}: logits rel-L2 vs oracle, fp32 all-reduce {errs['fp32']:.3e}, bf16 all-reduce {errs['bf16']:.3e}")


@pytest.mark.timeout(900)
@pytest.mark.parametrize("tp", [2, 4])
def test_tp_fused_allreduce_parity(tp):
    """NEXT-3: the row-parallel all-reduce fused into the residual + norm consumer over peer memory (each
    rank's GEMM stores bf16 into its exchange slot, an epoch flag is published, every consumer sums the
    ranks' slots in rank order). Ranks agree on every token; logits within the depth-2 bf16 tolerance of
    the fp64 oracle (reading C21: rel-L2 <= 2.2e-2, tokens exact where the oracle margin > 5e-2). On the
    local group the ranks meet at a host barrier after every epoch signal (no kernel waits on another
    rank's); the flags, slots, epoch parity and rank-order sum are the multi-GPU path's."""
    cfg = GQA2K
    w, prompts = setup(cfg, seed=32, jitter=0.1)
    merged = _tp_run(cfg, w, prompts, tp, 0, fused=True)
    _, rep = oracle_replay(cfg, w, prompts[0].tolist(), merged["steps"], 0)
    err = max(rel_l2(s["logits"][0].astype(np.float64), r["logits"]) for s, r in zip(merged["steps"], rep))
    assert err <= 2.2e-2, err
    for s, r in zip(merged["steps"], rep):
        for i in range(cfg.draft_len + 1):
            if O.top2_margin(r["logits"][i]) > 5e-2:
                assert s["greedy"][0][i] == r["greedy"][i]
    print(f"TP={tp}: fused peer-memory all-reduce, logits rel-L2 vs oracle {err:.3e}")


def test_tp_fused_attach_errors():
    """The exchange needs tp_size > 1 (SF_ERR_STATE) and, on a local group, the group attached first."""
    from paper_2511_20340_b200.engine import LocalGroup
    cfg = GQA2K
    w, _ = setup(cfg, seed=32, jitter=0.1)
    eng = Engine(EngineConfig.from_model(cfg, max_batch=1, max_seq=128), w)
    with pytest.raises(N.SpecFormerError):
        eng.xch_handle()
    eng.close()
    group = LocalGroup(2)
    eng = Engine(EngineConfig.from_model(cfg, max_batch=1, max_seq=128, tp_size=2, tp_rank=0), w)
    eng._group = group
    with pytest.raises(N.SpecFormerError):
        eng.attach_local_xch()  # (no sf_local_group_attach yet)
    assert len(eng.xch_handle()) == 64  # the region's IPC handle
    eng.close()
    group.close()


@pytest.mark.timeout(300)
def test_layer_seq_block_sizes_change_on_one_handle():
    """One handle (max_batch 64 -> 8-row prefill chunks) alternating layer-sequence launches of different
    block sizes -- prefill chunks of 8 rows, decode blocks of 5, the profiling step graph, a second
    prefill -- stays live (per-launch epoch stamps, no stale counters for rows a shorter block did not
    touch) and emits the same tokens as a fresh handle each time."""
    cfg = MID
    w, prompts = setup(cfg, seed=34, jitter=0.1)
    ms = max_seq_for(cfg, 40, cfg.draft_len)
    big = Engine(EngineConfig.from_model(cfg, max_batch=64, max_seq=ms, flags=N.SF_FLAG_CUDA_GRAPH), w)
    ref = run_gpu(cfg.replace(batch=1), w, prompts[:1], 12)["tokens"]
    for it in range(2):
        big.prefill(prompts[:1].cuda())
        em = torch.zeros(11, 1, cfg.draft_len + 1, dtype=torch.int32, device="cuda")
        if it == 1:
            big.profile(True)
        big.decode_steps(11, em, None)
        big.sync()
        big.profile(False)
        toks = [t for t in em.cpu().numpy().reshape(-1) if t >= 0]
        assert toks[:11] == ref[0][1:12], it


# ------------------------------------------------------------------ launch shapes that must not change bits
@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [W7D2.replace(name="7b-d2-b4", batch=4, prompt_len=200), GQA],
                         ids=["7b_width", "gqa4"])
def test_launch_shape_switches_bit_exact(cfg, monkeypatch):
    """Per-launch shape choices that keep every row's arithmetic: the residual + RMSNorm consumer with one
    or two virtual threads per real thread (SF_RN_FOLD 1 / 2: the canonical reduction tree either way) and
    the prefill in sequence groups or all sequences per pass (SF_PF_GROUP 1 / 0), and attention query tiles
    of 16 rows (two n-tiles, the default when a sequence's (query, head) rows exceed 8) or 8 (SF_ATTN_NQ=1).
    Logits, draft logits,
    tokens and accept lengths are bit-identical across the combinations, with ragged forced
    acceptance (prompt 200: prefill groups of 2 sequences)."""
    w, prompts = setup(cfg, seed=31, jitter=0.1)
    k, n_steps = cfg.draft_len, 4
    ar = run_gpu(cfg, w, prompts, n_steps * (k + 1) + k + 2, k=0)["tokens"]
    slots = corrupt_slots(n_steps, cfg.batch, k, seed=11)
    runs = []
    for fold, group, nq in (("1", "1", "0"), ("2", "1", "0"), ("1", "0", "0"), ("2", "0", "0"), ("1", "1", "1")):
        monkeypatch.setenv("SF_RN_FOLD", fold)
        monkeypatch.setenv("SF_PF_GROUP", group)
        monkeypatch.setenv("SF_ATTN_NQ", nq)  # 1: 8-row attention tiles only (GQA: 16-row tiles by default)
        runs.append(forced_run(cfg, w, prompts, n_steps, slots, ar))
    for other in runs[1:]:
        for s1, s2 in zip(runs[0]["steps"], other["steps"]):
            for key in ("logits", "draft_logits", "greedy", "m", "emitted", "seq_len", "last_token"):
                assert np.array_equal(s1[key], s2[key]), key
    check_commit_integers(cfg, prompts, runs[0])
