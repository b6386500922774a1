"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, and GPU-side invariants.

Tolerances (reading C21 of SURVEY §8c):
  fp32 mode: logits |gpu - oracle| <= 1e-5 (abs) + 1e-5 rel; tokens, drafts, accept lengths bit-exact.
  bf16 mode (Small): per-step logits rel-L2 <= 1.5e-2 and >= 99% of elements within 2e-2 rel / 1e-2 abs;
    greedy and draft tokens bit-exact wherever the oracle's top-1/top-2 margin > 5e-2;
    accept lengths == oracle accept(gpu draft, gpu greedy) (integer logic, always exact).
  GPU SD == GPU AR (k = 0 loop) bit-exact (batch-invariant kernels, reading C23).
"""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_helpers import make_engine, max_seq_for, oracle_replay, rel_l2, run_gpu, setup
from paper_2511_20340_b200 import Engine, EngineConfig
from paper_2511_20340_b200 import _native as N
from paper_2511_20340_b200 import run_gemm
from synth import get_config, make_prompts

pytestmark = pytest.mark.gpu

TINY = get_config("tiny")
SMALL = get_config("small")


# ------------------------------------------------------------------ GEMM kernel parity
@pytest.mark.parametrize("T,Nn,K", [(1, 128, 64), (5, 256, 128), (16, 384, 4096), (40, 768, 768), (77, 2304, 768),
                                    (320, 4096, 4096), (600, 1024, 256), (8, 32000, 768), (257, 512, 11008),
                                    (384, 4096, 4096), (336, 2304, 768), (352, 512, 11008)])
def test_gemm_bf16_tcgen05(T, Nn, K):
    g = torch.Generator().manual_seed(T * 7 + Nn + K)
    A = torch.randn(T, K, generator=g).to(torch.bfloat16)
    W = (0.02 * torch.randn(Nn, K, generator=g)).to(torch.bfloat16)
    ref = (A.double() @ W.double().T)
    out = run_gemm(A.cuda(), W.cuda()).cpu().double()
    torch.cuda.synchronize()
    err = (out - ref).abs()
    tol = 2e-5 * (A.double().abs() @ W.double().abs().T) + 1e-6
    assert (err <= tol).all(), f"max err {err.max().item()} worst ratio {(err / tol).max().item()}"


@pytest.mark.parametrize("Nn,K", [(4096, 4096), (22016, 4096), (512, 11008)])
def test_gemm_rows_independent_of_block(Nn, K):
    """Batch invariance of the tcgen05 GEMM across every accumulator shape: the rows of a 384-row block
    (two 192-column sub-tiles, one accumulator), a 320-row block (two 160-column sub-tiles, rotating
    through three TMEM slots), a 256-row block (one sub-tile, double-buffered) and a 16-row block are
    bit-identical."""
    g = torch.Generator().manual_seed(Nn + K)
    A = torch.randn(384, K, generator=g).to(torch.bfloat16).cuda()
    W = (0.02 * torch.randn(Nn, K, generator=g)).to(torch.bfloat16).cuda()
    full = run_gemm(A, W)
    for T in (320, 256, 16):
        part = run_gemm(A[:T].contiguous(), W)
        torch.cuda.synchronize()
        assert torch.equal(part, full[:T]), T


@pytest.mark.parametrize("T,Nn,K", [(1, 64, 16), (5, 512, 64), (33, 100, 70)])
def test_gemm_fp32_simt(T, Nn, K):
    g = torch.Generator().manual_seed(1)
    A, W = torch.randn(T, K, generator=g), torch.randn(Nn, K, generator=g)
    out = run_gemm(A.cuda(), W.cuda()).cpu().double()
    ref = A.double() @ W.double().T
    assert torch.allclose(out, ref, rtol=1e-5, atol=1e-5)


# ------------------------------------------------------------------ Tiny fp32 end to end
def _check_fp32(cfg, w, prompts, res, atol=1e-5):
    for b in range(prompts.shape[0]):
        plog, rep = oracle_replay(cfg, w, prompts[b].tolist(), res["steps"], b)
        for s, r in zip(res["steps"], rep):
            gl = s["logits"][b]
            assert np.all(np.abs(gl - r["logits"]) <= atol + 1e-5 * np.abs(r["logits"])), \
                np.abs(gl - r["logits"]).max()
            dl = s["draft_logits"][b]
            assert np.all(np.abs(dl - r["draft_logits"]) <= atol + 1e-5 * np.abs(r["draft_logits"])), \
                np.abs(dl - r["draft_logits"]).max()
            assert list(s["greedy"][b]) == r["greedy"]
            assert list(s["draft"][b]) == [O.argmax_lowest(x) for x in r["draft_logits"]]
            m, _ = O.accept(s["draft"][b], s["greedy"][b])
            assert m == s["m"][b]


@pytest.mark.parametrize("seed,jitter", [(0, 0.0), (3, 0.1)])
def test_tiny_fp32_matches_oracle(seed, jitter):
    w, prompts = setup(TINY, seed=seed, jitter=jitter)
    res = run_gpu(TINY, w, prompts, TINY.gen_len, want_logits=True)
    _check_fp32(TINY, w, prompts, res)
    W = O.Weights(TINY, w)
    assert res["tokens"][0] == O.decode_greedy(W, prompts[0].tolist(), TINY.gen_len)


def test_tiny_fp32_batch_and_paged_permutation():
    cfg = TINY.replace(batch=3)
    w, prompts = setup(cfg, seed=5, B=3)
    res = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
    _check_fp32(cfg, w, prompts, res)
    eng = res["engine"]
    pps = eng.cfg.max_seq // 16
    perm = torch.randperm(3 * pps, generator=torch.Generator().manual_seed(9)).reshape(3, pps)
    res2 = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True, block_table=perm)
    assert res2["tokens"] == res["tokens"]
    for s1, s2 in zip(res["steps"], res2["steps"]):
        assert np.array_equal(s1["logits"], s2["logits"])


def test_tiny_gpu_sd_equals_gpu_ar():
    cfg = TINY.replace(batch=2)
    w, prompts = setup(cfg, seed=2, B=2)
    sd = run_gpu(cfg, w, prompts, cfg.gen_len)
    ar = run_gpu(cfg, w, prompts, cfg.gen_len, k=0)
    assert sd["tokens"] == ar["tokens"]
    assert all(len(s["m"]) == 2 for s in ar["steps"])


# ------------------------------------------------------------------ Small bf16
@pytest.fixture(scope="module")
def small_run():
    w, prompts = setup(SMALL, seed=0)
    res = run_gpu(SMALL, w, prompts, 48, want_logits=True)
    return w, prompts, res


def test_small_bf16_logits_and_tokens(small_run):
    w, prompts, res = small_run
    flips = checked = 0
    for b in (0, 5):
        _, rep = oracle_replay(SMALL, w, prompts[b].tolist(), res["steps"], b)
        for s, r in zip(res["steps"], rep):
            gl, ol = s["logits"][b].astype(np.float64), r["logits"]
            assert rel_l2(gl, ol) <= 1.5e-2
            ok = np.abs(gl - ol) <= 1e-2 + 2e-2 * np.abs(ol)
            assert ok.mean() >= 0.99
            for i in range(SMALL.draft_len + 1):
                if O.top2_margin(ol[i]) > 5e-2:
                    checked += 1
                    assert s["greedy"][b][i] == r["greedy"][i]
            dl, odl = s["draft_logits"][b].astype(np.float64), r["draft_logits"]
            for j in range(SMALL.draft_len):
                if O.top2_margin(odl[j]) > 5e-2:
                    assert s["draft"][b][j] == O.argmax_lowest(odl[j])
            m, _ = O.accept(s["draft"][b], s["greedy"][b])
            assert m == s["m"][b]
    assert checked > 50


def test_small_bf16_sd_equals_ar_and_batch_invariance(small_run):
    w, prompts, res = small_run
    ar = run_gpu(SMALL, w, prompts, 48, k=0)
    assert ar["tokens"] == res["tokens"]
    solo = run_gpu(SMALL.replace(batch=1), w, prompts[3:4], 48)
    assert solo["tokens"][0] == res["tokens"][3]


def test_forced_perfect_drafts_accept_all():
    """Drafts replaced by the GPU's own AR continuation => every step accepts k (C11 step count)."""
    cfg = TINY
    w, prompts = setup(cfg, seed=1)
    N_ = cfg.gen_len
    ar = run_gpu(cfg, w, prompts, N_ + 2 * cfg.draft_len + 2, k=0)
    cont = torch.tensor(ar["tokens"], dtype=torch.int32).cuda()
    eng = make_engine(cfg, w, 1, N_)
    eng.prefill(prompts.cuda())
    eng.set_forced_drafts(cont, None)
    n_steps = -(-(N_ - 1) // (cfg.draft_len + 1))
    acc = torch.zeros(n_steps, 1, dtype=torch.int32, device="cuda")
    eng.decode_steps(n_steps, None, acc)
    eng.sync()
    assert (acc == cfg.draft_len).all()


# ------------------------------------------------------------------ errors
def test_state_machine_and_nonfinite():
    cfg = TINY
    w, prompts = setup(cfg, seed=0)
    eng = make_engine(cfg, w, 1, 32)
    with pytest.raises(N.SpecFormerError) as e:
        eng.draft_step()
    assert e.value.status == N.SF_ERR_STATE
    eng.prefill(prompts.cuda())
    with pytest.raises(N.SpecFormerError) as e:
        eng.accept_commit()
    assert e.value.status == N.SF_ERR_STATE
    with pytest.raises(N.SpecFormerError) as e:
        eng.prefill(torch.zeros(2, 4, dtype=torch.int32).cuda())
    assert e.value.status == N.SF_ERR_SHAPE
    w2 = dict(w)
    w2["lm_head"] = w["lm_head"].clone()
    w2["lm_head"][7, 3] = float("nan")
    eng2 = make_engine(cfg, w2, 1, 32)
    eng2.prefill(prompts.cuda())
    with pytest.raises(N.SpecFormerError) as e:
        eng2.sync()
    assert e.value.status == N.SF_ERR_NONFINITE


def test_capacity_error():
    cfg = TINY
    w, prompts = setup(cfg, seed=0)
    eng = make_engine(cfg, w, 1, 4)
    eng.prefill(prompts.cuda())
    with pytest.raises(N.SpecFormerError) as e:
        eng.decode_steps(100)
    assert e.value.status == N.SF_ERR_CAPACITY


# ------------------------------------------------------------------ hd=128 bf16 (tensor-core attention path)
MID = SMALL.replace(name="mid", n_layers=2, d_model=512, n_heads=4, n_kv_heads=4, head_dim=128, d_ff=1408,
                    vocab=4096, batch=4, prompt_len=300, gen_len=24)
GQA = MID.replace(name="gqa", d_model=1024, n_heads=8, n_kv_heads=2, prompt_len=200, batch=3)


def _check_bf16(cfg, w, prompts, res, seqs, rel_tol=1.5e-2, slot_causal=False, draft_tol=None):
    draft_tol = rel_tol if draft_tol is None else draft_tol
    checked = 0
    for b in seqs:
        _, rep = oracle_replay(cfg, w, prompts[b].tolist(), res["steps"], b, slot_causal)
        for s, r in zip(res["steps"], rep):
            gl, ol = s["logits"][b].astype(np.float64), r["logits"]
            assert rel_l2(gl, ol) <= rel_tol, rel_l2(gl, ol)
            for i in range(cfg.draft_len + 1):
                if O.top2_margin(ol[i]) > 5e-2:
                    checked += 1
                    assert s["greedy"][b][i] == r["greedy"][i]
            odl = r["draft_logits"]
            assert rel_l2(s["draft_logits"][b].astype(np.float64), odl) <= draft_tol
            for j in range(cfg.draft_len):
                if O.top2_margin(odl[j]) > 5e-2:
                    assert s["draft"][b][j] == O.argmax_lowest(odl[j])
            assert O.accept(s["draft"][b], s["greedy"][b])[0] == s["m"][b]
    return checked


@pytest.mark.parametrize("cfg", [MID, GQA], ids=["mha128", "gqa4"])
def test_hd128_bf16_matches_oracle_and_sd_equals_ar(cfg):
    w, prompts = setup(cfg, seed=4, jitter=0.1)
    res = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
    assert _check_bf16(cfg, w, prompts, res, seqs=(0, cfg.batch - 1)) > 20
    ar = run_gpu(cfg, w, prompts, cfg.gen_len, k=0)
    assert ar["tokens"] == res["tokens"]
    eng = res["engine"]
    pps = eng.cfg.max_seq // 16
    perm = torch.randperm(cfg.batch * pps, generator=torch.Generator().manual_seed(3)).reshape(cfg.batch, pps)
    res2 = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True, block_table=perm)
    for s1, s2 in zip(res["steps"], res2["steps"]):
        assert np.array_equal(s1["logits"], s2["logits"])


# ------------------------------------------------------------------ 7B width, depth 2 (fused paths)
W7D2 = get_config("7b").replace(name="7b-d2", n_layers=2, batch=3, prompt_len=200, gen_len=10)
GQA2K = get_config("70b").replace(name="70b-w2k", n_layers=2, d_model=2048, n_heads=16, n_kv_heads=2,
                                  d_ff=5632, batch=2, prompt_len=150, gen_len=8)


W13D2 = get_config("13b").replace(name="13b-d2", n_layers=2, batch=2, prompt_len=160, gen_len=8)


@pytest.mark.parametrize("cfg", [W7D2, GQA2K, W13D2], ids=["7b_width_depth2", "gqa_d2048", "13b_width_depth2"])
def test_full_width_depth2_bf16(cfg):
    """Reading C21 (iii)/(iv): full-width bf16 at depth 2 -- logits rel-L2 <= 2.2e-2 (2x the ideal
    pipeline's 1.1e-2 at depth 2) and tokens exact where the oracle margin > 5e-2; GPU SD ==
    GPU AR bit-exact; exercises the fused partial-GEMM -> residual/RMSNorm consumer and the
    flash-decoding attention at d = 4096 / 5120 / GQA. The draft logits pass through one more
    transformer block (the draft block) and W_D on top of the L base layers, so their ideal error is the
    depth-3 one, interpolated between the ideal depth-2 (1.1e-2) and depth-4 (1.5e-2) rows: 1.3e-2;
    asserted at 2x that, 2.6e-2 (C21)."""
    w, prompts = setup(cfg, seed=7, jitter=0.1)
    res = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
    assert _check_bf16(cfg, w, prompts, res, seqs=(0,), rel_tol=2.2e-2, draft_tol=2.6e-2) > 10
    ar = run_gpu(cfg, w, prompts, cfg.gen_len, k=0)
    assert ar["tokens"] == res["tokens"]


# ------------------------------------------------------------------ multi-segment flash-decoding
@pytest.mark.parametrize("cfg", [MID, GQA], ids=["mha128", "gqa4"])
def test_attention_segments_fold(cfg, monkeypatch):
    """Attention keys split into fixed 128-key segments (SF_ATTN_SEG; the default segment exceeds every
    BASELINE context but the 70B one): segment states are published and folded in segment order by the
    CTA that completes a (sequence, head, tile) group's last segment. Oracle parity, GPU SD == GPU AR
    bit-exact, and paged == identity page tables bit-exact (the per-page TMA fallback) under it."""
    monkeypatch.setenv("SF_ATTN_SEG", "128")
    w, prompts = setup(cfg, seed=5, jitter=0.1)
    res = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
    assert _check_bf16(cfg, w, prompts, res, seqs=(0, cfg.batch - 1)) > 20
    ar = run_gpu(cfg, w, prompts, cfg.gen_len, k=0)
    assert ar["tokens"] == res["tokens"]
    eng = res["engine"]
    pps = eng.cfg.max_seq // 16
    perm = torch.randperm(cfg.batch * pps, generator=torch.Generator().manual_seed(4)).reshape(cfg.batch, pps)
    res2 = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True, block_table=perm)
    for s1, s2 in zip(res["steps"], res2["steps"]):
        assert np.array_equal(s1["logits"], s2["logits"])


def test_attention_many_segments_fold(monkeypatch):
    """A context of more than 8 key segments (SF_ATTN_SEG=128, 1200-key prompts: 10 segments): the split
    schedule is off (it holds <= 8), so the group's own CTA publishes every segment's warp states and folds
    them in segment order, 8 segments' loads per batch (two batches here). Oracle parity at the bf16
    tolerance and GPU SD == GPU AR."""
    monkeypatch.setenv("SF_ATTN_SEG", "128")
    cfg = MID.replace(name="mid-long", batch=2, prompt_len=1200, gen_len=10)
    w, prompts = setup(cfg, seed=9, jitter=0.1)
    res = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
    assert _check_bf16(cfg, w, prompts, res, seqs=(0,)) > 4
    ar = run_gpu(cfg, w, prompts, cfg.gen_len, k=0)
    assert ar["tokens"] == res["tokens"]


@pytest.mark.parametrize("cfg", [MID, GQA], ids=["mha128", "gqa4"])
def test_fused_rope_epilogue_bit_exact(cfg, monkeypatch):
    """The QKV GEMM's fused RoPE / paged-append epilogue (small blocks) and the separate RoPE kernel
    (large blocks) rotate the same bf16 projections with the same operations: forcing either path
    for every block gives bit-identical logits, drafts and tokens (so choosing it per T keeps SD ==
    AR and batch invariance).
    The unfused path comes in two forms -- the GEMM's own head-tile fixup + the RoPE kernel, and
    k-segment partials reduced by the RoPE kernel (launch_rope_partial) -- with the same additions
    in the same order: all three agree bit for bit."""
    w, prompts = setup(cfg, seed=6, jitter=0.1)
    monkeypatch.setenv("SF_ROPE_FUSE_T", "0")
    monkeypatch.setenv("SF_QKV_PARTIAL", "1")
    partial = run_gpu(cfg, w, prompts, 12, want_logits=True)
    monkeypatch.setenv("SF_QKV_PARTIAL", "0")
    unfused = run_gpu(cfg, w, prompts, 12, want_logits=True)
    monkeypatch.setenv("SF_ROPE_FUSE_T", "100000")
    fused = run_gpu(cfg, w, prompts, 12, want_logits=True)
    assert fused["tokens"] == unfused["tokens"] == partial["tokens"]
    for s1, s2, s3 in zip(unfused["steps"], fused["steps"], partial["steps"]):
        assert np.array_equal(s1["logits"], s2["logits"]) and np.array_equal(s1["logits"], s3["logits"])
        assert np.array_equal(s1["draft_logits"], s2["draft_logits"])
        assert np.array_equal(s1["draft_logits"], s3["draft_logits"])


@pytest.mark.parametrize("cfg", [MID, GQA], ids=["mha128", "gqa4"])
def test_attention_schedules_bit_exact(cfg, monkeypatch):
    """The two flash-decoding schedules -- a CTA per (group, segment) that publishes its warp states
    (small batches) and a CTA per group folding its segments in registers (large batches) -- compute
    the same per-segment / per-warp folds: bit-identical logits and tokens with both forced."""
    monkeypatch.setenv("SF_ATTN_SEG", "128")
    w, prompts = setup(cfg, seed=8, jitter=0.1)
    monkeypatch.setenv("SF_ATTN_SPLIT", "1")
    a = run_gpu(cfg, w, prompts, 12, want_logits=True)
    monkeypatch.setenv("SF_ATTN_SPLIT", "0")
    b = run_gpu(cfg, w, prompts, 12, want_logits=True)
    assert a["tokens"] == b["tokens"]
    for s1, s2 in zip(a["steps"], b["steps"]):
        assert np.array_equal(s1["logits"], s2["logits"])
        assert np.array_equal(s1["draft_logits"], s2["draft_logits"])


# ------------------------------------------------------------------ fused LM-head argmax (NEXT-4)
@pytest.mark.parametrize("cfg", [MID, GQA], ids=["mha128", "gqa4"])
def test_fused_argmax_ties_and_no_logits(cfg):
    """The bf16 LM head reduces packed (logit, id) keys in its epilogue (lane butterfly, warps and CTAs
    via atomicMax) instead of a separate argmax pass. Greedy rule (P25; reading: lowest id on ties):
    every greedy / draft token equals the lowest-id argmax of the GPU's own fp32 logits. Ties are
    forced with duplicated LM-head rows (+u at ids 130 and 200, -u at 131 and 255: one 128-row tile,
    different lanes and warps, so the two logits are bit-identical) of a norm that makes one pair the
    maximum at most positions: the lower id must win every time. SF_FLAG_NO_LOGITS (logits not
    stored) gives the same tokens, drafts and accept lengths, and refuses to return logits."""
    w, prompts = setup(cfg, seed=9, jitter=0.1)
    g = torch.Generator().manual_seed(11)
    u = (0.5 * torch.randn(cfg.d_model, generator=g)).to(w["lm_head"].dtype)
    lm = w["lm_head"].clone()
    lm[130], lm[200], lm[131], lm[255] = u, u, -u, -u
    w["lm_head"] = lm
    res = run_gpu(cfg, w, prompts, 16, want_logits=True)
    hot = 0
    for s in res["steps"]:
        for key_l, key_t in (("logits", "greedy"), ("draft_logits", "draft")):
            L, tok = s[key_l], s[key_t]
            assert np.array_equal(L[..., 130], L[..., 200]) and np.array_equal(L[..., 131], L[..., 255])
            for b in range(L.shape[0]):
                for i in range(L.shape[1]):
                    assert tok[b][i] == O.argmax_lowest(L[b, i])
                    assert tok[b][i] not in (200, 255)
                    hot += tok[b][i] in (130, 131)
    assert hot > 50
    nl = run_gpu(cfg, w, prompts, 16, flags=N.SF_FLAG_NO_LOGITS)
    assert nl["tokens"] == res["tokens"]
    for s1, s2 in zip(res["steps"], nl["steps"]):
        for key in ("draft", "greedy", "m"):
            assert np.array_equal(s1[key], s2[key])
    eng = nl["engine"]
    with pytest.raises(N.SpecFormerError):
        eng.draft_step(want_logits=True)


def test_fused_argmax_nonfinite_flag():
    """A NaN reaching the bf16 LM head's fused argmax raises the sticky SF_ERR_NONFINITE (SPEC S26),
    as the separate argmax pass does in fp32 mode (test_state_machine_and_nonfinite)."""
    w, prompts = setup(MID, seed=3)
    w["lm_head"] = w["lm_head"].clone()
    w["lm_head"][77, 5] = float("nan")
    eng = make_engine(MID, w, MID.batch, 8)
    eng.prefill(prompts.cuda())
    with pytest.raises(N.SpecFormerError) as e:
        eng.sync()
    assert e.value.status == N.SF_ERR_NONFINITE


@pytest.mark.timeout(900)
def test_bench_configuration_matches_eager_path():
    """bench.py's launch configuration -- 7B shape at full depth, B = 64, each decode step one CUDA
    graph replay (specformer_decode_steps), SF_FLAG_NO_LOGITS -- emits the same tokens and accept
    lengths, step by step, as the eager draft / verify / accept calls with the logits kept: the path
    the oracle tests check (at full depth: test_full_depth_7b_*; across batch sizes: batch invariance)."""
    from synth import make_weights
    cfg = get_config("7b").replace(prompt_len=128)
    B, n_steps, k = 64, 6, cfg.draft_len
    w = make_weights(cfg, seed=0, device="cuda")
    prompts = make_prompts(B, cfg.prompt_len, cfg.vocab, seed=2).cuda()
    ms = max_seq_for(cfg, n_steps * (k + 1), k)
    eager = Engine(EngineConfig.from_model(cfg, max_batch=B, max_seq=ms), w)
    eager.prefill(prompts)
    ems, accs = [], []
    for _ in range(n_steps):
        eager.draft_step(want_logits=True)
        eager.verify_step(want_logits=True)
        m, em, _ = eager.accept_commit()
        eager.sync()
        accs.append(m.cpu())
        ems.append(em.cpu())
    eager.close()
    del eager
    graph = Engine(EngineConfig.from_model(cfg, max_batch=B, max_seq=ms,
                                           flags=N.SF_FLAG_CUDA_GRAPH | N.SF_FLAG_NO_LOGITS), w)
    graph.prefill(prompts)
    em_log = torch.zeros(n_steps, B, k + 1, dtype=torch.int32, device="cuda")
    acc_log = torch.zeros(n_steps, B, dtype=torch.int32, device="cuda")
    graph.decode_steps(n_steps, em_log, acc_log)
    graph.sync()
    assert torch.equal(acc_log.cpu(), torch.stack(accs).to(torch.int32))
    assert torch.equal(em_log.cpu(), torch.stack(ems).to(torch.int32))
    graph.close()


# ------------------------------------------------------------------ tensor parallelism
@pytest.mark.timeout(600)
@pytest.mark.parametrize("tp", [2, 4])
def test_tensor_parallel_matches_oracle(tp):
    """70B-shaped GQA model split over tp ranks -- tp handles on this GPU, one host thread each,
    reducing through a local group (the NCCL path uses the same hooks): the ranks agree on every
    token, the concatenated vocabulary shards of their logits match the fp64 oracle within the
    bf16 tolerance (reading C21), and the tokens match the oracle wherever its top-2 margin > 5e-2."""
    import threading

    from paper_2511_20340_b200.engine import LocalGroup

    cfg = GQA2K.replace(n_kv_heads=4, batch=2, gen_len=8)
    w, prompts = setup(cfg, seed=7, jitter=0.1)
    group = LocalGroup(tp)
    engines, res, errs = [], [None] * tp, []
    for r in range(tp):
        ec = EngineConfig.from_model(cfg, max_batch=cfg.batch, max_seq=max_seq_for(cfg, cfg.gen_len, cfg.draft_len),
                                     tp_size=tp, tp_rank=r)
        eng = Engine(ec, w)
        eng.attach_local_group(group, r)
        engines.append(eng)

    def run(r):
        try:
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
        assert res[r]["tokens"] == res[0]["tokens"]
    merged = {"tokens": res[0]["tokens"], "steps": []}
    for steps in zip(*[x["steps"] for x in res]):
        s = dict(steps[0])
        s["logits"] = np.concatenate([x["logits"] for x in steps], axis=-1)
        s["draft_logits"] = np.concatenate([x["draft_logits"] for x in steps], axis=-1)
        merged["steps"].append(s)
    assert merged["steps"][0]["logits"].shape[-1] == cfg.vocab
    assert _check_bf16(cfg, w, prompts, merged, seqs=(0,), rel_tol=2.2e-2) > 10
    for e in engines:
        e.close()
    group.close()


def test_draft_slot_causal_ablation_matches_oracle():
    """NEXT-2 "+Att Mask" (T4, P497-514): SF_FLAG_DRAFT_CAUSAL masks the draft block's slot attention
    causally; drafts and their logits follow the oracle's slot-causal block (and differ from the
    bidirectional run), the verify stays exact, GPU SD == GPU AR."""
    cfg = MID
    w, prompts = setup(cfg, seed=5, jitter=0.1)
    res = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True, flags=N.SF_FLAG_DRAFT_CAUSAL)
    assert _check_bf16(cfg, w, prompts, res, seqs=(0, cfg.batch - 1), slot_causal=True) > 20
    bi = run_gpu(cfg, w, prompts, 4, want_logits=True)
    assert not np.allclose(bi["steps"][0]["draft_logits"], res["steps"][0]["draft_logits"])
    ar = run_gpu(cfg, w, prompts, cfg.gen_len, k=0)
    assert ar["tokens"] == res["tokens"]


def test_draft_blocks_larger_matches_oracle():
    """NEXT-2 "+Larger" (T4, P497-514) as two stacked draft blocks: drafts and their logits follow
    the oracle's two-block head, the verify stays exact, GPU SD == GPU AR."""
    cfg = MID.replace(draft_blocks=2)
    w, prompts = setup(cfg, seed=5, jitter=0.1)
    res = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
    assert _check_bf16(cfg, w, prompts, res, seqs=(0, cfg.batch - 1)) > 20
    ar = run_gpu(cfg, w, prompts, cfg.gen_len, k=0)
    assert ar["tokens"] == res["tokens"]


@pytest.mark.parametrize("cfg", [W7D2, GQA2K], ids=["7b_width_depth2", "gqa_d2048"])
def test_chained_ffn_bit_exact(cfg, monkeypatch):
    """The gate/up -> down chain (one launch: the down projection's weights stream while the gate/up
    tiles finish; its activation k-blocks load as they are published) keeps both GEMMs' k
    segmentation: bit-identical logits, drafts and tokens with the chain on and off."""
    w, prompts = setup(cfg, seed=9, jitter=0.1)
    monkeypatch.setenv("SF_GEMM_CHAIN", "1")
    on = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
    monkeypatch.setenv("SF_GEMM_CHAIN", "0")
    off = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
    assert on["tokens"] == off["tokens"]
    for s1, s2 in zip(on["steps"], off["steps"]):
        assert np.array_equal(s1["logits"], s2["logits"])
        assert np.array_equal(s1["draft_logits"], s2["draft_logits"])


# ------------------------------------------------------------------ 7B shape at full depth (bf16)
def test_full_depth_7b_bf16():
    """Reading C21 (iii)/(iv) at full depth (32 layers, d = 4096): logits and draft logits rel-L2 within
    2x the ideal bf16 pipeline's (<= 9e-2; an ideal pipeline already gives ~4e-2 and flips ~4% of the
    margin > 5e-2 positions), so tokens are checked as epsilon-argmax (the GPU's token is
    within 4 sigma_diff of the oracle's best logit) and the strict flip rate is reported; accept
    lengths exact; GPU SD == GPU AR bit-exact (the hard losslessness assertion at depth)."""
    cfg = get_config("7b").replace(batch=1, prompt_len=48, gen_len=8)
    w, prompts = setup(cfg, seed=11, jitter=0.1)
    res = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
    _, rep = oracle_replay(cfg, w, prompts[0].tolist(), res["steps"], 0)
    flips = checked = 0
    for s, r in zip(res["steps"], rep):
        gl, ol = s["logits"][0].astype(np.float64), r["logits"]
        assert rel_l2(gl, ol) <= 9e-2, rel_l2(gl, ol)
        dl, odl = s["draft_logits"][0].astype(np.float64), r["draft_logits"]
        assert rel_l2(dl, odl) <= 9e-2, rel_l2(dl, odl)
        sig = float(np.std(gl - ol))
        for i in range(cfg.draft_len + 1):
            assert ol[i][s["greedy"][0][i]] >= ol[i].max() - 4 * sig  # epsilon-argmax
            if O.top2_margin(ol[i]) > 5e-2:
                checked += 1
                flips += int(s["greedy"][0][i] != r["greedy"][i])
        assert O.accept(s["draft"][0], s["greedy"][0])[0] == s["m"][0]
    print(f"full-depth 7B bf16: {flips}/{checked} argmax flips where the oracle margin > 5e-2 (reported)")
    ar = run_gpu(cfg, w, prompts, cfg.gen_len, k=0)
    assert ar["tokens"] == res["tokens"]


def test_full_depth_7b_fp32():
    """Reading C21 (iii)/(iv), fp32 mode at full depth (7B shape, 32 layers; SIMT GEMMs with a fixed
    blocked k order, split-KV attention): logits and draft logits elementwise within 1e-4 abs + 1e-5 rel
    of the fp64 oracle (SURVEY 8c C21 iii: an ideal blocked fp32 pipeline gives 5.5e-5 max abs), greedy
    and draft tokens bit-exact wherever the oracle margin exceeds 1e-4 (fp32-noise ties below that are
    reported), accept lengths exact."""
    cfg = get_config("7b").replace(dtype="fp32", batch=1, prompt_len=32, gen_len=6)
    w, prompts = setup(cfg, seed=12)  # unit norm scales, as in the SURVEY 8c ideal-pipeline figure
    res = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
    _, rep = oracle_replay(cfg, w, prompts[0].tolist(), res["steps"], 0)
    ties = 0
    for s, r in zip(res["steps"], rep):
        for gl, ol in ((s["logits"][0], r["logits"]), (s["draft_logits"][0], r["draft_logits"])):
            err = np.abs(gl.astype(np.float64) - ol)
            assert np.all(err <= 1e-4 + 1e-5 * np.abs(ol)), f"{float(err.max()):.3e}"
        for i in range(cfg.draft_len + 1):
            if s["greedy"][0][i] != r["greedy"][i]:
                assert O.top2_margin(r["logits"][i]) < 1e-4
                ties += 1
        for j in range(cfg.draft_len):
            if s["draft"][0][j] != O.argmax_lowest(r["draft_logits"][j]):
                assert O.top2_margin(r["draft_logits"][j]) < 1e-4
                ties += 1
        assert O.accept(s["draft"][0], s["greedy"][0])[0] == s["m"][0]
    print(f"full-depth 7B fp32: {ties} fp32-noise ties (oracle margin < 1e-4)")
