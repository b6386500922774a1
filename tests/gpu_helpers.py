"""Shared GPU-test plumbing: run the CUDA path through the C ABI, replay in the oracle."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
from paper_2511_20340_b200 import Engine, EngineConfig
from synth import make_prompts, make_weights


def max_seq_for(cfg, n_tokens, k):
    # worst case: each step commits 1 token but needs k+1 slots
    n = cfg.prompt_len + n_tokens + 2 * (k + 1) + 16
    return (n + 15) // 16 * 16


def make_engine(cfg, weights, B, n_tokens, k=None, flags=0):
    k = cfg.draft_len if k is None else k
    ec = EngineConfig.from_model(cfg, max_batch=B, max_seq=max_seq_for(cfg, n_tokens, k), draft_len=k, flags=flags)
    return Engine(ec, weights)


def run_gpu(cfg, weights, prompts, n_tokens, k=None, flags=0, want_logits=False, block_table=None, eng=None):
    """Greedy SD (k > 0) or AR (k == 0) through draft/verify/accept. Returns dict with per-sequence
    token lists and per-step records (numpy)."""
    B = prompts.shape[0]
    k = cfg.draft_len if k is None else k
    if eng is None:
        eng = make_engine(cfg, weights, B, n_tokens, k, flags)
    if block_table is not None:
        eng.set_block_table(block_table)
    g0 = eng.prefill(prompts.cuda())
    eng.sync()
    out = [[int(t)] for t in g0.cpu()]
    last = g0.cpu().numpy().copy()
    steps = []
    while min(len(o) for o in out) < n_tokens:
        rec = {"last": last.copy()}
        if k > 0:
            if want_logits:
                d, dl = eng.draft_step(want_logits=True)
                rec["draft_logits"] = dl.cpu().numpy()
            else:
                d = eng.draft_step()
        res = eng.verify_step(want_logits=want_logits)
        g, lg = res if want_logits else (res, None)
        m, em, sl = eng.accept_commit()
        eng.sync()
        rec["draft"] = d.cpu().numpy() if k > 0 else np.zeros((B, 0), np.int32)
        rec["greedy"] = g.cpu().numpy()
        rec["m"] = m.cpu().numpy()
        rec["seq_len"] = sl.cpu().numpy()
        if lg is not None:
            rec["logits"] = lg.cpu().numpy()
        em = em.cpu().numpy()
        for b in range(B):
            out[b] += [int(t) for t in em[b] if t >= 0]
            last[b] = rec["greedy"][b, rec["m"][b]]
        steps.append(rec)
    return {"tokens": [o[:n_tokens] for o in out], "steps": steps, "engine": eng}


def oracle_replay(cfg, weights, prompt, steps, b, slot_causal=False):
    traj = [dict(draft=s["draft"][b].tolist(), m=int(s["m"][b]), last=int(s["last"][b])) for s in steps]
    W = O.Weights(cfg, weights)
    return O.replay(W, list(prompt), traj, slot_causal)


def setup(cfg, seed=0, jitter=0.0, B=None, n_layers=None):
    w = make_weights(cfg, seed=seed, norm_jitter=jitter, n_layers=n_layers)
    prompts = make_prompts(B or cfg.batch, cfg.prompt_len, cfg.vocab)
    return w, prompts


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
