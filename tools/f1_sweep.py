"""NEXT-1: the paper's preliminary experiment (F1 `fig:tpt`, P43-48, P342-343) on one B200.

"We tested the GPU throughput achieved under different batch sizes and token counts": for each batch
B and tokens per sequence m, the verify forward -- base model over B x m rows, m = k + 1 (the last
accepted token + k drafts), LM head and argmax -- is timed inside the product's CUDA-graph decode
step: the kernel timeline (per-CTA %globaltimer probes, paper_2511_20340_b200/timeline.py) gives the
span from the verify-row builder's dependency release to the accept kernel's, per step. Throughput =
B m / span. Synthetic 7B-shaped weights (synth/), uniform-random prompts; no new kernels.

The analytics the paper attaches to it (Eq.1-3, P72-95): AI_m = 2 M / (bytes M) = 1 for bf16
weights; AI_c = peak FLOP/s / bandwidth; the redundancy rho = AI_c / AI_m; a draft budget k is
"free" while the verify block stays below rho tokens, k <= rho / bs (Eq.3). Measured here: rho_eff =
the tokens per forward at which the throughput reaches 90% of its largest measured value, and the
per-B free budget m_free(B) = the largest m whose verify time is within 10% of m = 1's, i.e. the
block size up to which the extra draft tokens are (nearly) free.

  CFG=7b python tools/f1_sweep.py [out.json]     (one GPU; ~5 min)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_20340_b200 import Engine, EngineConfig, timeline
from paper_2511_20340_b200 import _native as N
from synth import get_config, make_prompts, make_weights
from synth.weights import weight_shapes

KT_ROWS, KT_ACCEPT = 13, 10


def verify_spans(rec):
    """per step: verify-row builder release -> accept release (us)"""
    return timeline.spans_between(rec, KT_ROWS << 24, KT_ACCEPT)


def main(out_path=None):
    name = os.environ.get("CFG", "7b")
    base_cfg = get_config(name)
    Bs = [int(x) for x in os.environ.get("BS", "1,4,16,64").split(",")]
    Ms = [int(x) for x in os.environ.get("MS", "1,2,3,5,9,17").split(",")]
    max_rows = int(os.environ.get("MAX_ROWS", "1088"))
    steps = int(os.environ.get("STEPS", "6"))
    P = int(os.environ.get("PROMPT", "256"))
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    base_w = make_weights(base_cfg, seed=0, device="cuda")
    base_shapes = dict(weight_shapes(base_cfg))
    rows = []
    buf = np.zeros(1 << 21, dtype=timeline.REC)
    lib = N.lib()
    for m in Ms:
        k = m - 1
        cfg = base_cfg.replace(draft_len=k, prompt_len=P)
        # draft-head tensors whose shape depends on k are drawn for this k; the rest is shared
        diff = [n for n, s in weight_shapes(cfg) if base_shapes.get(n) != s]
        w = dict(base_w)
        w.update(make_weights(cfg, seed=0, device="cuda", names=set(diff)))
        for B in Bs:
            if B * m > max_rows:
                continue
            max_seq = (P + (steps + 8) * (k + 1) + 32 + 15) // 16 * 16
            eng = Engine(EngineConfig.from_model(cfg, max_batch=B, max_seq=max_seq, flags=N.SF_FLAG_CUDA_GRAPH), w)
            eng.prefill(make_prompts(B, P, cfg.vocab, seed=1).cuda())
            eng.decode_steps(3)
            eng.sync()
            lib.sf_debug_ktrace_enable(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
            eng.decode_steps(steps)
            e1.record(eng.stream)
            eng.sync()
            n = lib.sf_debug_ktrace(C.c_void_p(buf.ctypes.data), buf.size)
            lib.sf_debug_ktrace_enable(0)
            spans = verify_spans(buf[:n])
            t_us = float(np.median(spans)) if spans else float("nan")
            rows.append({"B": B, "m": m, "k": k, "tokens": B * m, "verify_us": t_us,
                         "tokens_per_s": B * m / (t_us / 1e6), "step_ms": e0.elapsed_time(e1) / steps,
                         "steps": len(spans)})
            print(f"B={B:4d} m={m:3d} tokens={B*m:5d} verify {t_us:9.1f} us  {B*m/(t_us/1e6):12.0f} tok/s", flush=True)
            eng.close()
            del eng
            torch.cuda.empty_cache()
    # analytics (Eq.1-3)
    ai_m = 2.0 / 2.0  # bf16 weights: 2 FLOPs per 2-byte parameter read (Eq.1)
    ai_c_nom = 2.25e15 / 7.7e12
    ai_c_meas = peaks["bf16_tflops_sustained"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    tps = [r["tokens_per_s"] for r in rows]
    best = max(tps)
    knee = min((r["tokens"] for r in rows if r["tokens_per_s"] >= 0.9 * best), default=None)
    per_b = {}
    for B in Bs:
        rb = sorted((r for r in rows if r["B"] == B), key=lambda r: r["m"])
        if not rb:
            continue
        t1 = rb[0]["verify_us"]
        free = [r["m"] for r in rb if r["verify_us"] <= 1.1 * t1]
        per_b[B] = {"m_free": max(free), "k_free": max(free) - 1,
                    "eq3_k_budget_rho_meas": ai_c_meas / ai_m / B, "eq3_k_budget_rho_250": 250.0 / B}
    out = {"config": name, "prompt_len": P, "steps_per_point": steps, "rows": rows,
           "analytics": {"AI_m": ai_m, "AI_c_nominal": ai_c_nom, "AI_c_measured": ai_c_meas,
                         "rho_nominal": ai_c_nom / ai_m, "rho_measured": ai_c_meas / ai_m,
                         "rho_eff_tokens_at_90pct_peak_throughput": knee, "peak_tokens_per_s": best,
                         "per_batch": per_b},
           "method": "verify span = build_verify_rows release -> accept release on the kernel timeline of "
                     "CUDA-graph decode steps (median over steps); m = k + 1 tokens per sequence; m_free = "
                     "largest m whose verify time is within 10% of m = 1"}
    print(json.dumps(out["analytics"], indent=1))
    if out_path:
        json.dump(out, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
