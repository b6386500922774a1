"""Per-CTA timeline of the last in-step (CUDA graph) GEMM launch of weight shape N=SF_GEMM_TRACE_N.
  SF_GEMM_TRACE=1 SF_GEMM_TRACE_N=22016 B=64 python tools/gemm_trace_step.py"""
import os, sys, ctypes as C
os.environ.setdefault("SF_GEMM_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_20340_b200 import Engine, EngineConfig
from paper_2511_20340_b200 import _native as N
from synth import get_config, make_prompts, make_weights
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

cfg = get_config(os.environ.get("CFG", "7b")); B = int(os.environ.get("B", "64"))
w = make_weights(cfg, seed=0, device="cuda")
eng = Engine(EngineConfig.from_model(cfg, max_batch=B, max_seq=cfg.prompt_len + 32 * (cfg.draft_len + 1),
                                     flags=N.SF_FLAG_CUDA_GRAPH), w)
del w
eng.prefill(make_prompts(B, cfg.prompt_len, cfg.vocab).cuda())
eng.decode_steps(4); eng.sync()
buf = np.zeros(2 * 160 * 128, dtype=np.uint64)
N.lib().sf_debug_gemm_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
eng.decode_steps(1); eng.sync()
N.lib().sf_debug_gemm_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
tr = buf.reshape(-1, 128).astype(np.int64); tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min(); R = np.where(tr > 0, (tr - t0) / 1e3, np.nan)
print(f"== in-step GEMM N={os.environ.get('SF_GEMM_TRACE_N')} B={B}: {len(tr)} CTAs, span {np.nanmax(R):.2f} us")
for k, c in {"start": 0, "setup": 1, "prod0": 2, "mma_full0": 3, "mma_last": 4, "epi_done": 5}.items():
    v = R[:, c]; print(f"  {k:10s} min {np.nanmin(v):7.2f} med {np.nanmedian(v):7.2f} max {np.nanmax(v):7.2f} us")
for sg in range(4):
    v = R[:, 8 + 4 * sg: 12 + 4 * sg]
    if np.all(np.isnan(v)): continue
    print(f"  seg{sg}: mma_start/issued/epi_ready/epi_done med " + " ".join(f"{np.nanmedian(v[:, j]):7.2f}" for j in range(4)) +
          "   max " + " ".join(f"{np.nanmax(v[:, j]):7.2f}" for j in range(4)))
u = R[:, 24:64]; d = np.diff(u, axis=1)
print("  per-unit full-barrier interval (us): med %.3f  p90 %.3f" % (np.nanmedian(d), np.nanpercentile(d, 90)))
print("  unit pass times CTA0:", " ".join(f"{x:.2f}" for x in u[0, :20]))
print("  producer issue CTA0: ", " ".join(f"{x:.2f}" for x in R[0, 64:84]))
print("  final phase (med): flags %.2f bulk %.2f chunks(tmem+add/stored): %s" % (np.nanmedian(R[:, 104]), np.nanmedian(R[:, 105]),
      " ".join(f"{np.nanmedian(R[:, c]):.2f}/{np.nanmedian(R[:, c + 1]):.2f}" for c in (106, 108, 110, 112))))
order = np.argsort(-np.nan_to_num(R[:, 4]))
print("  slowest CTAs (mma_last): cta: seg(mma_start, issued, epi_ready, epi_done)...")
for i in list(order[:6]) + list(order[len(order) // 2: len(order) // 2 + 2]):
    segs = []
    for sg in range(4):
        v = R[i, 8 + 4 * sg: 12 + 4 * sg]
        if not np.all(np.isnan(v)): segs.append("(" + ",".join(f"{x:.1f}" for x in v) + ")")
    print(f"    cta {i:3d} full0 {R[i,3]:.1f} mma_last {R[i,4]:.1f} epi_done {R[i,5]:.1f}: " + " ".join(segs))
print("  final phase per CTA (flags, bulk, chunk0 add/stored, chunk1 add/stored, ...), epi_done:")
for i in list(order[:6]) + list(order[len(order) // 2: len(order) // 2 + 2]):
    print(f"    cta {i:3d}: " + " ".join(f"{x:.2f}" for x in R[i, 104:114]) + f"  | {R[i, 5]:.2f}")
print("  chunk detail per CTA (c0=0: tmem, add, staged, stored | c0=96: tmem, add, staged, stored):")
for i in list(order[:6]) + list(order[len(order) // 2: len(order) // 2 + 2]):
    print(f"    cta {i:3d}: " + " ".join(f"{x:.2f}" for x in [R[i,114], R[i,106], R[i,116], R[i,107]]) + " | " +
          " ".join(f"{x:.2f}" for x in [R[i,118], R[i,108], R[i,120], R[i,109]]))
print("  small-T head epilogue per CTA (epi_ready(last seg), flags, tmem+fixup, stored, epi_done):")
for i in list(order[:6]) + list(order[len(order) // 2: len(order) // 2 + 2]):
    ns = [sg for sg in range(4) if not np.isnan(R[i, 10 + 4 * sg])]
    er = R[i, 10 + 4 * ns[-1]] if ns else np.nan
    print(f"    cta {i:3d}: " + " ".join(f"{x:.2f}" for x in [er, R[i,122], R[i,123], R[i,124], R[i, 11 + 4 * ns[-1]] if ns else np.nan]))
print("  setup detail (start, barriers init, tmem alloc, syncthreads, cluster sync = setup) med: " +
      " ".join(f"{np.nanmedian(R[:, c]):.2f}" for c in (0, 125, 126, 127, 1)))
late = np.argsort(-np.nan_to_num(R[:, 0]))[:4]
for i in late:
    print(f"    late cta {i:3d}: " + " ".join(f"{R[i, c]:.2f}" for c in (0, 125, 126, 127, 1, 2, 3)))
