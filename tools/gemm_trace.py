"""Per-CTA timeline of one tcgen05 GEMM launch (SF_GEMM_TRACE=1): where a launch's time goes.
  SF_GEMM_TRACE=1 SHAPE=gu T=320 python tools/gemm_trace.py"""
import os, sys, ctypes as C
os.environ.setdefault("SF_GEMM_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_20340_b200.engine import run_gemm, pack_matrix
from paper_2511_20340_b200 import _native as N

shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (22016, 4096), "down": (4096, 11008), "lm": (32000, 4096)}
for spec in os.environ.get("SPECS", "gu:320").split():
    name, T = spec.split(":"); T = int(T)
    Nn, K = shapes[name]
    W = pack_matrix((0.02 * torch.randn(Nn, K, device="cuda")).to(torch.bfloat16))
    A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
    buf = np.zeros(2 * 160 * 128, dtype=np.uint64)
    for it in range(4):
        run_gemm(A, W, w_tiled=True); torch.cuda.synchronize()
        n = N.lib().sf_debug_gemm_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
    tr = buf.reshape(-1, 128).astype(np.int64)
    tr = tr[tr[:, 0] > 0]
    t0 = tr[:, 0].min()
    rel = lambda v: np.where(v > 0, (v - t0) / 1e3, np.nan)
    R = rel(tr)
    print(f"== {name} T={T} N={Nn} K={K}: {len(tr)} CTAs, span {np.nanmax(R):.2f} us")
    cols = {"start": 0, "setup": 1, "prod0": 2, "mma_full0": 3, "mma_last": 4, "epi_done": 5}
    for k, c in cols.items():
        v = R[:, c]
        print(f"  {k:10s} min {np.nanmin(v):7.2f} med {np.nanmedian(v):7.2f} max {np.nanmax(v):7.2f} us")
    for sg in range(4):
        v = R[:, 8 + 4 * sg: 12 + 4 * sg]
        if np.all(np.isnan(v)): continue
        print(f"  seg{sg}: mma_start/issued/epi_ready/epi_done med " +
              " ".join(f"{np.nanmedian(v[:, j]):7.2f}" for j in range(4)) + "   max " +
              " ".join(f"{np.nanmax(v[:, j]):7.2f}" for j in range(4)))
    u = R[:, 24:64]
    d = np.diff(u, axis=1)
    print("  per-unit full-barrier interval (us): med %.3f  p90 %.3f" % (np.nanmedian(d), np.nanpercentile(d, 90)))
    print("  unit pass times CTA0:", " ".join(f"{x:.2f}" for x in u[0, :16]))
    pr = R[:, 64:104]
    print("  producer issue CTA0:  ", " ".join(f"{x:.2f}" for x in pr[0, :16]))
    if len(R) > 1:
        print("  producer issue CTA1:  ", " ".join(f"{x:.2f}" for x in pr[1, :16]))
        print("  unit pass times CTA1:", " ".join(f"{x:.2f}" for x in u[1, :16]))
