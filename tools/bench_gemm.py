"""GEMM main loop in isolation: standalone stream-K EPI_PARTIAL launch vs the same GEMM as a one-phase
layer-sequence launch (sf_bench_gemm). python tools/bench_gemm.py [T,N,K ...]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_20340_b200 import _native as N
torch.cuda.init()
lib = N.lib()
shapes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]] or \
    [(5, 12288, 4096), (5, 4096, 11008), (5, 4096, 4096), (5, 4096, 32768), (5, 4096, 1024), (80, 12288, 4096)]
reps = int(os.environ.get("REPS", "50"))
for (T, Nn, K) in shapes:
    row = []
    for impl in (0, 1):
        ms = C.c_float()
        st = lib.sf_bench_gemm(impl, T, Nn, K, reps, C.byref(ms))
        gbs = Nn * K * 2 / max(1e-9, ms.value / 1e3) / 1e9
        row.append(f"impl{impl} {ms.value * 1e3:7.2f} us {gbs:6.0f} GB/s (st {st})")
    print(f"T={T:3d} N={Nn:5d} K={K:5d}: " + " | ".join(row), flush=True)
