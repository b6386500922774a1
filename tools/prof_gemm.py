"""GEMM microbenchmark: 7B-shaped weight GEMMs through sf_test_gemm (the hot path's kernels)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_20340_b200.engine import run_gemm, pack_matrix

shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (22016, 4096), "down": (4096, 11008), "lm": (32000, 4096)}
Ts = [int(x) for x in os.environ.get("TS", "5,80,320").split(",")]
iters = int(os.environ.get("ITERS", "20"))
only = os.environ.get("ONLY")
res = {}
for name, (N, K) in shapes.items():
    if only and name not in only.split(","):
        continue
    W = pack_matrix((0.02 * torch.randn(N, K, device="cuda")).to(torch.bfloat16))
    for T in Ts:
        A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        for _ in range(3):
            run_gemm(A, W, w_tiled=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(iters):
            run_gemm(A, W, w_tiled=True)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        by = N * K * 2 + T * K * 2 + T * N * 4
        fl = 2 * T * N * K
        res[f"{name}_T{T}"] = dict(us=ms * 1e3, gbs=by / ms / 1e6, tflops=fl / ms / 1e9)
        print(f"{name:5s} T={T:4d} N={N:6d} K={K:6d}: {ms*1e3:8.1f} us  {by/ms/1e6:7.0f} GB/s  {fl/ms/1e9:7.1f} TFLOP/s", flush=True)
json.dump(res, open(os.environ.get("OUT", "/dev/null"), "w"), indent=1)
