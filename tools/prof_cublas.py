"""cuBLAS reference timings (torch.matmul bf16) for the 7B GEMM shapes -- context for our kernel."""
import torch, os
shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (22016, 4096), "down": (4096, 11008), "lm": (32000, 4096)}
for name, (N, K) in shapes.items():
    W = (0.02 * torch.randn(N, K, device="cuda")).to(torch.bfloat16)
    for T in [int(x) for x in os.environ.get("TS", "5,80,256,320").split(",")]:
        A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        for _ in range(5): (A @ W.T)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(30): (A @ W.T)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 30
        by = N * K * 2 + T * K * 2 + T * N * 2
        print(f"cublas {name:5s} T={T:4d}: {ms*1e3:8.1f} us {by/ms/1e6:7.0f} GB/s {2*T*N*K/ms/1e9:7.1f} TFLOP/s", flush=True)
