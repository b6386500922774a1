"""Per-phase timeline of the layer-sequence kernel (SF_KTRACE=1; csrc/gemm_seq.cuh items):
epilogue phase start / dependency met / end per CTA and the producers' activation-ready times.
  CFG=7b B=1 python tools/seq_trace.py"""
import os, sys, ctypes as C
os.environ["SF_KTRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_20340_b200 import Engine, EngineConfig
from paper_2511_20340_b200 import _native as N
from paper_2511_20340_b200.timeline import REC, critical_path, name
from synth import get_config, make_prompts, make_weights

cfg = get_config(os.environ.get("CFG", "7b")); B = int(os.environ.get("B", "1"))
w = make_weights(cfg, seed=0, device="cuda")
eng = Engine(EngineConfig.from_model(cfg, max_batch=B, max_seq=cfg.prompt_len + 64 * (cfg.draft_len + 1),
                                     flags=N.SF_FLAG_CUDA_GRAPH), w)
del w
eng.prefill(make_prompts(B, cfg.prompt_len, cfg.vocab).cuda())
eng.decode_steps(4); eng.sync()
buf = np.zeros(1 << 21, dtype=REC)
lib = N.lib()
lib.sf_debug_ktrace(buf.ctypes.data_as(C.c_void_p), buf.size)
eng.decode_steps(1); eng.sync()
n = lib.sf_debug_ktrace(buf.ctypes.data_as(C.c_void_p), buf.size)
rec = buf[:n]
items = rec[(rec["kid"] >> 24) == 18]
rest = rec[(rec["kid"] >> 24) != 18]
seqs = rest[(rest["kid"] >> 24) == 19]
print(f"{cfg.name} B={B}: {len(seqs)} seq CTA records")
# take the 3rd seq launch (a middle layer)
order = np.argsort(seqs["t0"])
seqs = seqs[order]
starts = seqs["t0"]
# split launches by gaps
cut = [0] + [i for i in range(1, len(seqs)) if seqs["t0"][i] > seqs["t1"][:i].max()] + [len(seqs)]
L = [(cut[i], cut[i + 1]) for i in range(len(cut) - 1)]
print(f"  launches: {len(L)}")
a, b = L[min(3, len(L) - 1)]
s = seqs[a:b]
T0 = s["t0"].min(); TW = s["tw"].min(); T1 = s["t1"].max()
print(f"  launch 3: CTAs {b - a}, start->dep {(TW - T0) / 1e3:.2f} us, dep->end {(T1 - TW) / 1e3:.2f} us")
it = items[(items["t0"] >= T0) & (items["t1"] <= T1 + 1000)]
par = it["kid"] & 0xFFFFFF
for role, nm in ((0x80, "epilogue"), (0x40, "producer act-ready")):
    sel = (par >> 16) == role
    ph = (par[sel] >> 8) & 0xFF
    for p_ in sorted(set(ph.tolist())):
        m = ph == p_
        x = it[sel][m]
        if nm == "epilogue":
            print(f"  phase {p_} {nm}: start med {np.median(x['t0'] - TW) / 1e3:7.2f} dep-met med {np.median(x['tw'] - TW) / 1e3:7.2f} "
                  f"max {np.max(x['tw'] - TW) / 1e3:7.2f} end med {np.median(x['t1'] - TW) / 1e3:7.2f} max {np.max(x['t1'] - TW) / 1e3:7.2f}")
        else:
            print(f"  phase {p_} {nm}: min {np.min(x['t0'] - TW) / 1e3:7.2f} med {np.median(x['t0'] - TW) / 1e3:7.2f} max {np.max(x['t0'] - TW) / 1e3:7.2f}")
sel = (par >> 16) == 0x20
x = it[sel]
ph = (x["kid"] >> 8) & 0xFF
nu = x["kid"] & 0xFF
for p_ in sorted(set(ph.tolist())):
    m = ph == p_
    dt = (x["t1"][m] - x["t0"][m]) / 1e3
    rate = dt / np.maximum(1, nu[m])
    print(f"  phase {p_} MMA segments: n {m.sum()} first-full med {np.median(x['t0'][m] - TW) / 1e3:7.2f} last med "
          f"{np.median(x['t1'][m] - TW) / 1e3:7.2f} max {np.max(x['t1'][m] - TW) / 1e3:7.2f}; us/unit med {np.median(rate):.3f} "
          f"units med {np.median(nu[m]):.0f}")
sel = (par >> 16) == 0x10
x = it[sel]
ph = (x["kid"] >> 8) & 0xFF
kind = x["kid"] & 0x3
for p_ in sorted(set(ph.tolist())):
    for kd, nm in ((1, "head"), (2, "tail"), (3, "full"), (0, "mid")):
        m = (ph == p_) & (kind == kd)
        if not m.any(): continue
        print(f"  phase {p_} {nm:4s} seg epilogue: n {m.sum():3d} accf-wait med {np.median(x['tw'][m] - x['t0'][m]) / 1e3:6.2f} "
              f"work med {np.median(x['t1'][m] - x['tw'][m]) / 1e3:6.2f} max {np.max(x['t1'][m] - x['tw'][m]) / 1e3:6.2f} "
              f"accf-passed max {np.max(x['tw'][m] - TW) / 1e3:7.2f} done max {np.max(x['t1'][m] - TW) / 1e3:7.2f}")
cp = critical_path(rest)
print(f"  step span {cp['span_us']:.1f} us")
for k in sorted(cp['exposed'], key=lambda k: -cp['exposed'][k])[:8]:
    print(f"  {k:24s} {cp['count'][k]:5d} {cp['exposed'][k]:9.1f} us  {cp['dur'][k] / cp['count'][k]:7.2f} us/launch")
