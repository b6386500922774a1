"""Kernel timeline of CUDA-graph decode steps (SF_KTRACE=1): per-launch start / dependency-resolved
/ end stamps from every CTA, reconstructed into launches and attributed to the step's critical path.
  CFG=7b B=64 STEPS=2 python tools/ktrace.py"""
import os, sys, collections, ctypes as C
os.environ["SF_KTRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_20340_b200 import Engine, EngineConfig
from paper_2511_20340_b200 import _native as N
from synth import get_config, make_prompts, make_weights

KIND = {1: "gemm", 2: "resid_norm", 3: "rope", 4: "attn", 5: "rmsnorm", 6: "group_rms", 7: "embed", 8: "argmax_p",
        9: "argmax_f", 10: "accept", 11: "bidir", 12: "gather", 13: "rows", 14: "gemm_simt", 15: "attn_part",
        16: "attn_comb", 17: "misc", 18: "item"}
REC = np.dtype([("kid", "<u4"), ("sm", "<u4"), ("t0", "<u8"), ("tw", "<u8"), ("t1", "<u8"), ("pad", "<u8")])


def launches(rec):
    rec = np.sort(rec, order="t0")
    open_, out = {}, []
    for r in rec:
        k = int(r["kid"])
        L = open_.get(k)
        if L is None or r["t0"] > L["t1"]:
            L = {"kid": k, "t0": int(r["t0"]), "tw": int(r["tw"]), "t1": int(r["t1"]), "n": 0}
            open_[k] = L
            out.append(L)
        L["tw"] = min(L["tw"], int(r["tw"]))
        L["t1"] = max(L["t1"], int(r["t1"]))
        L["n"] += 1
    return sorted(out, key=lambda L: L["tw"])


def name(kid):
    k, p = kid >> 24, kid & 0xFFFFFF
    n = KIND.get(k, str(k))
    return f"{n}[N={p}]" if n == "gemm" else n


def main():
    cfg = get_config(os.environ.get("CFG", "7b"))
    B = int(os.environ.get("B", "64")); steps = int(os.environ.get("STEPS", "2"))
    w = make_weights(cfg, seed=0, device="cuda")
    eng = Engine(EngineConfig.from_model(cfg, max_batch=B, max_seq=cfg.prompt_len + 32 * (cfg.draft_len + 1),
                                         flags=N.SF_FLAG_CUDA_GRAPH), w)
    del w
    eng.prefill(make_prompts(B, cfg.prompt_len, cfg.vocab).cuda())
    eng.decode_steps(4); eng.sync()
    buf = np.zeros(1 << 21, dtype=REC)
    lib = N.lib()
    lib.sf_debug_ktrace(buf.ctypes.data_as(C.c_void_p), buf.size)  # clear
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(eng.stream); eng.decode_steps(steps); e1.record(eng.stream); eng.sync()
    ms = e0.elapsed_time(e1)
    n = lib.sf_debug_ktrace(buf.ctypes.data_as(C.c_void_p), buf.size)
    items = buf[:n][(buf[:n]["kid"] >> 24) == 18]
    rest = buf[:n][(buf[:n]["kid"] >> 24) != 18]
    if len(items):
        par = items["kid"] & 0xFFFFFF
        seg, nseg, nch = par & 0xFF, (par >> 8) & 0xFF, par >> 16
        dt_c = (items["tw"] - items["t0"]) / 1e3; dt_m = (items["t1"] - items["tw"]) / 1e3
        for sg in sorted(set(seg.tolist())):
            msk = seg == sg
            print(f"  attention items seg {sg}: n={msk.sum()} chunks med {np.median(nch[msk]):.0f} "
                  f"chunk-loop med {np.median(dt_c[msk]):.2f} us (per chunk {np.median(dt_c[msk] / nch[msk]):.2f}) "
                  f"merge/publish med {np.median(dt_m[msk]):.2f} p90 {np.percentile(dt_m[msk], 90):.2f} us")
    Ls = launches(rest)
    t_first = Ls[0]["tw"]
    span = (max(L["t1"] for L in Ls) - t_first) / 1e3
    exposed = collections.defaultdict(float); dur = collections.defaultdict(float); cnt = collections.Counter()
    gap = 0.0; run_end = t_first
    for L in Ls:
        s = max(L["tw"], run_end)
        if L["tw"] > run_end: gap += (L["tw"] - run_end) / 1e3
        exposed[name(L["kid"])] += max(0, L["t1"] - s) / 1e3
        dur[name(L["kid"])] += (L["t1"] - L["tw"]) / 1e3
        cnt[name(L["kid"])] += 1
        run_end = max(run_end, L["t1"])
    print(f"{cfg.name} B={B}: {steps} graph steps, events {ms/steps*1e3:.1f} us/step, traced span "
          f"{span/steps:.1f} us/step, {len(Ls)/steps:.0f} launches/step, {n} CTA records")
    print(f"  idle gaps on the critical path: {gap/steps:.1f} us/step")
    print(f"  {'kernel':22s} {'launch/step':>11s} {'exposed us/step':>15s} {'share':>6s} {'us/launch(dep->end)':>20s}")
    for k in sorted(exposed, key=lambda k: -exposed[k]):
        print(f"  {k:22s} {cnt[k]/steps:11.1f} {exposed[k]/steps:15.1f} {100*exposed[k]/span:5.1f}% {dur[k]/cnt[k]:20.2f}")
    if os.environ.get("SEQ"):
        for L in Ls[: int(os.environ["SEQ"])]:
            print(f"    {name(L['kid']):20s} start {(L['t0']-t_first)/1e3:9.2f} dep {(L['tw']-t_first)/1e3:9.2f} "
                  f"end {(L['t1']-t_first)/1e3:9.2f} ctas {L['n']}")


if __name__ == "__main__":
    main()
