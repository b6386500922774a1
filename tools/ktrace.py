"""Kernel timeline of CUDA-graph decode steps (SF_KTRACE=1): per-launch start / dependency-resolved
/ end stamps from every CTA, reconstructed into launches and attributed to the step's critical path.
  CFG=7b B=64 STEPS=2 python tools/ktrace.py"""
import os, sys, ctypes as C
os.environ["SF_KTRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_20340_b200 import Engine, EngineConfig
from paper_2511_20340_b200 import _native as N
from synth import get_config, make_prompts, make_weights

from paper_2511_20340_b200.timeline import REC, critical_path, name


def main():
    cfg = get_config(os.environ.get("CFG", "7b"))
    if os.environ.get("K"):
        cfg = cfg.replace(draft_len=int(os.environ["K"]))
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
    cp = critical_path(rest)
    span, gap, Ls = cp["span_us"], cp["gap_us"], cp["_launches"]
    exposed, dur, cnt = cp["exposed"], cp["dur"], cp["count"]
    t_first = cp["_t_first"]
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
