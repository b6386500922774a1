"""Print the key numbers of bench.py JSON lines: python tools/show_bench.py file..."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(f).read().strip().splitlines() if l.startswith("{")][-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    r, s = d["roofline"], d["step_roofline"]
    cl = r.get("event_classes", r.get("classes", {}))
    kp = r.get("event_profiled_steps", r.get("profiled_steps", 1))
    print(f"{f}: B={d['config']['batch_per_gpu']} ms/step={d['ms_per_step']:.3f} tok/s={d['value']:.0f} "
          f"step_frac={s['frac']:.3f} dom={r['kernel']}:{r['bound']} {r['achieved']:.0f}{r['unit']} frac={r['frac']:.3f} "
          f"e2e={d['e2e']['value']:.0f} sm={d['clocks']['sm_mhz']}")
    print("    event classes ms/step: " + " ".join(f"{k}={v['ms_total']/kp:.3f}" for k, v in cl.items()))
    tl = r.get("timeline")
    if tl:
        print(f"    timeline: span {tl['span_ms_per_step']:.3f} ms/step (events {tl['events_ms_per_step']:.3f}), gaps "
              f"{tl['idle_gap_ms_per_step']:.3f}; " + " ".join(
                  f"{c}={v['exposed_ms_per_step']:.3f}/{v['launches_per_step']:.0f}" for c, v in tl["classes"].items()))
    fa = d.get("forced_acceptance")
    if fa:
        print(f"    forced: tok/s={fa['tokens_per_s']:.0f} a={fa['mean_accepted_length']:.3f} (target {fa['a_target']}) "
              f"ms/step={fa['ms_per_step']:.3f}")
