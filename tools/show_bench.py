"""Print the key numbers of bench.py JSON lines: python tools/show_bench.py file..."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(f).read().strip().splitlines() if l.startswith("{")][-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    r, s = d["roofline"], d["step_roofline"]
    cl = r.get("classes", {})
    print(f"{f}: B={d['config']['batch_per_gpu']} ms/step={d['ms_per_step']:.3f} tok/s={d['value']:.0f} "
          f"step_frac={s['frac']:.3f} dom={r['kernel']}:{r['bound']} {r['achieved']:.0f}{r['unit']} frac={r['frac']:.3f} "
          f"e2e={d['e2e']['value']:.0f} sm={d['clocks']['sm_mhz']}")
    print("    classes ms/step: " + " ".join(f"{k}={v['ms_total']/r['profiled_steps']:.3f}" for k, v in cl.items()))
    fa = d.get("forced_acceptance")
    if fa:
        print(f"    forced: tok/s={fa['tokens_per_s']:.0f} a={fa['mean_accepted_length']:.3f} (target {fa['a_target']}) "
              f"ms/step={fa['ms_per_step']:.3f}")
