"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[1:]:
    if r[hdr.index("Metric Name")] != "gpu__time_duration.sum": continue
    name = r[ki].split("(")[0].replace("void ", "")[:60]
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")]
    v = v / 1e3 if unit in ("nsecond", "ns") else v * (1e3 if unit in ("msecond", "ms") else 1)
    tot[name] += v; cnt[name] += 1
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
S = sum(tot.values())
print(f"total {S/steps:.1f} us/step over {sum(cnt.values())/steps:.0f} launches/step")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v/steps:10.1f} us/step {100*v/S:5.1f}%  {cnt[k]/steps:6.0f} launches  {v/cnt[k]:8.2f} us/launch  {k}")
