"""Summarise an ncu launch-list CSV (metrics gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) per kernel: time share, per-launch time and DRAM traffic. Writes a text
summary and (optionally) the per-launch DRAM traffic of the GEMM and attention kernels as JSON
(bench.py reports it as roofline.traffic)."""
import csv, collections, json, sys

def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, ui, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
        per[r[ii]][r[mi]] = v * scale
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "")
    return per, names

def main(path, steps, out_txt, out_json=None):
    per, names = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    lines = [f"source: {path}", f"kernel time per step (ncu, serialised): {tot/steps:.1f} us over "
             f"{sum(a[0] for a in agg.values())/steps:.0f} launches", "",
             f"{'us/step':>10} {'share':>6} {'launch/step':>11} {'us/launch':>10} {'DRAM MB/launch':>14} {'GB/s':>7}  kernel"]
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{t/steps:10.1f} {100*t/tot:5.1f}% {n/steps:11.0f} {t/n:10.2f} {b/n/1e6:14.2f} {b/t/1e3 if t else 0:7.0f}  {k}")
    open(out_txt, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if out_json:
        traffic, tot = {}, collections.defaultdict(lambda: [0, 0.0])
        for k, (n, t, b) in agg.items():
            cls = "gemm" if k.startswith(("gemm_sk_kernel", "gemm_seq_kernel")) else ("attention" if k.startswith("attn_fd_kernel") else None)
            if cls:
                tot[cls][0] += n
                tot[cls][1] += b
        for cls, (n, b) in tot.items():
            traffic[cls] = b / n  # DRAM bytes per launch, averaged over the class's launches
        json.dump({"traffic_bytes_per_launch": traffic, "source": path}, open(out_json, "w"), indent=1)

if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
