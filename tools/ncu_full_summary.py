"""Key counters per captured launch of an `ncu --set full` report: python tools/ncu_full_summary.py rep.ncu-rep"""
import csv, io, subprocess, sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "sm__cycles_elapsed.avg.per_second"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
        vals = []
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                vals.append(f"{w}={r[i]} {units[i]}".strip())
        out.append(f"{d.get('ID', '?'):>4} {name}\n      " + "\n      ".join(vals))
    print(f"source: {path} (ncu --set full --clock-control none, one launch per row)\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
