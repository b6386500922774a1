"""Copy one tools/profile_r02.sh run (gpurun_out/r02prof) into profiles/r02: launch lists (+ summaries),
kernel timelines, ncu --set full summaries, the default bench line, and the per-launch DRAM traffic table
bench.py reports as roofline.traffic. python tools/refresh_profiles.py"""
import contextlib, io, json, shutil, subprocess, sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import profile_summary as ps

src = "gpurun_out/r02prof"
out = {}
for B in (64, 16, 1):
    shutil.copy(f"{src}/launches_b{B}.csv", f"profiles/r02/launches_7b_b{B}.csv")
    with contextlib.redirect_stdout(io.StringIO()):
        ps.main(f"profiles/r02/launches_7b_b{B}.csv", 2, f"profiles/r02/launches_7b_b{B}.txt", f"/tmp/tr{B}.json")
    t = json.load(open(f"/tmp/tr{B}.json"))
    t["source"] = (f"profiles/r02/launches_7b_b{B}.csv (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                   f"dram__bytes_write.sum --clock-control none, timed window of bench.py --batch {B} --steps 2 "
                   "--windows 1, cold-cache serialised)")
    out[f"7b_b{B}"] = t
    shutil.copy(f"{src}/ktrace_b{B}.txt", f"profiles/r02/ktrace_7b_b{B}.txt")
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
for n in ("b64", "b1", "attn_b64"):
    r = subprocess.run(["python", "tools/ncu_full_summary.py", f"{src}/full_{n}.ncu-rep"], capture_output=True, text=True)
    open(f"profiles/r02/full_7b_{n}.txt".replace("full_7b_attn_b64", "full_7b_b64_attn"), "w").write(r.stdout)
shutil.copy(f"{src}/bench_default.json", "profiles/r02/bench/bench_7b_default.json")
d = json.loads(open(f"{src}/bench_default.json").read().strip().splitlines()[-1])
print("B64", round(d["value"]), round(d["ms_per_step"], 3), [round(x, 1) for x in d["windows"]["ms"]],
      round(d["verify_steps_per_s"], 1), "gemm frac", round(d["roofline"]["frac"], 3), round(d["roofline"]["achieved"]),
      "step frac", round(d["step_roofline"]["frac"], 3), d["clocks"], "e2e", round(d["e2e"]["value"]),
      "forced", round(d["forced_acceptance"]["tokens_per_s"]), "cpu", d["cpu_baseline"]["value"],
      "prefill", round(d["prefill"]["ms"], 1), round(d["prefill"]["frac_roofline"], 3))
for s in d["batch_sweep"]:
    print("B", s["batch_per_gpu"], round(s["ms_per_step"], 3), round(s["verify_steps_per_s"], 1), "e2e", round(s["e2e"]["value"]),
          "step", round(s["step_roofline"]["frac"], 3), "gemm", round(s["roofline"]["frac"], 3), s["clocks"]["sm_mhz"])
