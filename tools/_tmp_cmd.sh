python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B=64 FULL=1 bash tools/profile_round.sh r02q
B=16 bash tools/profile_round.sh r02q
B=1 bash tools/profile_round.sh r02q
for B in 64 1; do CFG=7b B=$B STEPS=2 timeout 300 python tools/ktrace.py > gpurun_out/r02q/ktrace_7b_b$B.txt 2>&1; done
NO_NCU=1 bash tools/gpu_check.sh r02q_check
