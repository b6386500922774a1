python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/r02r
CMD="python bench.py --batch 64 --steps 2 --warmup 3 --no-cpu-baseline --forced-steps 0 --e2e-steps 2"
$CMD > gpurun_out/r02r/plain.log 2>&1 && ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:attn_fd_kernel|resid_norm" -s 4 -c 3 -o gpurun_out/r02r/attn_b64 -f $CMD > gpurun_out/r02r/ncu.log 2>&1; echo rc=$?
