mkdir -p gpurun_out/r03l
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r03l/build.log 2>&1
timeout 120 python -m pytest tests -m gpu -x -q -k "chained" > gpurun_out/r03l/pytest_chain.log 2>&1; echo "chain rc=$?"; tail -2 gpurun_out/r03l/pytest_chain.log
for B in 1 64; do SF_GEMM_CHAIN=1 timeout 150 python bench.py --batch $B --steps 32 --warmup 4 --no-cpu-baseline --forced-steps 0 --e2e-steps 8 > gpurun_out/r03l/b${B}_chain.json 2>/dev/null; echo "b$B rc=$?"; done
python tools/show_bench.py gpurun_out/r03l/*.json | grep -v event
