mkdir -p gpurun_out/r03h
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r03h/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r03h/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r03h/pytest_gpu.log
bash tools/knob_sweep.sh r03h "1 16 64" SF_GEMM_CHAIN=0 SF_GEMM_CHAIN=1 SF_GEMM_CHAIN=0 SF_GEMM_CHAIN=1
for B in 1 64; do CFG=7b B=$B STEPS=2 timeout 300 python tools/ktrace.py > gpurun_out/r03h/kt_b$B.txt 2>&1; done
