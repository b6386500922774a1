mkdir -p gpurun_out/r03f
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r03f/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r03f/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r03f/pytest_gpu.log
bash tools/knob_sweep.sh r03f "1 16 64" SF_GEMM_TICKET=0 SF_GEMM_TICKET=1 SF_GEMM_TICKET=0 SF_GEMM_TICKET=1
