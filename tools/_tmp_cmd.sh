mkdir -p gpurun_out/r01x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r01x/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01x/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r01x/pytest_gpu.log
bash tools/knob_sweep.sh r01x "1 16 64" SF_QKV_PARTIAL=0 SF_QKV_PARTIAL=1
