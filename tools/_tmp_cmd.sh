mkdir -p gpurun_out/r02z
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02z/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02z/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02z/pytest_gpu.log
bash tools/knob_sweep.sh r02z "1 16 64" SF_X=0
