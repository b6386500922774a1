mkdir -p gpurun_out/r02n
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02n/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02n/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02n/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
bash tools/knob_sweep.sh r02n "1 64" SF_X=0
