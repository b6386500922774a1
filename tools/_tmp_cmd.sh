mkdir -p gpurun_out/r02i
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02i/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "rope" > gpurun_out/r02i/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02i/pytest_gpu.log
bash tools/knob_sweep.sh r02i "16 64" SF_X=0
CFG=7b B=64 STEPS=2 timeout 300 python tools/ktrace.py > gpurun_out/r02i/kt_b64.txt 2>&1
