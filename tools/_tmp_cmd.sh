mkdir -p gpurun_out/r02o
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02o/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02o/pytest_gpu.log
bash tools/knob_sweep.sh r02o "1 4 16" SF_ATTN_PF=0 SF_ATTN_PF=1
CFG=7b B=1 STEPS=4 timeout 300 python tools/ktrace.py > gpurun_out/r02o/kt_b1.txt 2>&1
