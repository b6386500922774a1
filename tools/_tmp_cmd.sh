mkdir -p gpurun_out/r02g
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02g/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "tensor_parallel" > gpurun_out/r02g/pytest_tp.log 2>&1; echo "tp rc=$?"; tail -30 gpurun_out/r02g/pytest_tp.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02g/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02g/pytest_gpu.log
