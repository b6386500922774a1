mkdir -p gpurun_out/r02e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02e/build.log 2>&1
SF_GEMM_TRACE_N=12288 B=1 timeout 300 python tools/gemm_trace_step.py > gpurun_out/r02e/gtrace_b1_12288.txt 2>&1
SF_GEMM_TRACE_N=4096 B=1 timeout 300 python tools/gemm_trace_step.py > gpurun_out/r02e/gtrace_b1_4096.txt 2>&1
