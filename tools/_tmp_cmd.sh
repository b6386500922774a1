python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
bash tools/knob_sweep.sh r03d "64" SF_GEMM_DSTG=0 SF_GEMM_DSTG=2 SF_GEMM_DSTG=4 SF_GEMM_DSTG=0 SF_GEMM_DSTG=2
