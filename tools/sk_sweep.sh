for st in 0 4 6 8; do echo "== STAGES=$st"; SF_GEMM_STAGES=$st ITERS=30 TS=${TS:-5,80,256,320} python tools/prof_gemm.py 2>&1; done
