for occ in 1 2; do for ws in 0 1; do echo "== OCC=$occ WSPLIT=$ws"; SF_SK_OCC=$occ SF_SK_WSPLIT=$ws ITERS=30 TS=5,80,256 python tools/prof_gemm.py 2>&1; done; done
echo "== V1"; SF_GEMM_V1=1 ITERS=30 TS=5,80,256 python tools/prof_gemm.py 2>&1
