# run prof_gemm against the instrumented library (SF_GEMM_PROFILE printf build)
cp paper_2511_20340_b200/libspecformer.so /tmp/lib_orig.so
cp tools/micro/libspecformer_prof.so paper_2511_20340_b200/libspecformer.so
ONLY=${ONLY:-lm} TS=${TS:-5,80,320} ITERS=1 python tools/prof_gemm.py 2>&1 | sort | uniq | head -30
cp /tmp/lib_orig.so paper_2511_20340_b200/libspecformer.so
