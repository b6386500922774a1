#!/bin/bash
# sweep GEMM tiling knobs (env overrides) -- two passes each to expose run-to-run variance
for mh in 1 2; do for st in 0 2 3 4 6; do
  echo "== MH=$mh STAGES=$st"; SF_GEMM_MH=$mh SF_GEMM_STAGES=$st ITERS=30 TS=${TS:-5,80,256,320} python tools/prof_gemm.py 2>&1 | grep -v "^$"
done; done
