#!/bin/bash
# One gpurun call: plain bench (must exit 0), then the ncu launch list of the same bench command
# (timed window only: bench brackets it with cudaProfilerStart/Stop), then ncu --set full of the top
# kernels. Output under gpurun_out/$TAG; summaries are copied to profiles/ by tools/profile_summary.py.
TAG=${1:-prof}; B=${B:-64}
OUT=gpurun_out/$TAG; mkdir -p $OUT
CMD="python bench.py --batch $B --steps 2 --warmup 3 --no-cpu-baseline --forced-steps 0 --e2e-steps 2"
$CMD > $OUT/plain_b$B.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/launches_b$B.csv $CMD > $OUT/ncu_list_b$B.log 2>&1
echo "launch list rc=$?"
if [ -n "$FULL" ]; then
  $CMD > $OUT/plain2_b$B.log 2>&1 && \
  ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k "regex:gemm_sk_kernel|attn_fd_kernel|resid_norm|rope_append|rope_partial" -s ${SKIP:-12} -c ${COUNT:-6} \
      -o $OUT/full_b$B -f $CMD > $OUT/ncu_full_b$B.log 2>&1
  echo "full rc=$?"
fi
