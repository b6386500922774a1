#!/bin/bash
# Round-2 evidence (one gpurun call): for each batch, the plain bench command (must exit 0), then the ncu
# launch list of the same command's timed window (bench.py brackets it with cudaProfilerStart/Stop), the
# in-graph kernel timeline (tools/ktrace.py), then ncu --set full of the top kernels at B = 64 and B = 1.
OUT=gpurun_out/r02prof; mkdir -p $OUT
for B in 64 16 1; do
  CMD="python bench.py --batch $B --steps 2 --warmup 3 --windows 1 --sweep none --no-cpu-baseline --forced-steps 0 --e2e-steps 2 --timeline-steps 0 --profile-steps 1"
  $CMD > $OUT/plain_b$B.log 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file $OUT/launches_b$B.csv $CMD > $OUT/ncu_list_b$B.log 2>&1
  echo "B=$B launch list rc=$?"
  B=$B timeout 300 python tools/ktrace.py > $OUT/ktrace_b$B.txt 2>&1
done
CMD="python bench.py --batch 64 --steps 2 --warmup 3 --windows 1 --sweep none --no-cpu-baseline --forced-steps 0 --e2e-steps 2 --timeline-steps 0 --profile-steps 1"
ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:gemm_sk_kernel|attn_fd_kernel|resid_norm|rope_partial" -s 12 -c 6 -o $OUT/full_b64 -f $CMD > $OUT/ncu_full_b64.log 2>&1
echo "full b64 rc=$?"
ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:attn_fd_kernel" -s 2 -c 1 -o $OUT/full_attn_b64 -f $CMD > $OUT/ncu_full_attn_b64.log 2>&1
echo "full attn b64 rc=$?"
CMD1="python bench.py --batch 1 --steps 2 --warmup 3 --windows 1 --sweep none --no-cpu-baseline --forced-steps 0 --e2e-steps 2 --timeline-steps 0 --profile-steps 1"
ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:gemm_sk_kernel|attn_fd_kernel" -s 8 -c 5 -o $OUT/full_b1 -f $CMD1 > $OUT/ncu_full_b1.log 2>&1
echo "full b1 rc=$?"
