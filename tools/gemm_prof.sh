#!/bin/bash
# GEMM microbench + ncu --set full captures of single GEMM launches.
OUT=gpurun_out/${1:-gemm}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
ITERS=50 TS=${TS:-5,20,80,160,256,320} timeout 300 python tools/prof_gemm.py > $OUT/micro.txt 2>&1; cat $OUT/micro.txt
for spec in ${SPECS:-gu:320 down:320 gu:5}; do
  n=${spec%%:*}; t=${spec##*:}
  ONLY=$n TS=$t ITERS=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_sk --launch-skip 3 -c 1 \
     -o $OUT/${n}_T$t -f python tools/prof_gemm.py > $OUT/ncu_${n}_T$t.log 2>&1
  echo "ncu $spec rc=$?"
done
