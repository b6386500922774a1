#!/bin/bash
# A/B timing of two prebuilt libraries on one box (abl/libA.so vs abl/libB.so, built here), alternated
# ROUNDS times per batch: bench ms/step plus the timeline's per-class exposed ms.
#   gpurun -- 'bash tools/ab.sh [batches] [rounds]'
BATCHES=${1:-64}; ROUNDS=${2:-2}; OUT=gpurun_out/ab; mkdir -p $OUT
LIB=paper_2511_20340_b200/libspecformer.so
for B in $BATCHES; do
  for r in $(seq $ROUNDS); do
    for v in A B; do
      cp abl/lib$v.so $LIB
      timeout 300 python bench.py --batch $B --steps 32 --windows 1 --sweep none --no-cpu-baseline --forced-steps 0 \
        --e2e-steps 2 --profile-steps 2 $AB_ARGS > $OUT/b${B}_${v}_$r.json 2> $OUT/b${B}_${v}_$r.err
      echo "B=$B $v r$r rc=$? $(python tools/show_bench.py $OUT/b${B}_${v}_$r.json 2>&1 | head -3 | tr '\n' ' ')"
    done
  done
done
