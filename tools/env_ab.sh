#!/bin/bash
# A/B of one build under two environment settings, alternated ROUNDS times per batch.
#   gpurun -- 'ENV_A="SF_X=0" ENV_B="SF_X=1" bash tools/env_ab.sh "1 16 64" 2'
BATCHES=${1:-64}; ROUNDS=${2:-2}; OUT=gpurun_out/envab; mkdir -p $OUT
for B in $BATCHES; do
  for r in $(seq $ROUNDS); do
    for v in A B; do
      E=$ENV_A; [ $v = B ] && E=$ENV_B
      env $E timeout 300 python bench.py --batch $B --steps 32 --windows 1 --sweep none --no-cpu-baseline \
        --forced-steps 0 --e2e-steps 2 --profile-steps 2 > $OUT/b${B}_${v}_$r.json 2> $OUT/b${B}_${v}_$r.err
      echo "B=$B $v($E) r$r rc=$? $(python tools/show_bench.py $OUT/b${B}_${v}_$r.json 2>&1 | head -3 | tr '\n' ' ')"
    done
  done
done
