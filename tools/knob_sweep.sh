#!/bin/bash
# One gpurun call: bench.py at a few batches under env-knob settings (short runs).
#   gpurun -- 'bash tools/knob_sweep.sh TAG "B1 B2" "VAR=v1" "VAR=v2" ...'
TAG=$1; shift; BS=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
for KV in "$@"; do
  for B in $BS; do
    f=$OUT/b${B}_${KV//[=,]/_}_$RANDOM.json
    env $KV timeout 300 python bench.py --batch $B --steps 32 --warmup 4 --no-cpu-baseline --forced-steps 0 --e2e-steps 8 > $f 2> $f.err
    echo "$KV B=$B rc=$?"
  done
done
python tools/show_bench.py $OUT/*.json
