#!/bin/bash
# One gpurun call: build, GPU parity tests, smoke, 1-GPU bench at B = 64 / 16 / 1, ncu launch list.
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [tag]'
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_b64.json 2> $OUT/bench_b64.err; echo "bench b64 rc=$?"
timeout 300 python bench.py --batch 16 --no-cpu-baseline > $OUT/bench_b16.json 2> $OUT/bench_b16.err; echo "bench b16 rc=$?"
timeout 300 python bench.py --batch 1 --no-cpu-baseline > $OUT/bench_b1.json 2> $OUT/bench_b1.err; echo "bench b1 rc=$?"
if [ -z "$NO_NCU" ]; then
  for B in 64 1; do
    B=$B STEPS=2 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file $OUT/launches_b$B.csv python tools/launch_list.py > $OUT/ncu_b$B.log 2>&1
    echo "ncu b$B rc=$?"
    python tools/profile_summary.py $OUT/launches_b$B.csv 2 $OUT/launches_b$B.txt $OUT/traffic_b$B.json > /dev/null 2>&1
  done
fi
echo done
