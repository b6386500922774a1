mkdir -p gpurun_out/r02k
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02k/build.log 2>&1
for K in 4 6 8; do timeout 900 python bench.py --config 13b --draft-len $K --steps 32 --no-cpu-baseline > gpurun_out/r02k/bench_13b_k$K.json 2> gpurun_out/r02k/bench_13b_k$K.err; echo "13b k$K rc=$?"; done
timeout 600 python bench.py --config small --batch 8 --no-cpu-baseline > gpurun_out/r02k/bench_small.json 2> gpurun_out/r02k/bench_small.err; echo "small rc=$?"
