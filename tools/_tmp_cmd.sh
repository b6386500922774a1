mkdir -p gpurun_out/r02p
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02p/build.log 2>&1
for B in 1 16 64; do timeout 600 python bench.py --batch $B --no-cpu-baseline --forced-steps 0 > gpurun_out/r02p/b$B.json 2> gpurun_out/r02p/b$B.err; echo "b$B rc=$?"; done
python tools/show_bench.py gpurun_out/r02p/*.json | grep -v "event\|timeline"
