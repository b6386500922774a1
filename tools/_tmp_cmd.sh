python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B=64 FULL=1 bash tools/profile_round.sh r01y
B=16 bash tools/profile_round.sh r01y
B=1 bash tools/profile_round.sh r01y
ls -la gpurun_out/r01y
