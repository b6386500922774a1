python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for CAP in 64 512; do for B in 1 4; do echo "cap $CAP B $B"; SF_PF_CAP=$CAP B=$B timeout 300 python tools/prefill_prof.py 2>&1 | head -1; done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
