mkdir -p gpurun_out/seg
for B in 1 16 64; do for S in 2048 512 256; do
  SF_ATTN_SEG=$S timeout 300 python bench.py --batch $B --steps 32 --windows 1 --sweep none --no-cpu-baseline --forced-steps 0 --e2e-steps 2 --profile-steps 2 > gpurun_out/seg/b${B}_s$S.json 2>/dev/null
  echo "B=$B seg=$S $(python tools/show_bench.py gpurun_out/seg/b${B}_s$S.json 2>&1 | head -3 | tr '\n' ' ')"
done; done
