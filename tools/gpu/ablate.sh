for ab in 0 1 2 4 8 6 14; do
  echo "=== ablate $ab"
  GFX_MLP_ABLATE=$ab GFX_TRACE_MLP=1 timeout 60 python tools/kernel_bench.py 21 1 2>&1 | grep -A6 "layer 1 K=3136 N=3136" | head -7
done
