exec > gpurun_out/wgate.log 2>&1
timeout 120 python __graft_entry__.py 2>&1 | tail -1
for g in 0 1 2 3 5 9; do
  for m in 0 21; do echo "gate $g model $m"; GFX_MLP_ABLATE=$((g<<8)) GFX_MLP_REPEAT=200 timeout 120 python tools/kernel_bench.py $m 1 2>&1 | grep repeat | tail -1; done
done
GFX_MLP_ABLATE=$((1<<8)) timeout 120 python __graft_entry__.py 2>&1 | tail -1
