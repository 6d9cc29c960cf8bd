exec > gpurun_out/k1_abl.log 2>&1
for ab in 0 2 4 6; do echo "ablate $ab"; for m in 0 21; do GFX_MLP_ABLATE=$ab GFX_MLP_REPEAT=200 timeout 60 python tools/kernel_bench.py $m 1 2>&1 | grep repeat | tail -1; done; done
