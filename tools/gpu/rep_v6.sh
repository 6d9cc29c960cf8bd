exec > gpurun_out/rep_v6.log 2>&1
for m in 0 7 15 21; do GFX_MLP_REPEAT=200 timeout 120 python tools/kernel_bench.py $m 1 2>&1 | grep repeat | tail -1; done
for m in 0 7 15 21; do GFX_MLP_ABLATE=64 GFX_MLP_REPEAT=200 timeout 120 python tools/kernel_bench.py $m 1 2>&1 | grep repeat | tail -1; done
