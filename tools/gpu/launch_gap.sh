exec > gpurun_out/launch_gap.log 2>&1
for m in 0; do for mode in 0 4 5; do GFX_MLP_REPEAT=200 GFX_MLP_REPEAT_MODE=$mode timeout 120 python tools/kernel_bench.py $m 1 2>&1 | grep repeat | tail -1; done; done
for m in 0; do for mode in 0 4 5; do GFX_MLP_NOCOOP=1 GFX_MLP_REPEAT=200 GFX_MLP_REPEAT_MODE=$mode timeout 120 python tools/kernel_bench.py $m 1 2>&1 | grep repeat | tail -1; done; done
