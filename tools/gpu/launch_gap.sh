exec > gpurun_out/launch_gap.log 2>&1
for mode in 0 4 5 6; do GFX_MLP_REPEAT=200 GFX_MLP_REPEAT_MODE=$mode timeout 120 python tools/kernel_bench.py 0 1 2>&1 | grep repeat | tail -1; done
