exec > gpurun_out/k1_extra.log 2>&1
timeout 120 python __graft_entry__.py 2>&1 | tail -1
for m in 0 7 15 21; do GFX_MLP_REPEAT=200 timeout 60 python tools/kernel_bench.py $m 1 2>&1 | grep repeat | tail -1; done
for m in 0 7 15 21; do GFX_MLP_UNIFORM=1 GFX_MLP_REPEAT=200 timeout 60 python tools/kernel_bench.py $m 1 2>&1 | grep repeat | tail -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
