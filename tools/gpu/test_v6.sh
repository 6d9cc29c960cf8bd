set -x
exec > gpurun_out/test_v6.log 2>&1
timeout 120 python __graft_entry__.py 2>&1 | tail -3
GFX_MLP_ABLATE=1 timeout 120 python __graft_entry__.py 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
for m in 0 15 21; do timeout 120 python tools/kernel_bench.py $m 200 2>&1 | tail -1; done
for m in 0 15 21; do GFX_MLP_LAYERWISE=1 timeout 120 python tools/kernel_bench.py $m 200 2>&1 | tail -1; done
