exec > gpurun_out/tests_all.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python __graft_entry__.py 2>&1 | tail -2
for m in 0 15 21; do GFX_MLP_REPEAT=200 timeout 120 python tools/kernel_bench.py $m 1 2>&1 | grep repeat | tail -1; done
