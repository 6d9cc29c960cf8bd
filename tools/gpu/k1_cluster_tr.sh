exec > gpurun_out/k1_cluster_tr.log 2>&1
GFX_MLP_CLUSTER=1 GFX_TRACE_MLP=1 timeout 60 python tools/kernel_bench.py 0 1 2>&1 | grep -A28 "\[trace\]" | head -30
GFX_TRACE_MLP=1 timeout 60 python tools/kernel_bench.py 0 1 2>&1 | grep -A28 "\[trace\]" | head -30
