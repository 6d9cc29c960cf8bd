set -x
timeout 120 python tools/kernel_bench.py 21 200 2>&1 | tail -1
timeout 120 python tools/kernel_bench.py 0 200 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bert.py -x -q 2>&1 | tail -4
GFX_TRACE_MLP=1 timeout 60 python tools/kernel_bench.py 21 1 2>&1 | grep -A6 "layer 1 K=3136 N=3136" | head -7
timeout 300 python tools/profile_catalog.py bert_c5 3 2>&1 | tail -2
