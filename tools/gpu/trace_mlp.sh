GFX_TRACE_MLP=1 timeout 120 python tools/kernel_bench.py 21 2 2>&1 | grep -A8 "\[trace\]" | tail -40
