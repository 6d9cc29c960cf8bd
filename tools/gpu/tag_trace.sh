exec > gpurun_out/tag_trace.log 2>&1
GFX_TRACE_MLP=1 timeout 60 python tools/kernel_bench.py 21 1 2>&1 | tail -120
