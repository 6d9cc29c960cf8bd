exec > gpurun_out/k1_steps.log 2>&1
GFX_TRACE_MLP=1 timeout 60 python tools/kernel_bench.py 21 1 2>&1 | grep -B2 -A80 "CTA 0 steps" | head -85
