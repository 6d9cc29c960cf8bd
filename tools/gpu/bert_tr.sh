exec > gpurun_out/bert_tr.log 2>&1
GFX_TRACE_GEMM=1 timeout 300 python tools/bert_bench.py 1 2>&1 | grep -A40 "K 3072" | head -45
