exec > gpurun_out/attn_tr.log 2>&1
GFX_TRACE_ATTN=1 timeout 120 python tools/bert_bench.py 1 2>&1 | grep "\[attn\]" | head -10
