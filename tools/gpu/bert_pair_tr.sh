exec > gpurun_out/bert_pair_tr.log 2>&1
GFX_GEMM_PAIR=1 timeout 300 python tools/bert_bench.py 20 2>&1 | tail -1
GFX_GEMM_PAIR=1 GFX_TRACE_GEMM=1 timeout 300 python tools/bert_bench.py 1 2>&1 | grep -A40 "K 768 N 3072" | head -42
