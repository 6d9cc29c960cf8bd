exec > gpurun_out/bert_pf.log 2>&1
timeout 300 python tools/bert_bench.py 50 2>&1 | tail -1
timeout 300 python tools/bert_bench.py 50 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_bert.py -x -q 2>&1 | tail -2
GFX_TRACE_GEMM=1 timeout 120 python tools/bert_bench.py 1 2>&1 | grep -A22 "K 768 N 3072" | head -24
