exec > gpurun_out/bert_mp.log 2>&1
timeout 300 python -m pytest tests/test_gpu_bert.py -x -q -s 2>&1 | grep -E "worst|passed|failed|Error" | tail -3
timeout 120 python tools/bert_bench.py 50
timeout 120 python tools/bert_bench.py 50
GFX_TRACE_GEMM=1 timeout 120 python tools/bert_bench.py 1 2>&1 | grep -A10 "gemm trace" | grep -v "stages\|^ *[0-9]" | head -40
