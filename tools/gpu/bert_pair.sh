exec > gpurun_out/bert_pair.log 2>&1
timeout 120 python -m pytest tests/test_gpu_bert.py -x -q -s 2>&1 | grep -E "worst|passed|failed|Error" | tail -3
GFX_GEMM_PAIR=1 timeout 120 python -m pytest tests/test_gpu_bert.py -x -q -s 2>&1 | grep -E "worst|passed|failed|Error" | tail -3
timeout 120 python tools/bert_bench.py 50
GFX_GEMM_PAIR=1 timeout 120 python tools/bert_bench.py 50
