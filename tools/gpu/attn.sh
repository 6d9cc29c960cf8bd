exec > gpurun_out/attn.log 2>&1
timeout 120 python -m pytest tests/test_gpu_bert.py -x -q -s 2>&1 | grep -E "worst|passed|failed|Error|assert" | tail -5
timeout 120 python tools/bert_bench.py 50
GFX_ATTN_MMASYNC=1 timeout 120 python tools/bert_bench.py 50
