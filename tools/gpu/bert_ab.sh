exec > gpurun_out/bert_ab.log 2>&1
timeout 600 python -m pytest tests/test_gpu_bert.py -x -q -s 2>&1 | grep -E "worst|passed|failed|Error" | tail -5
timeout 300 python tools/bert_bench.py 50
timeout 300 python tools/bert_bench.py 50
