set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 120 python tools/bert_bench.py 20 flow 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_bert.py -x -q 2>&1 | tail -15
timeout 300 python tools/bert_bench.py 50 flow 2>&1 | tail -3
timeout 300 python tools/bert_bench.py 50 perop 2>&1 | tail -3
