export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests/test_gpu_bert.py -x -q -k "widths or c5_shape or epilogue" --durations=5 2>&1 | tail -12
timeout 300 python tools/bert_bench.py 30 perop
