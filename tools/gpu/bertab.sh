# BERT per-op A/B: parity tests + forward times.
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_bert.py -x -q 2>&1 | tail -3
for i in 1 2; do timeout 300 python tools/bert_bench.py 50 perop; done
