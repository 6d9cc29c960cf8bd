# C5 BERT: parity tests + wall time per forward (single-CTA and 2-SM GEMMs).
exec > gpurun_out/r2_bert.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_bert.py -m gpu -q -x 2>&1 | tail -15
timeout 300 python tools/bert_bench.py 50 0
timeout 300 python tools/bert_bench.py 50 1
