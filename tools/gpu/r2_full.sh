# Full GPU check: -m gpu suite, smoke, K1 back-to-back timings, BERT forward.
exec > gpurun_out/r2_full.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -x --durations=8 2>&1 | tail -20
echo "pytest rc=$?"
timeout 300 python __graft_entry__.py 2>&1 | tail -2
timeout 300 python tools/k1_bench.py 200 0,7,15,21 2>&1 | tail -6
timeout 300 python tools/bert_bench.py 50 0 2>&1 | tail -1
