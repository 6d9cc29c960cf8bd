# Full GPU check: -m gpu suite, smoke, K1 back-to-back timings (release build).
exec > gpurun_out/r2_full.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 2>&1 | tail -40
echo "pytest rc=$?"
timeout 300 python __graft_entry__.py 2>&1 | tail -2
timeout 300 python tools/k1_bench.py 200 0,3,7,12,15,18,21 2>&1 | tail -10
