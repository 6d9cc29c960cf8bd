set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
for m in 0 15 21; do timeout 120 python tools/kernel_bench.py $m 200 2>&1 | tail -1; done
bash tools/gpu/trace_mlp.sh
