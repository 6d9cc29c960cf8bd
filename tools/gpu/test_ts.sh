set -x
timeout 120 python tools/kernel_bench.py 21 200 2>&1 | tail -1
timeout 120 python tools/kernel_bench.py 0 200 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
bash tools/gpu/trace_mlp.sh 2>&1 | head -34
