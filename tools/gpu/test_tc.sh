set -x
timeout 120 python tools/kernel_bench.py 21 100 2>&1 | tail -3
timeout 120 python tools/kernel_bench.py 0 100 2>&1 | tail -3
timeout 300 python __graft_entry__.py 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
