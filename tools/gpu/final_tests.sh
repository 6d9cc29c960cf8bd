exec > gpurun_out/final_tests.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout 300 python __graft_entry__.py 2>&1 | tail -1
