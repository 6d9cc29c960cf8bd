exec > gpurun_out/edge.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k edge 2>&1 | tail -15
