exec > gpurun_out/r2_cluster.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cluster.py -m gpu -q -x 2>&1 | tail -30
