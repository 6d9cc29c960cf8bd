exec > gpurun_out/test_ipc.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ipc.py -x -q 2>&1 | tail -25
