exec > gpurun_out/r2_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_live.py tests/test_gpu_multidevice.py tests/test_gpu_parity.py -m gpu -q -x -rs 2>&1 | tail -8
