exec > gpurun_out/rand_shapes.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "random_shapes or edge" 2>&1 | tail -5
