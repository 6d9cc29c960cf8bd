exec > gpurun_out/c3.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_c3.py -x -q 2>&1 | tail -25
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/c3_bench.json 2> gpurun_out/c3_bench.err
tail -3 gpurun_out/c3_bench.err
