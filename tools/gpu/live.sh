exec > gpurun_out/live.log 2>&1
timeout 900 python -m pytest tests/test_gpu_live.py -x -q 2>&1 | tail -25
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/live_bench.json 2> gpurun_out/live_bench.err
tail -3 gpurun_out/live_bench.err
