exec > gpurun_out/pipe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k pipelined 2>&1 | tail -5
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/pipe_bench.json 2> gpurun_out/pipe_bench.err
tail -3 gpurun_out/pipe_bench.err
