exec > gpurun_out/bench_r1c.log 2>&1
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python __graft_entry__.py 2>&1 | tail -2
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c_err.log; tail -3 gpurun_out/bench_r1c_err.log
cat gpurun_out/bench_r1c.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r1c_ref.json 2>/dev/null; cat gpurun_out/bench_r1c_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
ls -la gpurun_out | tail -5
