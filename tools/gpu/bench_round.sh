# One GPU call: bench line, kernel micro-bench, ncu launch list of a short bench.
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_line.json 2> gpurun_out/bench_err.log; tail -5 gpurun_out/bench_err.log
cat gpurun_out/bench_line.json
python tools/kernel_bench.py 21 200 2>&1 | tail -1
python tools/kernel_bench.py 0 200 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_line.json 2>gpurun_out/bench_ref_err.log; cat gpurun_out/bench_ref_line.json; tail -3 gpurun_out/bench_ref_err.log
