exec > gpurun_out/bench_r1b.log 2>&1
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python __graft_entry__.py 2>&1 | tail -2
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b_err.log; tail -3 gpurun_out/bench_r1b_err.log
cat gpurun_out/bench_r1b.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r1b_ref.json 2>/dev/null; cat gpurun_out/bench_r1b_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 430 -c 85 --csv --log-file gpurun_out/bert_launches.csv python tools/bert_bench.py 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 40 -c 4 -o gpurun_out/k2_full_r1b python tools/bert_bench.py 1 > /dev/null 2>&1
ls -la gpurun_out | tail -5
