# One GPU call: parity suite, smoke, kernel micro-benches, bench line (both arms),
# ncu launch list of a short bench, ncu --set full of K1 (in the replay) and K2.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python __graft_entry__.py 2>&1 | tail -3
for m in 0 15 21; do timeout 120 python tools/kernel_bench.py $m 200 2>&1 | tail -1; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_line.json 2> gpurun_out/bench_err.log; tail -5 gpurun_out/bench_err.log
cat gpurun_out/bench_line.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_line.json 2> gpurun_out/bench_ref_err.log; cat gpurun_out/bench_ref_line.json; tail -3 gpurun_out/bench_ref_err.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 400 --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc -s 300 -c 4 -o gpurun_out/k1_full_replay python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 48 -c 4 -o gpurun_out/k2_full python tools/profile_catalog.py bert_c5 1 > /dev/null 2>&1
ls -la gpurun_out/
