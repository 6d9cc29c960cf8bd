set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 600 python tools/profile_catalog.py mlp_c2 10 > gpurun_out/profile_mlp_c2.log 2>&1; tail -3 gpurun_out/profile_mlp_c2.log
timeout 600 python tools/profile_catalog.py bert_c5 5 > gpurun_out/profile_bert_c5.log 2>&1; tail -3 gpurun_out/profile_bert_c5.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_line.json 2> gpurun_out/bench_err.log; tail -3 gpurun_out/bench_err.log; cat gpurun_out/bench_line.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mlp_tc|softmax" -c 300 --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tc -s 9 -c 1 -o gpurun_out/k1_full python tools/kernel_bench.py 21 4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 24 -c 4 -o gpurun_out/k2_full python tools/profile_catalog.py bert_c5 1 > /dev/null 2>&1
ls -la gpurun_out/
