set -x
timeout 120 python tools/kernel_bench.py 21 100 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mlp_tc -c 24 --csv --log-file gpurun_out/tc_launches.csv python tools/kernel_bench.py 21 4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tc -s 8 -c 4 -o gpurun_out/tc_prof python tools/kernel_bench.py 21 4 > gpurun_out/tc_ncu.log 2>&1
tail -2 gpurun_out/tc_ncu.log
