set -x
python tools/kernel_bench.py 21 200 2>&1 | tail -2
python tools/kernel_bench.py 0 200 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mlp_layer -c 40 --csv --log-file gpurun_out/k1_launches.csv python tools/kernel_bench.py 21 10 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:mlp_layer -s 8 -c 4 -o gpurun_out/k1_prof python tools/kernel_bench.py 21 5 > gpurun_out/k1_ncu.log 2>&1
tail -3 gpurun_out/k1_ncu.log
