exec > gpurun_out/prof_v6.log 2>&1
set -x
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 300 -c 200 --csv --log-file gpurun_out/v6_launches.csv python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_forward -s 300 -c 3 -o gpurun_out/k1v6_replay python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
ls -la gpurun_out
