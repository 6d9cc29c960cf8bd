exec > gpurun_out/prof_v6.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_forward -s 5 -c 1 -o gpurun_out/k1v6_full python tools/kernel_bench.py 21 8
