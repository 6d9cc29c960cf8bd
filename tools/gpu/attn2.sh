exec > gpurun_out/attn2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem --clock-control none -k regex:attention -s 5 -c 3 --csv python tools/bert_bench.py 1 2>&1 | tail -15
