exec > gpurun_out/prof_final.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 300 -c 200 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
echo rc=$?
