exec > gpurun_out/bert_prof.log 2>&1
timeout 300 python tools/bert_bench.py 50
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 120 --csv --log-file gpurun_out/bert_launch_warm.csv python tools/bert_bench.py 1 > /dev/null 2>&1
echo done
