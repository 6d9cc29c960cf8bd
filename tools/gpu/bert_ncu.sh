exec > gpurun_out/bert_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 430 -c 85 --csv --log-file gpurun_out/bert_launches.csv python tools/bert_bench.py 1 > /dev/null 2>&1
ls -la gpurun_out/bert_launches.csv
timeout 600 python -m pytest tests/test_gpu_bert.py -x -q -s 2>&1 | grep -E "worst|passed|failed|Error" | tail -5
timeout 300 python tools/bert_bench.py 50
