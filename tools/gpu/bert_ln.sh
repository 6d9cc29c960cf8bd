exec > gpurun_out/bert_ln.log 2>&1
timeout 300 python tools/bert_bench.py 50 2>&1 | tail -1
GFX_BERT_UNFUSED_LN=1 timeout 300 python tools/bert_bench.py 50 2>&1 | tail -1
timeout 300 python tools/bert_bench.py 50 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_bert.py -x -q 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 120 --csv --log-file gpurun_out/bert_launch_warm3.csv python tools/bert_bench.py 1 > /dev/null 2>&1
