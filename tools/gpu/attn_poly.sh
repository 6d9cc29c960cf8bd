exec > gpurun_out/attn_poly.log 2>&1
timeout 300 python tools/bert_bench.py 50 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_bert.py -x -q -s 2>&1 | grep -E "worst per-layer|passed|failed|^E " | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:attention -c 12 --csv --log-file gpurun_out/attn_poly.csv python tools/bert_bench.py 1 > /dev/null 2>&1
