set -x
timeout 600 python -m pytest tests/test_gpu_bert.py -x -q 2>&1 | tail -4
timeout 300 python tools/profile_catalog.py bert_c5 3 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"gemm|attention|layernorm|pooler" -s 30 -c 12 --csv --log-file gpurun_out/k2_launches.csv python tools/profile_catalog.py bert_c5 1 > /dev/null 2>&1
