exec > gpurun_out/k2dbg.log 2>&1
timeout 300 python tools/bert_bench.py 3 0 2>&1 | cat
