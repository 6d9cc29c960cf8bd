exec > gpurun_out/bert_ab.log 2>&1
timeout 300 python tools/bert_bench.py 50
GFX_BERT_BN=256 timeout 300 python tools/bert_bench.py 50
