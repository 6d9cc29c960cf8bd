exec > gpurun_out/bert_ab2.log 2>&1
for i in 1 2; do
timeout 300 python tools/bert_bench.py 50
GFX_BERT_ERFF=1 timeout 300 python tools/bert_bench.py 50
done
timeout 600 python -m pytest tests/test_gpu_bert.py -x -q -s 2>&1 | grep -E "worst|passed|failed|Error" | tail -3
