exec > gpurun_out/bert_t.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bert.py -x -q 2>&1 | tail -3
