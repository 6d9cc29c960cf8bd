exec > gpurun_out/attn_poly2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bert.py -x -q 2>&1 | grep -E "^E |Error|assert" | head -20
