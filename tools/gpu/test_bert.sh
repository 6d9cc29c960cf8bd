set -x
timeout 900 python -m pytest tests/test_gpu_bert.py -x -q -s 2>&1 | tail -15
bash tools/gpu/trace_mlp.sh
