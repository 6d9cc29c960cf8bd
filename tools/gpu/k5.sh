# K5 check + timing + debug timeline on the box.
export PATH=/usr/local/cuda/bin:$PATH
timeout 120 python tools/bert_bench.py 20 flow
timeout 900 python -m pytest tests/test_gpu_bert.py -x -q -k "c5_shape or ragged or one_layer or every_layer" 2>&1 | tail -3
timeout 120 python tools/bert_bench.py 50 flow
make K5_DEBUG=1 -j16 > gpurun_out/k5build.log 2>&1 || { tail -20 gpurun_out/k5build.log; exit 1; }
GFX_K5_TRACE=gpurun_out/k5.trace timeout 120 python tools/bert_bench.py 10 flow
python tools/k5_trace.py gpurun_out/k5.trace
