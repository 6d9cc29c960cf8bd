# K5 debug timeline on the box: rebuild with K5_DEBUG=1 (scratch copy), trace one warm forward.
export PATH=/usr/local/cuda/bin:$PATH
make K5_DEBUG=1 -j16 > gpurun_out/k5build.log 2>&1 || { tail -20 gpurun_out/k5build.log; exit 1; }
GFX_K5_TRACE=gpurun_out/k5.trace timeout 120 python tools/bert_bench.py 10 flow
python tools/k5_trace.py gpurun_out/k5.trace
