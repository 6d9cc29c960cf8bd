# K1 release timings: back-to-back forwards per C2 model + interleaved; then smoke.
exec > gpurun_out/r2_k1.log 2>&1
timeout 300 python tools/k1_bench.py 300 0,3,7,12,15,16,18,21 2>&1 | tail -12
timeout 300 python __graft_entry__.py 2>&1 | tail -2
