# K1 debug build (make K1_DEBUG=1: watchdogs + per-CTA phase table every 64 launches).
exec > gpurun_out/k1dbg.log 2>&1
timeout 120 python tools/k1_bench.py 72 21 2>&1 | head -80
timeout 120 python __graft_entry__.py 2>&1 | tail -3
