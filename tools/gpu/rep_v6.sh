exec > gpurun_out/rep_v6.log 2>&1
timeout 120 python __graft_entry__.py 2>&1 | tail -1
for m in 0 7 15 21; do GFX_MLP_REPEAT=200 timeout 120 python tools/kernel_bench.py $m 1 2>&1 | grep repeat | tail -1; done
GFX_TRACE_MLP=1 timeout 60 python tools/kernel_bench.py 21 1 2>&1 | grep -E "mma first|mma last|end " | head -10
