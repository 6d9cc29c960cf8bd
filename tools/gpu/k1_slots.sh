exec > gpurun_out/k1_slots.log 2>&1
timeout 120 python __graft_entry__.py 2>&1 | tail -1
for m in 0 21; do GFX_MLP_REPEAT=200 timeout 60 python tools/kernel_bench.py $m 1 2>&1 | grep repeat | tail -1; done
GFX_TRACE_MLP=1 timeout 60 python tools/kernel_bench.py 21 1 2>&1 | grep -E "L1 mma first|L1 mma last|L2 mma first|L2 mma last"
