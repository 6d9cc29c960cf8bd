exec > gpurun_out/rep_v6.log 2>&1
for ab in 0 128; do echo "== ablate $ab"; GFX_MLP_ABLATE=$ab GFX_MLP_REPEAT=200 timeout 120 python tools/kernel_bench.py 21 1 2>&1 | grep repeat | tail -1
GFX_MLP_ABLATE=$ab GFX_TRACE_MLP=1 timeout 60 python tools/kernel_bench.py 21 1 2>&1 | grep -E "L0 |L1 mma first|end " | head -17; done
