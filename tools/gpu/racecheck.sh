exec > gpurun_out/racecheck.log 2>&1
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 python tools/kernel_bench.py 0 1 2>&1 | grep -v "^=========     and" | head -60
