exec > gpurun_out/bench_time.log 2>&1
start=$(date +%s); timeout 1500 python bench.py > gpurun_out/bench_default.json 2>/dev/null; echo "default bench rc=$? secs=$(( $(date +%s) - start ))"
start=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_default_ref.json 2>/dev/null; echo "reference arm rc=$? secs=$(( $(date +%s) - start ))"
tail -c 300 gpurun_out/bench_default_ref.json
