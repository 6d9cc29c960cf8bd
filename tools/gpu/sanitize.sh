exec > gpurun_out/sanitize.log 2>&1
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/kernel_bench.py 0 1 2>&1 | tail -8
echo "---- memcheck bert"
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/bert_bench.py 1 2>&1 | tail -8
echo "---- synccheck mlp"
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/kernel_bench.py 0 1 2>&1 | tail -6
echo "---- racecheck mlp"
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/kernel_bench.py 0 1 2>&1 | tail -8
