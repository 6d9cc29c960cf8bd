export PATH=/usr/local/cuda/bin:$PATH
echo ---- memcheck op 4
timeout 200 compute-sanitizer --tool memcheck --print-limit 4 python tools/bert_op.py 4 512 2>&1 | tail -3
echo ---- memcheck op 5 pair
timeout 200 compute-sanitizer --tool memcheck --print-limit 4 python tools/bert_op.py 0 512 1 2>&1 | tail -3
for i in 1 2; do timeout 300 python tools/bert_bench.py 50 perop; done
