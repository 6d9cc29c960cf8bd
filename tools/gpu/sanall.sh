# compute-sanitizer matrix over every product kernel family (small shapes), then the GPU suite.
export PATH=/usr/local/cuda/bin:$PATH
run() { echo "---- $1 $2"; shift 2; timeout 600 compute-sanitizer --print-limit 4 "$@" 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok|done|us/inference|Error" | head -4; }
for t in memcheck synccheck; do
  run $t "K1 mlp" --tool $t python tools/kernel_bench.py 0 1
  run $t "BERT per-op 2 layers" --tool $t python tools/bert_small.py 2 2 perop
  run $t "BERT per-op d1024" --tool $t python tools/bert_small.py 1 2 perop 1024
  run $t "BERT 2-SM pair" --tool $t python tools/bert_small.py 1 2 pair
  run $t "BERT flow K5" --tool $t python tools/bert_small.py 2 3 flow
done
run racecheck "BERT per-op" --tool racecheck python tools/bert_small.py 1 2 perop
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2
