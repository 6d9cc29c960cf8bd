#!/usr/bin/env bash
# One entry point for the GPU-box jobs this repo runs through gpurun:
#   /usr/local/graft/bin/gpurun --timeout S -- 'bash tools/gpu/run.sh <task> [<task> ...]'
# Each task writes gpurun_out/<task>.log (plus its own artefacts) and never
# aborts the tasks after it.
#
#   tests      -m gpu suite + smoke
#   bench      bench.py as the driver runs it: reference arm, then the product arm (N = 1)
#   bench2     bench.py --gpus 2 under torchrun (both ranks on one B200: the N > 1 path)
#   k1         K1 back-to-back forwards per C2 model and interleaved (tools/k1_bench.py)
#   bert       C5 BERT forward (single-CTA and 2-SM GEMMs) and the cuBLAS/torch baseline
#   launches   ncu launch list of one bench step (gpu__time_duration + DRAM bytes per launch)
#   ncu-k1     ncu --set full of two K1 forwards (tools/k1_prof.py)
#   ncu-bert   ncu launch list of one BERT forward + --set full of its K2 GEMMs / attention
#   sanitize   compute-sanitizer memcheck / synccheck / racecheck on K1 and BERT
set -u
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH

run_task() {
  local t=$1
  case "$t" in
  tests)
    nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
    timeout 2400 python -m pytest tests -m gpu -q --durations=8 2>&1 | tail -20
    timeout 300 python __graft_entry__.py 2>&1 | tail -2 ;;
  bench)
    timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
    echo "ref rc=$?"
    timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
    echo "bench rc=$?"; nproc ;;
  bench2)
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
    echo "rc=$?"; tail -3 gpurun_out/bench_n2.err ;;
  k1)
    timeout 300 python tools/k1_bench.py 300 0,3,7,12,15,16,18,21 2>&1 | tail -12 ;;
  bert)
    timeout 300 python tools/bert_bench.py 50 perop
    timeout 300 python tools/bert_bench.py 50 pair
    timeout 300 python tools/cublas_bert.py 50 ;;
  launches)
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -s 300 -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-extras > /dev/null 2>&1
    echo "rc=$?" ;;
  ncu-k1)
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mlp_forward -s 2 -c 2 \
      -o gpurun_out/k1_full -f python tools/k1_prof.py 3
    echo "rc=$?" ;;
  ncu-bert)
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -s 130 -c 61 --csv --log-file gpurun_out/bert_launches.csv python tools/bert_bench.py 2 perop > /dev/null 2>&1
    echo "list rc=$?"
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16|attention" -s 130 -c 5 \
      -o gpurun_out/bert_full -f python tools/bert_bench.py 2 perop
    echo "full rc=$?" ;;
  sanitize)
    for tool in memcheck synccheck racecheck; do
      echo "---- $tool mlp"
      timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/kernel_bench.py 0 1 2>&1 | tail -8
    done
    echo "---- memcheck bert"
    timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/bert_bench.py 1 2>&1 | tail -8 ;;
  *) echo "unknown task $t"; return 2 ;;
  esac
}

for t in "$@"; do
  run_task "$t" > "gpurun_out/$t.log" 2>&1
  echo "$t done (rc=$?)"
done
