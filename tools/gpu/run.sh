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
#   sanitize   compute-sanitizer memcheck / synccheck on K1, BERT per-op (d 768 / 1024), 2-SM, K5; racecheck BERT
#   bertmodes  C5 forward per BERT path (per-op, 2-SM GEMMs, K5 dataflow) + the BERT parity tests
#   bertbatch  12-layer BERT-base forward at 32 / 64 / 128 sequences, per-op vs K5
#   k5trace    K5 debug build (make K5_DEBUG=1) and one forward's per-item timeline (tools/k5_trace.py)
#   h2d        pinned host -> device copy rate (tools/h2d_rate.cu)
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
    san() { echo "---- $1 $2"; shift 2; timeout 600 compute-sanitizer --print-limit 4 "$@" 2>&1 | tail -3; }
    for tool in memcheck synccheck; do
      san $tool "K1 mlp" --tool $tool python tools/kernel_bench.py 0 1
      san $tool "BERT per-op 2 layers" --tool $tool python tools/bert_small.py 2 2 perop
      san $tool "BERT per-op d1024" --tool $tool python tools/bert_small.py 1 2 perop 1024
      san $tool "BERT 2-SM pair" --tool $tool python tools/bert_small.py 1 2 pair
      san $tool "BERT flow K5" --tool $tool python tools/bert_small.py 2 3 flow
    done
    san racecheck "BERT per-op" --tool racecheck python tools/bert_small.py 1 2 perop ;;
  bertmodes)
    for m in perop pair flow; do timeout 300 python tools/bert_bench.py 50 $m; done
    timeout 1500 python -m pytest tests/test_gpu_bert.py -q 2>&1 | tail -3 ;;
  bertbatch)
    for S in 32 64 128; do for m in perop flow; do timeout 300 python tools/bert_small.py 12 $S $m 768 20 | head -1; done; done ;;
  k5trace)
    make K5_DEBUG=1 -j16 > gpurun_out/k5build.log 2>&1 || { tail -20 gpurun_out/k5build.log; return 1; }
    GFX_K5_TRACE=gpurun_out/k5.trace timeout 120 python tools/bert_bench.py 10 flow
    python tools/k5_trace.py gpurun_out/k5.trace ;;
  h2d)
    mkdir -p tools/_bin && nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/h2d_rate.cu -o tools/_bin/h2d_rate \
      && timeout 120 tools/_bin/h2d_rate ;;
  *) echo "unknown task $t"; return 2 ;;
  esac
}

for t in "$@"; do
  run_task "$t" > "gpurun_out/$t.log" 2>&1
  echo "$t done (rc=$?)"
done
