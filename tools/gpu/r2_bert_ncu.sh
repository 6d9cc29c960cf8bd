exec > gpurun_out/r2_bert_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 8 -c 4 \
  -o gpurun_out/r2_k2_full python tools/bert_bench.py 1 0
echo "rc=$?"
