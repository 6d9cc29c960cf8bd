exec > gpurun_out/k2_ncu_v3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16|attention_tc|layernorm" -s 40 -c 6 -o gpurun_out/k2_full_v3 python tools/bert_bench.py 1 > /dev/null 2>&1
echo rc=$?
ls -la gpurun_out/k2_full_v3.ncu-rep
