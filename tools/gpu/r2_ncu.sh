# ncu --set full of K1 (two models: squeezenet1.1 and vgg19, warm launches).
exec > gpurun_out/r2_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mlp_forward -s 2 -c 2 \
  -o gpurun_out/r2_k1_full python tools/k1_prof.py 3
echo "full rc=$?"
