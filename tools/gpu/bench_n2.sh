exec > gpurun_out/bench_n2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-extras > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "rc=$?"
tail -5 gpurun_out/bench_n2.err
cat gpurun_out/bench_n2.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 2>/dev/null
echo "ref rc=$?"
