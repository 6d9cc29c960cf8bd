# Full bench (product arm with extras) + reference arm, as the driver runs them.
mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?" > gpurun_out/bench_rc.txt
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench_rc.txt
nproc >> gpurun_out/bench_rc.txt
