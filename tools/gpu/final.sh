# Round-end validation: GPU tests + smoke, both bench arms, launch list, BERT forwards, H2D rate.
export PATH=/usr/local/cuda/bin:$PATH
bash tools/gpu/run.sh tests bench launches
timeout 300 python tools/bert_bench.py 50 perop > gpurun_out/bert_modes.log 2>&1
timeout 300 python tools/bert_bench.py 50 flow >> gpurun_out/bert_modes.log 2>&1
timeout 300 python tools/bert_bench.py 50 pair >> gpurun_out/bert_modes.log 2>&1
mkdir -p tools/_bin && nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/h2d_rate.cu -o tools/_bin/h2d_rate && timeout 120 tools/_bin/h2d_rate > gpurun_out/h2d_rate.txt 2>&1
