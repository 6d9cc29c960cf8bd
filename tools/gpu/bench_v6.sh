exec > gpurun_out/bench_v6.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/bench_v6_line.json 2> gpurun_out/bench_v6_err.log; tail -3 gpurun_out/bench_v6_err.log
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_v6_line.json')); print(d['value'], d['e2e']['value'], d['roofline'])
PY
GFX_MLP_LAYERWISE=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/bench_v5_line.json 2>/dev/null
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_v5_line.json')); print(d['value'], d['e2e']['value'], d['roofline'])
PY
