exec > gpurun_out/fleet.log 2>&1
timeout 900 python - <<'PY'
import sys, json, time
sys.path.insert(0, '.')
import bench
import paper_2303_05601_b200 as gfx
gfx.register_models(gfx.load_model_specs("mlp_c2"))
t=time.time()
print(json.dumps(bench.locality_extras(gfx, 1), indent=1))
print("took", time.time()-t)
PY
