"""First GPU bring-up: smoke + one timed C2 replay (1950 requests) per policy."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as ge
t = time.time()
ge.smoke()
print("smoke s", time.time() - t)
import paper_2303_05601_b200 as gfx
cat = gfx.catalog_text("mlp_c2")
for pol in ("lb", "lalbo3"):
    cfg = gfx.sim_config(gpus=1, capacity_mb=204.0, policy=pol)
    rep = gfx.Replay(cat, cfg, record_kernels=True, record_requests=True)
    for i in range(3):
        r = rep.run()
        print(pol, i, json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.raw.items()}))
    print(pol, "req/s", r.n_requests / (r.device_ms / 1e3), "H2D GB/s", r.h2d_bytes / (r.h2d_ms * 1e6) if r.h2d_ms else 0,
          "kernel TFLOP/s", r.mlp_flops / (r.kernel_ms * 1e9) if r.kernel_ms else 0)
    rep.close()
