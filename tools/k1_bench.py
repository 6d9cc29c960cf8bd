"""K1 back-to-back forward time per C2 model (resident weights, one arena holding
every model), wall time over many stream-ordered launches, and the roofline
fraction against MEASURED_PEAKS.json. usage: python tools/k1_bench.py [iters]"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.environ.get("GFX_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # GFX_PKG_ROOT: A/B a copy of the package
sys.path.insert(0, ROOT)
import paper_2303_05601_b200 as gfx
from paper_2303_05601_b200 import _ffi as F
import torch

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rows = [int(r) for r in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 7, 12, 15, 21]
specs = gfx.load_model_specs("mlp_c2")
gfx.register_models(specs)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
a = C.c_void_p()
F.check(F.gfx_arena_create(0, 2048 << 20, C.byref(a)))
for r in rows:
    F.check(F.gfx_load_h2d(a, r, None))
F.check(F.gfx_synchronize(a))
x = torch.empty(32 * 1024, device="cuda").uniform_(-1, 1)
y = torch.empty(2 * 32 * 1000, device="cuda")
for r in rows:
    s = specs[r]
    for _ in range(5):
        F.check(F.gfx_infer(a, r, x.data_ptr(), y.data_ptr(), 32, None))
    F.check(F.gfx_synchronize(a))
    t0 = time.perf_counter()
    for _ in range(iters):
        F.check(F.gfx_infer(a, r, x.data_ptr(), y.data_ptr(), 32, None))
    t_enq = time.perf_counter() - t0
    F.check(F.gfx_synchronize(a))
    per = (time.perf_counter() - t0) / iters
    alg = sum(4 * (k * n + n) for k, n in zip(s.dims[:-1], s.dims[1:])) + 4 * 32 * (s.dims[0] + 2 * s.dims[-1])
    print(f"row {r:2d} {s.model_id:18s} {'x'.join(map(str, s.dims)):28s} {per*1e6:7.1f} us  "
          f"{alg/per/1e9:6.0f} GB/s = {alg/per/1e9/peak:.3f} of HBM  (host enqueue {t_enq / iters * 1e6:.1f} us)", flush=True)
# all rows interleaved (a different model every launch, as in a replay of hits)
t0 = time.perf_counter()
for i in range(iters):
    r = rows[i % len(rows)]
    F.check(F.gfx_infer(a, r, x.data_ptr(), y.data_ptr(), 32, None))
F.check(F.gfx_synchronize(a))
print(f"interleaved: {(time.perf_counter() - t0) / iters * 1e6:.1f} us per forward")
F.gfx_arena_destroy(a)
