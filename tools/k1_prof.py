"""Minimal K1 workload for ncu --set full: two C2 models (rows 0 and 21) resident in
an arena sized for them, a few forwards each (small memory footprint, so each of
ncu's replay passes saves/restores little). usage: python tools/k1_prof.py [launches]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05601_b200 as gfx
from paper_2303_05601_b200 import _ffi as F

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
specs = gfx.load_model_specs("mlp_c2")
rows = [0, 21]
for r in rows:
    F.check(F.gfx_model_register(r, C.byref(specs[r].desc())))
pages = sum(specs[r].pages for r in rows)
a = C.c_void_p()
F.check(F.gfx_arena_create(0, C.c_uint64((pages + 2) << 21), C.byref(a)))
x, y = C.c_void_p(), C.c_void_p()
F.check(F.gfx_device_alloc(a, 32 * 1024 * 4, C.byref(x)))
F.check(F.gfx_device_alloc(a, 2 * 32 * 1000 * 4, C.byref(y)))
F.check(F.gfx_fill_params(a, C.cast(x, C.POINTER(C.c_float)), 32 * 1024, F.gfx_input_seed(0), 0xFFFFFFFF, 1.0))
for r in rows:
    F.check(F.gfx_load_h2d(a, r, None))
for r in rows:
    for _ in range(n):
        F.check(F.gfx_infer(a, r, x, y, 32, None))
F.check(F.gfx_synchronize(a))
F.gfx_arena_destroy(a)
print("ok")
