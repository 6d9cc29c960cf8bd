"""Micro-benchmark of the K1 inference path on one resident model via the C-ABI
(gfx_arena_create / gfx_load_h2d / gfx_infer), CUDA-event timed.
usage: python tools/kernel_bench.py [model_row] [iters]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05601_b200 as gfx
from paper_2303_05601_b200 import _ffi as F
import torch

row = int(sys.argv[1]) if len(sys.argv) > 1 else 21
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
specs = gfx.load_model_specs("mlp_c2")
gfx.register_models(specs)
a = C.c_void_p()
F.check(F.gfx_arena_create(0, 204 << 20, C.byref(a)))
F.check(F.gfx_load_h2d(a, row, None))
F.check(F.gfx_synchronize(a))
s = specs[row]
x = torch.empty(32 * s.dims[0], device="cuda").uniform_(-1, 1)
y = torch.empty(2 * 32 * s.dims[-1], device="cuda")
for _ in range(5):
    F.check(F.gfx_infer(a, row, x.data_ptr(), y.data_ptr(), 32, None))
F.check(F.gfx_synchronize(a))
t0 = time.perf_counter()
for _ in range(iters):
    F.check(F.gfx_infer(a, row, x.data_ptr(), y.data_ptr(), 32, None))
F.check(F.gfx_synchronize(a))
t1 = time.perf_counter()
flops = sum(2 * 32 * k * n for k, n in zip(s.dims[:-1], s.dims[1:]))
per = (t1 - t0) / iters
print(f"model {s.model_id} dims {s.dims}: {per*1e6:.1f} us/inference  {flops/per/1e12:.2f} TFLOP/s  "
      f"weights {s.bytes/per/1e9:.0f} GB/s")
