"""Device time of one BERT-base (C5) forward through the C-ABI: model 0 of the
bert_c5 catalog resident, `iters` back-to-back gfx_infer calls, wall time of the
synchronised loop (host launch cost ~0.2 ms/forward < device time).
usage: python tools/bert_bench.py [iters] [flow|perop|pair]
  flow: the encoder dataflow kernel K5 (default); perop: per-op K2-K4 launches;
  pair: per-op with 2-SM GEMMs"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05601_b200 as gfx  # noqa: E402
from paper_2303_05601_b200 import _ffi as F  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
specs = gfx.load_model_specs("bert_c5")
gfx.register_models(specs[:1])
s = specs[0]
a = C.c_void_p()
F.check(F.gfx_arena_create(0, C.c_uint64(s.pages << 21), C.byref(a)))
mode = sys.argv[2] if len(sys.argv) > 2 else "flow"
assert mode in ("flow", "perop", "pair"), mode
F.check(F.gfx_arena_set_option(a, F.GFX_OPT_GEMM_PAIR, int(mode == "pair")))
F.check(F.gfx_arena_set_option(a, F.GFX_OPT_BERT_FLOW, int(mode == "flow")))
F.check(F.gfx_load_h2d(a, 0, None))
inb, outb = C.c_uint64(), C.c_uint64()
F.check(F.gfx_model_io_bytes(0, C.byref(inb), C.byref(outb)))
x, y = C.c_void_p(), C.c_void_p()
F.check(F.gfx_device_alloc(a, inb.value, C.byref(x)))
F.check(F.gfx_device_alloc(a, outb.value, C.byref(y)))
batch = s.dims[5]
for _ in range(5):
    F.check(F.gfx_infer(a, 0, x, y, batch, None))
F.check(F.gfx_synchronize(a))
t0 = time.perf_counter()
for _ in range(iters):
    F.check(F.gfx_infer(a, 0, x, y, batch, None))
F.check(F.gfx_synchronize(a))
dt = (time.perf_counter() - t0) / iters
L, D, FF, S = s.dims[0], s.dims[1], s.dims[3], s.dims[4]
T = batch * S
flops = L * (2.0 * T * (4 * D * D + 2 * D * FF) + 4.0 * T * S * D) + 2.0 * batch * D * D
print(f"bert {s.model_id} ({mode}): {dt * 1e3:.3f} ms/forward  {flops / dt / 1e12:.1f} TFLOP/s")
