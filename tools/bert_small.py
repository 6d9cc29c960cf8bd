"""BERT forwards through the C-ABI (sanitizer driver, batch-size sweeps): L layers, S
sequences, mode flow | perop | pair, width d; with iters > 0 also times `iters` back-to-back
forwards. usage: python tools/bert_small.py [L] [S] [mode] [d] [iters]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05601_b200 as gfx  # noqa: E402
from paper_2303_05601_b200 import _ffi as F  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mode = sys.argv[3] if len(sys.argv) > 3 else "perop"
d = int(sys.argv[4]) if len(sys.argv) > 4 else 768
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 0
desc = gfx.models.bert_desc(L, S, gfx.model_seed("bert-small"), d=d, heads=d // 64, ffn=4 * d)
F.check(F.gfx_model_register(0, C.byref(desc)))
pages = C.c_int32()
F.check(F.gfx_model_pages(0, C.byref(pages)))
a = C.c_void_p()
F.check(F.gfx_arena_create(0, C.c_uint64((pages.value + 1) << 21), C.byref(a)))
F.check(F.gfx_arena_set_option(a, F.GFX_OPT_GEMM_PAIR, int(mode == "pair")))
F.check(F.gfx_arena_set_option(a, F.GFX_OPT_BERT_FLOW, int(mode == "flow")))
F.check(F.gfx_load_h2d(a, 0, None))
inb, outb = C.c_uint64(), C.c_uint64()
F.check(F.gfx_model_io_bytes(0, C.byref(inb), C.byref(outb)))
x, y = C.c_void_p(), C.c_void_p()
F.check(F.gfx_device_alloc(a, inb.value, C.byref(x)))
F.check(F.gfx_device_alloc(a, outb.value, C.byref(y)))
for i in range(2):
    F.check(F.gfx_infer(a, 0, x, y, S, None))
    F.check(F.gfx_synchronize(a))
    if not iters:
        print(f"forward {i} ok", flush=True)
if iters:
    import time
    t0 = time.perf_counter()
    for _ in range(iters):
        F.check(F.gfx_infer(a, 0, x, y, S, None))
    F.check(F.gfx_synchronize(a))
    dt = (time.perf_counter() - t0) / iters
    T = S * 128
    flops = L * (2.0 * T * (4 * d * d + 2 * d * 4 * d) + 4.0 * T * 128 * d) + 2.0 * S * d * d
    print(f"bert L={L} S={S} d={d} {mode}: {dt * 1e3:.3f} ms/forward  {flops / dt / 1e12:.1f} TFLOP/s", flush=True)
F.check(F.gfx_arena_destroy(a))
print(f"bert small L={L} S={S} d={d} {mode}: done", flush=True)
