"""One K2 GEMM op of a small BERT through gfx_bert_gemm (sanitizer driver).
usage: python tools/bert_op.py <op 0..5> [tokens] [pair 0|1]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05601_b200 as gfx  # noqa: E402
from paper_2303_05601_b200 import _ffi as F  # noqa: E402

op = int(sys.argv[1])
T = int(sys.argv[2]) if len(sys.argv) > 2 else 256
pair = int(sys.argv[3]) if len(sys.argv) > 3 else 0
desc = gfx.models.bert_desc(1, T // 128, gfx.model_seed("bert-op"))
F.check(F.gfx_model_register(0, C.byref(desc)))
pages = C.c_int32()
F.check(F.gfx_model_pages(0, C.byref(pages)))
a = C.c_void_p()
F.check(F.gfx_arena_create(0, C.c_uint64((pages.value + 1) << 21), C.byref(a)))
F.check(F.gfx_arena_set_option(a, F.GFX_OPT_GEMM_PAIR, pair))
F.check(F.gfx_load_h2d(a, 0, None))
bufs = []
for n in (T * 3072 * 2, T * 3072 * 2, T * 3072 * 2):
    p = C.c_void_p()
    F.check(F.gfx_device_alloc(a, n, C.byref(p)))
    bufs.append(p)
F.check(F.gfx_bert_gemm(a, 0, 0, op, bufs[0], bufs[1], bufs[2], T))
F.check(F.gfx_synchronize(a))
print(f"bert op {op} T {T} pair {pair}: ok", flush=True)
F.check(F.gfx_arena_destroy(a))
