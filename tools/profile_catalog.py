"""B200 profiling pass for a model catalog (the paper's offline profiling step,
PAPER.md:372-374): per model, the pinned-host H2D load time and the batched
inference time, CUDA-event-free wall timing of synchronised C-ABI calls over
several repetitions (median). Writes gpurun_out/profile_<name>.json, consumed by
tools/make_mlp_catalog.py --profile / tools/make_bert_catalog.py --infer-ms."""
import ctypes as C
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05601_b200 as gfx  # noqa: E402
from paper_2303_05601_b200 import _ffi as F  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mlp_c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
specs = gfx.load_model_specs(name)
gfx.register_models(specs)
maxpages = max(s.pages for s in specs)
a = C.c_void_p()
F.check(F.gfx_arena_create(0, C.c_uint64(maxpages << 21), C.byref(a)))
out = {}
for i, s in enumerate(specs):
    inb, outb = C.c_uint64(), C.c_uint64()
    F.check(F.gfx_model_io_bytes(i, C.byref(inb), C.byref(outb)))
    x, y = C.c_void_p(), C.c_void_p()
    F.check(F.gfx_device_alloc(a, inb.value, C.byref(x)))
    F.check(F.gfx_device_alloc(a, outb.value, C.byref(y)))
    loads, infers = [], []
    for r in range(reps + 2):
        t0 = time.perf_counter()
        F.check(F.gfx_load_h2d(a, i, None))
        F.check(F.gfx_synchronize(a))
        t1 = time.perf_counter()
        batch = s.dims[5] if s.family == "bert" else 32
        for _ in range(5):
            F.check(F.gfx_infer(a, i, x, y, batch, None))
        F.check(F.gfx_synchronize(a))
        t2 = time.perf_counter()
        F.check(F.gfx_evict(a, i))
        if r >= 2:
            loads.append(t1 - t0)
            infers.append((t2 - t1) / 5)
    out[s.model_id] = {"load_s": statistics.median(loads), "infer_s": statistics.median(infers),
                       "bytes": s.bytes}
    F.check(F.gfx_device_free(a, x))
    F.check(F.gfx_device_free(a, y))
    print(s.model_id, f"load {out[s.model_id]['load_s'] * 1e3:.3f} ms  infer {out[s.model_id]['infer_s'] * 1e6:.1f} us",
          flush=True)
F.check(F.gfx_arena_destroy(a))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/profile_{name}.json", "w"), indent=1)
