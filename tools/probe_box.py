"""One-off hardware probe for the GPU box: host cores, PCIe H2D/D2H pinned bandwidth,
per-2MiB-chunk copy cost, D2D bandwidth. Output -> gpurun_out/probe.txt"""
import os, subprocess, time, torch
out = []
def p(*a):
    s = " ".join(str(x) for x in a); print(s); out.append(s)
p("nproc", os.cpu_count())
try:
    p(subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:1500])
except Exception as e:
    p("lscpu failed", e)
p(subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout)
p(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
dev = torch.device("cuda:0")
props = torch.cuda.get_device_properties(0)
p("props", props)
for mb in [2, 16, 64, 256, 1024]:
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            d.copy_(h, non_blocking=True)
        s.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        reps = max(2, 2048 // mb)
        e0.record(s)
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record(s); s.synchronize()
        t = e0.elapsed_time(e1) / reps
        p(f"H2D {mb} MiB: {t*1e3:.1f} us  {n/t/1e6:.2f} GB/s")
        e0.record(s)
        for _ in range(reps):
            h.copy_(d, non_blocking=True)
        e1.record(s); s.synchronize()
        t = e0.elapsed_time(e1) / reps
        p(f"D2H {mb} MiB: {t*1e3:.1f} us  {n/t/1e6:.2f} GB/s")
# chunked: 64 MiB as 32 x 2MiB copies
n = 64 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for reps in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        for i in range(32):
            d[i << 21:(i + 1) << 21].copy_(h[i << 21:(i + 1) << 21], non_blocking=True)
        e1.record(s)
        t1 = time.perf_counter()
        s.synchronize()
        t = e0.elapsed_time(e1)
        p(f"H2D 64MiB as 32x2MiB: {t*1e3:.1f} us {n/t/1e6:.2f} GB/s host-enqueue {1e6*(t1-t0):.1f} us")
x = torch.empty(1 << 30, dtype=torch.uint8, device=dev); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): y.copy_(x)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10
p(f"D2D 1GiB copy: {t:.3f} ms  {2*(1<<30)/t/1e6:.1f} GB/s (r+w)")
os.makedirs("gpurun_out", exist_ok=True)
open("gpurun_out/probe.txt", "w").write("\n".join(out))
