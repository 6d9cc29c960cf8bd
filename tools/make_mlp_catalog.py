"""Builds the configs[1] (C2) model catalog: the 22 Table-I model ids re-cast as
fp32 MLP classifiers 1024 -> h -> h -> h -> 1000 whose weights are ~ Table-I
occupation / 40. This keeps the size ordering, hence the
reference's model mapping (proj/src/workload.cpp:44-77) and the cache-pressure
ratio against an arena of 8192/40 ~ 204 MiB.

occupation_mb = 2 x arena pages (2 MiB each), so the reference capacity model
charges exactly what the paged HBM arena allocates. load/infer times come from
B200 measurements (--profile JSON from bench/profile runs) or, without one,
from the measured link rate (55 GB/s pinned H2D on this pool, gpurun_out/probe)
and a conservative FFMA rate. Writes paper_2303_05601_b200/data/mlp_c2_{catalog,models}.csv.
"""
import argparse
import csv
import json
import math
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAGE = 2 << 20


def mlp_bytes(dims):
    """Mirrors mlp_layout in csrc/device/manager.cu: per layer 16 KB-aligned
    weight tiles (rows padded to 128) then the 256 B-aligned bias."""
    align = lambda v, a: (v + a - 1) // a * a  # noqa: E731
    off = 0
    for k, n in zip(dims[:-1], dims[1:]):
        off = align(off, 16384) + 4 * k * align(n, 128)
        off = align(off, 256) + 4 * n
    return align(off, 256)


def mlp_flops(dims, batch=32):
    return sum(2.0 * batch * k * n for k, n in zip(dims[:-1], dims[1:]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--table1", default=os.path.join(ROOT, "tests", "golden", "table1_models.csv"))
    ap.add_argument("--scale", type=float, default=40.0)
    ap.add_argument("--profile", default=None, help="JSON {model_id: {load_s, infer_s}} measured on B200")
    ap.add_argument("--h2d-gbs", type=float, default=50.0)
    ap.add_argument("--tflops", type=float, default=30.0)
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2303_05601_b200", "data"))
    ap.add_argument("--name", default="mlp_c2")
    ap.add_argument("--paper-times", action="store_true",
                    help="keep Table-I load/infer seconds (the paper's regime) instead of B200 times")
    ap.add_argument("--c3", action="store_true",
                    help="configs[2]/[3] (C3/C4) catalog: 20 models of 25-100 MB evenly spaced, Table-I times "
                         "interpolated at size x scale (the paper regime), ids c3-00..c3-19")
    a = ap.parse_args()
    prof = json.load(open(a.profile)) if a.profile else {}
    rows = list(csv.DictReader(open(a.table1)))
    if a.c3:
        t1 = sorted(rows, key=lambda r: float(r["occupation_mb"]))
        occ = [float(r["occupation_mb"]) / a.scale for r in t1]

        def interp(x, key):
            ys = [float(r[key]) for r in t1]
            if x <= occ[0]:
                return ys[0]
            for i in range(1, len(occ)):
                if x <= occ[i]:
                    f = (x - occ[i - 1]) / max(occ[i] - occ[i - 1], 1e-9)
                    return ys[i - 1] + f * (ys[i] - ys[i - 1])
            return ys[-1]
        rows = []
        for j in range(20):
            mb = 25.0 + 75.0 * j / 19
            rows.append({"model_id": f"c3-{j:02d}", "occupation_mb": mb * a.scale,
                         "load_time_s": round(interp(mb, "load_time_s"), 2),
                         "infer_time_s": round(interp(mb, "infer_time_s"), 2)})
        a.paper_times = True
        a.name = "mlp_c3"
    cat, spec = [], []
    for r in rows:
        target = float(r["occupation_mb"]) / a.scale * (1 << 20)
        # 2h^2 + 2027h + 1000 floats ~ target/4
        h = (-2027 + math.sqrt(2027 ** 2 + 8 * (target / 4 - 1000))) / 4
        h = max(64, int(round(h / 64.0)) * 64)
        dims = [1024, h, h, h, 1000]
        nbytes = mlp_bytes(dims)
        pages = -(-nbytes // PAGE)
        mid = r["model_id"]
        if a.paper_times:
            load_s, infer_s = float(r["load_time_s"]), float(r["infer_time_s"])
        elif mid in prof:
            load_s, infer_s = prof[mid]["load_s"], prof[mid]["infer_s"]
        else:
            load_s = nbytes / (a.h2d_gbs * 1e9)
            infer_s = mlp_flops(dims) / (a.tflops * 1e12) + 20e-6
        cat.append((mid, 2 * pages, max(1e-6, round(load_s, 6)), max(1e-6, round(infer_s, 6))))
        spec.append((mid, "mlp", len(dims) - 1, "x".join(map(str, dims)), nbytes, pages))
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, f"{a.name}_catalog.csv"), "w") as f:
        f.write("model_id,occupation_mb,load_time_s,infer_time_s\n")
        for mid, occ, ls, inf in cat:
            f.write(f"{mid},{occ},{ls:.6f},{inf:.6f}\n")
    with open(os.path.join(a.out, f"{a.name}_models.csv"), "w") as f:
        f.write("model_id,family,layers,dims,bytes,pages\n")
        for s in spec:
            f.write(",".join(map(str, s)) + "\n")
    for c, s in zip(cat, spec):
        print(c, s[3], f"{s[4] / 2**20:.1f} MiB")


if __name__ == "__main__":
    main()
