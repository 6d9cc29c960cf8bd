"""Summarise a K5 (encoder dataflow kernel) per-item timeline written by a
`make K5_DEBUG=1` build with GFX_K5_TRACE=<file> (bert_encoder_flow, one warm
forward). usage: python tools/k5_trace.py <file>

Per item: [0] item, [1] claimed, [2] inputs ready, [3] first stage in the MMA
warp, [4] last MMA issued, [5] epilogue saw the accumulator, [6] epilogue done,
[7] LayerNorm ran here."""
import sys

import numpy as np

OPS = ["qkv", "att", "o", "ffn1", "ffn2"]

raw = open(sys.argv[1], "rb").read()
ctas, per, M, L = np.frombuffer(raw[:16], np.int32)
v = np.frombuffer(raw[16:], np.uint64).reshape(ctas, per, 8).astype(np.int64)
valid = (v[:, :, 1] > 0) & (((v[:, :, 0] >> 29) & 7) != 7)
t0 = v[:, :, 1][valid].min()
t = np.where(valid[:, :, None], (v - t0) / 1e3, np.nan)  # µs
t[:, :, 0] = v[:, :, 0]
t[:, :, 7] = np.where(v[:, :, 7] > 1, (v[:, :, 7] - t0) / 1e3, 0.0)
items = v[:, :, 0][valid]
op = (items >> 29) & 7
span = np.nanmax(t[:, :, 6])
print(f"K5 trace: {ctas} CTAs, {M} row blocks, {L} layers, {valid.sum()} items, forward span {span:.1f} us")


def stat(x):
    x = x[np.isfinite(x)]
    if not len(x):
        return "-"
    return f"{np.mean(x):6.2f} {np.median(x):6.2f} {np.percentile(x, 90):6.2f} {x.max():7.2f}"


f = {k: t[:, :, k][valid] for k in range(8)}
print("phase (us): mean median p90 max")
for o in range(5):
    s = op == o
    print(f"  {OPS[o]:5s} n={s.sum():5d}  popped->1st stage {stat(f[3][s] - f[1][s])}"
          f" | MMA {stat(f[4][s] - f[3][s])} | MMA->epi {stat(f[5][s] - f[4][s])} | epilogue {stat(f[6][s] - f[5][s])}")
ln = f[7] > 0
for o in (2, 4):
    s = ln & (op == o)
    print(f"  LayerNorm after {OPS[o]}: n={s.sum():4d}  stats+count -> LN start {stat(f[7][s] - f[5][s])} | LN {stat(f[6][s] - f[7][s])}")
# MMA pipe occupancy: time between consecutive items' MMA phases.
mma_items = ((t[:, :, 0].astype(np.int64) >> 29) & 7) < 5
busy = np.nansum(np.where(mma_items, t[:, :, 4] - t[:, :, 3], 0.0))
print(f"MMA phases cover {busy / (ctas * span):.3f} of CTAs x span")
gaps, dep_gaps = [], []
for c in range(ctas):
    n = int(valid[c].sum())
    for j in range(1, n):
        g = t[c, j, 3] - t[c, j - 1, 4]
        if not np.isfinite(g):
            continue
        gaps.append(g)
        dep_gaps.append(max(0.0, t[c, j, 2] - t[c, j - 1, 4]))
gaps, dep_gaps = np.array(gaps), np.array(dep_gaps)
print(f"gaps between a CTA's MMA phases: total {np.nansum(gaps) / ctas:.1f} us per CTA,"
      f" of which waiting for inputs {np.nansum(np.minimum(dep_gaps, np.maximum(gaps, 0))) / ctas:.1f} us")
first = np.nanmin(t[:, :, 3])
last = np.nanmax(t[:, :, 4])
print(f"first MMA {first:.1f} us, last MMA {last:.1f} us, tail after last MMA {span - last:.1f} us")
# Per layer progress: when the layer's first item started and its last finished.
lay = (items >> 24) & 31
for l in range(L):
    s = lay == l
    print(f"  layer {l:2d}: claimed {np.min(f[1][s]):7.1f} .. {np.max(f[1][s]):7.1f}  done {np.min(f[6][s]):7.1f} .. {np.max(f[6][s]):7.1f}")
# Concurrency histogram: MMA phases active per 5 us bucket.
edges = np.arange(0, span + 5, 5.0)
act = np.zeros(len(edges) - 1)
for c in range(ctas):
    for j in range(int(valid[c].sum())):
        a, b = t[c, j, 3], t[c, j, 4]
        if np.isfinite(a) and np.isfinite(b):
            lo, hi = np.searchsorted(edges, a), np.searchsorted(edges, b)
            for k in range(max(lo - 1, 0), min(hi, len(act))):
                act[k] += max(0.0, min(b, edges[k + 1]) - max(a, edges[k])) / 5.0
print("CTAs in an MMA phase per 5 us:", " ".join(f"{int(round(x))}" for x in act))
