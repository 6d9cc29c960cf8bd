"""Builds the configs[4] (C5) catalog: 20 BERT-base encoders (12 layers, d 768,
12 heads, ffn 3072, 128-token sequences, 32 sequences per request, bf16),
different parameter seeds. occupation_mb = 2 x arena pages of the blob
(bert_layout in csrc/device/bert.cu). load = blob bytes / 50 GB/s pinned H2D;
infer from --infer-ms (B200-measured) or an estimate at 1.0 PFLOP/s.
Writes paper_2303_05601_b200/data/bert_c5_{catalog,models}.csv."""
import argparse
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAGE = 2 << 20


def bert_bytes(L=12, d=768, ffn=3072):
    align = lambda v, a: (v + a - 1) // a * a  # noqa: E731
    off = 0

    def wmat(n, k):
        nonlocal off
        off = align(off, 16384) + align(n, 128) * k * 2

    def vec(n):
        nonlocal off
        off = align(off, 256) + 4 * n

    for _ in range(L):
        wmat(3 * d, d); vec(3 * d); wmat(d, d); vec(d); vec(d); vec(d)
        wmat(ffn, d); vec(ffn); wmat(d, ffn); vec(d); vec(d); vec(d)
    wmat(d, d); vec(d)
    return align(off, 256)


def bert_flops(L=12, d=768, ffn=3072, seq=128, seqs=32):
    T = seqs * seq
    return L * (2.0 * T * (3 * d * d + d * d + 2 * d * ffn) + 4.0 * T * seq * d) + 2.0 * seqs * d * d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", type=int, default=20)
    ap.add_argument("--infer-ms", type=float, default=None)
    ap.add_argument("--h2d-gbs", type=float, default=50.0)
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2303_05601_b200", "data"))
    a = ap.parse_args()
    nb = bert_bytes()
    pages = -(-nb // PAGE)
    infer_s = a.infer_ms / 1e3 if a.infer_ms else bert_flops() / 1.0e15
    load_s = nb / (a.h2d_gbs * 1e9)
    with open(os.path.join(a.out, "bert_c5_catalog.csv"), "w") as f:
        f.write("model_id,occupation_mb,load_time_s,infer_time_s\n")
        for i in range(a.models):
            f.write(f"bert-{i:02d},{2 * pages},{load_s:.6f},{infer_s:.6f}\n")
    with open(os.path.join(a.out, "bert_c5_models.csv"), "w") as f:
        f.write("model_id,family,layers,dims,bytes,pages\n")
        for i in range(a.models):
            f.write(f"bert-{i:02d},bert,12,12x768x12x3072x128x32,{nb},{pages}\n")
    print(f"{a.models} models, {nb / 2**20:.1f} MiB ({pages} pages) each, load {load_s * 1e3:.2f} ms, "
          f"infer {infer_s * 1e3:.3f} ms, {bert_flops() / 1e12:.3f} TFLOP/request")


if __name__ == "__main__":
    main()
