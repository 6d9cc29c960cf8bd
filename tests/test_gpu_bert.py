"""C5 model family on B200: BERT-base encoder (bf16 activations, fp32
accumulation, post-LN, tanh pooler) — tcgen05 GEMMs with fused bias / GELU /
residual epilogues, tcgen05 attention, LayerNorm — against the oracle's fp64
restatement with the same bf16 rounding points. Tolerance (north star, bf16):
normwise relative error <= 1e-3.

Why teacher forcing: this bf16 network is chaotic with respect to rounding
flips — perturbing ONE of the 196 608 input values by one bf16 ulp moves the
pooled output by 6e-4 after one layer and 1.7e-3 after two (measured with the
oracle alone; fp32 vs fp64 accumulation differs by 1.6e-3 after two layers).
End-to-end 1e-3 parity of a deep stack is therefore ill-posed for ANY
implementation that is not the oracle's exact operation order. The well-posed
check is per layer: feed each oracle layer the GPU's own input to that layer
and compare outputs — done here for all 12 layers of full BERT-base, at
2 x 128 tokens and at the C5 request shape (32 sequences x 128 tokens = 4096
tokens, where every persistent GEMM CTA runs 2-3 tiles and reuses its TMEM
accumulators), for the encoder dataflow kernel K5 (the production path) and
the per-op launches with single-CTA and 2-SM GEMM kernels, plus K5 at ragged
batches (1, 3, 37 sequences). Each fused GEMM
epilogue (bias, GELU, residual) is also checked alone against a numpy fp64
GEMM with the same bf16 rounding point."""
import ctypes as C
import os

import numpy as np
import pytest

import simabi

pytestmark = pytest.mark.gpu
TOL = 1e-3
D, SEQ = 768, 128


@pytest.fixture(scope="module")
def gfx():
    import paper_2303_05601_b200 as g
    n = C.c_int(0)
    g.check(g._ffi.gfx_device_count(C.byref(n)))
    assert n.value >= 1
    return g


@pytest.fixture(scope="module")
def olib():
    lib = C.CDLL(simabi.ORACLE_SO)
    lib.orc_bert_forward.restype = C.c_int
    lib.orc_bert_forward.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                     C.c_void_p, C.c_int]
    lib.orc_bert_layer.restype = C.c_int
    lib.orc_bert_layer.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_int]
    lib.orc_bert_layer_masked.restype = C.c_int
    lib.orc_bert_layer_masked.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
    lib.orc_bert_pool.restype = C.c_int
    lib.orc_bert_pool.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    lib.orc_fill_params.restype = None
    lib.orc_fill_params.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_float, C.c_void_p]
    return lib


def bf16_to_f32(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run_gpu(gfx, idx, layers, seqs, seed, request_id=7, debug=True, mode="perop", d=D, ffn=3072, lengths=None,
            seq=SEQ):
    desc = gfx.models.bert_desc(layers, seqs, seed, d=d, heads=d // 64, ffn=ffn, seq=seq)
    gfx.check(gfx._ffi.gfx_model_register(idx, C.byref(desc)))
    inb, outb = C.c_uint64(), C.c_uint64()
    gfx.check(gfx._ffi.gfx_model_io_bytes(idx, C.byref(inb), C.byref(outb)))
    assert inb.value == seqs * seq * d * 2 and outb.value == seqs * d * 4
    pages = C.c_int32()
    gfx.check(gfx._ffi.gfx_model_pages(idx, C.byref(pages)))
    a = C.c_void_p()
    gfx.check(gfx._ffi.gfx_arena_create(0, (pages.value + 2) << 21, C.byref(a)))
    try:
        gfx.check(gfx._ffi.gfx_arena_set_option(a, gfx._ffi.GFX_OPT_GEMM_PAIR, int(mode == "pair")))
        gfx.check(gfx._ffi.gfx_arena_set_option(a, gfx._ffi.GFX_OPT_BERT_FLOW, int(mode == "flow")))
        x_bits = np.zeros(inb.value // 2, np.uint16)
        gfx.check(gfx._ffi.gfx_host_fill_input(idx, request_id, x_bits.ctypes.data, inb.value))
        xd, yd, hd = C.c_void_p(), C.c_void_p(), C.c_void_p()
        hbytes = (layers + 1) * inb.value
        gfx.check(gfx._ffi.gfx_device_alloc(a, inb.value, C.byref(xd)))
        gfx.check(gfx._ffi.gfx_device_alloc(a, outb.value, C.byref(yd)))
        gfx.check(gfx._ffi.gfx_device_alloc(a, hbytes, C.byref(hd)))
        gfx.check(gfx._ffi.gfx_memcpy_h2d(a, xd, x_bits.ctypes.data, inb.value))
        gfx.check(gfx._ffi.gfx_load_h2d(a, idx, None))
        lp = None if lengths is None else np.ascontiguousarray(lengths, np.int32)

        def infer(hid=None):
            if lp is None and hid is None:
                gfx.check(gfx._ffi.gfx_infer(a, idx, xd, yd, seqs, None))  # production (PDL-chained) path
            elif lp is None:
                gfx.check(gfx._ffi.gfx_infer_debug(a, idx, xd, yd, seqs, hid))
            else:
                gfx.check(gfx._ffi.gfx_infer_masked(a, idx, xd, yd, seqs, lp.ctypes.data, hid, None))
        infer()
        pooled = np.zeros((seqs, d), np.float32)
        gfx.check(gfx._ffi.gfx_memcpy_d2h(a, pooled.ctypes.data, yd, outb.value))
        infer()
        again = np.zeros_like(pooled)
        gfx.check(gfx._ffi.gfx_memcpy_d2h(a, again.ctypes.data, yd, outb.value))
        hidden = None
        if debug:
            infer(hd)
            hidden = np.zeros((layers + 1, seqs * seq * d), np.uint16)
            gfx.check(gfx._ffi.gfx_memcpy_d2h(a, hidden.ctypes.data, hd, hbytes))
            dbg = np.zeros_like(pooled)
            gfx.check(gfx._ffi.gfx_memcpy_d2h(a, dbg.ctypes.data, yd, outb.value))
            assert np.array_equal(dbg, pooled), "debug path must compute the same result"
        for p in (xd, yd, hd):
            gfx.check(gfx._ffi.gfx_device_free(a, p))
    finally:
        gfx._ffi.gfx_arena_destroy(a)
    return x_bits, pooled, again, hidden


def test_bert_base_every_layer_teacher_forced(gfx, olib):
    """Full BERT-base depth (12 layers), 2 sequences x 128 tokens."""
    layers, seqs = 12, 2
    seed = gfx.model_seed("bert-base-c5-test")
    x_bits, pooled, again, hidden = run_gpu(gfx, 70, layers, seqs, seed)
    assert np.array_equal(pooled, again), "inference must be deterministic"
    assert np.array_equal(hidden[0], x_bits)
    threads = os.cpu_count() or 1
    worst = 0.0
    for l in range(layers):
        want = np.zeros_like(hidden[l])
        assert olib.orc_bert_layer(seed, l, D, 12, 3072, SEQ, seqs, hidden[l].ctypes.data, want.ctypes.data,
                                   threads) == 0
        err = rel(bf16_to_f32(hidden[l + 1]), bf16_to_f32(want))
        worst = max(worst, err)
        assert err <= TOL, f"layer {l}: {err:.3e}"
    want_pool = np.zeros((seqs, D), np.float32)
    assert olib.orc_bert_pool(seed, layers, D, SEQ, seqs, hidden[layers].ctypes.data, want_pool.ctypes.data) == 0
    assert rel(pooled, want_pool) <= TOL
    print(f"worst per-layer normwise error {worst:.2e}")


def test_bert_one_layer_end_to_end(gfx, olib):
    seqs = 3
    seed = gfx.model_seed("bert-test-1-3")
    x_bits, pooled, _, _ = run_gpu(gfx, 71, 1, seqs, seed, debug=False)
    want = np.zeros((seqs, D), np.float32)
    assert olib.orc_bert_forward(seed, 1, D, 12, 3072, SEQ, seqs, x_bits.ctypes.data, want.ctypes.data,
                                 os.cpu_count() or 1) == 0
    assert np.isfinite(pooled).all()
    assert rel(pooled, want) <= TOL


def teacher_forced(olib, seed, layers, seqs, hidden, pooled, check_layers=None, d=D, ffn=3072, seq=SEQ, lengths=None):
    threads = os.cpu_count() or 1
    worst = 0.0
    for l in (range(layers) if check_layers is None else check_layers):
        want = np.zeros_like(hidden[l])
        if lengths is None:
            assert olib.orc_bert_layer(seed, l, d, d // 64, ffn, seq, seqs, hidden[l].ctypes.data, want.ctypes.data,
                                       threads) == 0
        else:
            assert olib.orc_bert_layer_masked(seed, l, d, d // 64, ffn, seq, seqs, lengths.ctypes.data,
                                              hidden[l].ctypes.data, want.ctypes.data, threads) == 0
        err = rel(bf16_to_f32(hidden[l + 1]), bf16_to_f32(want))
        worst = max(worst, err)
        assert err <= TOL, f"layer {l}: {err:.3e}"
    want_pool = np.zeros((seqs, d), np.float32)
    assert olib.orc_bert_pool(seed, layers, d, seq, seqs, hidden[layers].ctypes.data, want_pool.ctypes.data) == 0
    assert rel(pooled, want_pool) <= TOL
    return worst


@pytest.mark.parametrize("mode", ["flow", "perop", "pair"])
def test_bert_c5_shape_teacher_forced(gfx, olib, mode):
    """The C5 request: 32 sequences x 128 tokens (T = 4096) through all 12
    layers: the production encoder dataflow kernel K5 ("flow") and the per-op
    launches (single-CTA or 2-SM GEMMs); every layer (flow, perop) or layers
    0, 1, 6, 11 (pair) teacher-forced against the oracle, plus the pooler."""
    layers, seqs = 12, 32
    seed = gfx.model_seed("bert-base-c5-fullshape")
    x_bits, pooled, again, hidden = run_gpu(gfx, 72, layers, seqs, seed, request_id=11, mode=mode)
    assert np.array_equal(pooled, again), "inference must be deterministic"
    assert np.array_equal(hidden[0], x_bits)
    assert np.isfinite(pooled).all()
    worst = teacher_forced(olib, seed, layers, seqs, hidden, pooled, None if mode != "pair" else (0, 1, 6, 11))
    print(f"C5 shape ({mode}): worst per-layer normwise error {worst:.2e}")


@pytest.mark.parametrize("d,ffn,layers,seqs", [(1024, 4096, 2, 32), (1024, 4096, 3, 3), (512, 2048, 3, 5)])
def test_bert_other_widths_teacher_forced(gfx, olib, d, ffn, layers, seqs):
    """Widths beyond BERT-base on the per-op path: BERT-large layers (d 1024, 16
    heads, ffn 4096) at the C5 request shape (32 x 128 tokens: persistent GEMMs
    with 2-3 tiles per CTA, the residual + LayerNorm epilogue in 4-CTA clusters)
    and at 3 sequences, and d 512 (8 heads, 2-CTA clusters); every layer and the
    pooler teacher-forced against the oracle."""
    seed = gfx.model_seed(f"bert-width-{d}-{layers}-{seqs}")
    x_bits, pooled, again, hidden = run_gpu(gfx, 74, layers, seqs, seed, request_id=3, d=d, ffn=ffn)
    assert np.array_equal(pooled, again)
    assert np.array_equal(hidden[0], x_bits)
    worst = teacher_forced(olib, seed, layers, seqs, hidden, pooled, d=d, ffn=ffn)
    print(f"d {d}: worst per-layer normwise error {worst:.2e}")


@pytest.mark.parametrize("seq,seqs,layers,masked,d", [(256, 4, 2, False, D), (384, 2, 2, False, D), (512, 9, 2, False, D),
                                                      (512, 4, 2, True, D), (512, 3, 1, True, 1024)])
def test_bert_longer_sequences_teacher_forced(gfx, olib, seq, seqs, layers, masked, d):
    """Sequences of 256 / 384 / 512 tokens (K3 with every key tile's scores in TMEM:
    exact softmax over up to 512 keys; P over 2-8 swizzled 64-key blocks), padded
    ones (lengths 1 .. seq) included; every layer and the pooler teacher-forced."""
    seed = gfx.model_seed(f"bert-seq-{seq}-{seqs}-{masked}")
    lengths = None
    if masked:
        lengths = np.random.default_rng(seq).integers(1, seq + 1, seqs).astype(np.int32)
        lengths[:2] = [1, seq]
    ffn = 4 * d
    x_bits, pooled, again, hidden = run_gpu(gfx, 77, layers, seqs, seed, request_id=2, seq=seq, lengths=lengths, d=d,
                                            ffn=ffn)
    assert np.array_equal(pooled, again)
    assert np.array_equal(hidden[0], x_bits)
    teacher_forced(olib, seed, layers, seqs, hidden, pooled, seq=seq, lengths=lengths, d=d, ffn=ffn)


def test_bert_large_batch_pooler(gfx, olib):
    """A request of 130 sequences (more [CLS] rows than one pooler block stages:
    pooler blocks of 64 sequences) through one layer; teacher-forced + pooler."""
    seed = gfx.model_seed("bert-batch-130")
    x_bits, pooled, again, hidden = run_gpu(gfx, 75, 1, 130, seed, request_id=9)
    assert np.array_equal(pooled, again)
    teacher_forced(olib, seed, 1, 130, hidden, pooled)


def test_bert_padding_mask_teacher_forced(gfx, olib):
    """Padded sequences (gfx_infer_masked): lengths 1, 64, 65, 127, 128 and random
    ones at the C5 request shape (32 x 128 tokens) through 3 layers; every layer
    teacher-forced against the oracle's masked layer, the pooler too; a bad
    length is refused."""
    seqs, layers = 32, 3
    rng = np.random.default_rng(5)
    lengths = rng.integers(1, 129, seqs).astype(np.int32)
    lengths[:5] = [1, 64, 65, 127, 128]
    seed = gfx.model_seed("bert-masked")
    x_bits, pooled, again, hidden = run_gpu(gfx, 76, layers, seqs, seed, request_id=4, lengths=lengths)
    assert np.array_equal(pooled, again)
    threads = os.cpu_count() or 1
    for l in range(layers):
        want = np.zeros_like(hidden[l])
        assert olib.orc_bert_layer_masked(seed, l, D, 12, 3072, SEQ, seqs, lengths.ctypes.data, hidden[l].ctypes.data,
                                          want.ctypes.data, threads) == 0
        err = rel(bf16_to_f32(hidden[l + 1]), bf16_to_f32(want))
        assert err <= TOL, f"layer {l}: {err:.3e}"
    want_pool = np.zeros((seqs, D), np.float32)
    assert olib.orc_bert_pool(seed, layers, D, SEQ, seqs, hidden[layers].ctypes.data, want_pool.ctypes.data) == 0
    assert rel(pooled, want_pool) <= TOL
    with pytest.raises(gfx.GfxError):
        bad = lengths.copy()
        bad[3] = 0
        run_gpu(gfx, 76, layers, seqs, seed, request_id=4, lengths=bad, debug=False)


@pytest.mark.parametrize("seqs", [1, 3, 37])
def test_bert_flow_ragged_batches(gfx, olib, seqs):
    """K5 at batches that do not fill the 148 SMs (1, 3 row blocks) or leave a
    ragged last wave (37): all layers teacher-forced against the oracle, and
    layer 0's output within tolerance of the per-op launches' (same rounding
    points; only the softmax denominator's summation order differs)."""
    layers = 12 if seqs == 1 else 4
    seed = gfx.model_seed(f"bert-flow-ragged-{seqs}")
    x_bits, pooled, again, hidden = run_gpu(gfx, 73, layers, seqs, seed, request_id=5, mode="flow")
    assert np.array_equal(pooled, again)
    teacher_forced(olib, seed, layers, seqs, hidden, pooled)
    _, _, _, hidden_op = run_gpu(gfx, 73, layers, seqs, seed, request_id=5, mode="perop")
    assert rel(bf16_to_f32(hidden[1]), bf16_to_f32(hidden_op[1])) <= TOL


def bf16_round(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint32) << 16
    return u.view(np.float32)


def bf16_bits(x):
    return (bf16_round(x).view(np.uint32) >> 16).astype(np.uint16)


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("op,tokens", [(0, 4096), (1, 4096), (1, 8192), (2, 4096), (3, 4096), (3, 8192),
                                       (4, 256), (4, 4096), (4, 8192), (5, 4096), (5, 8192)])
def test_bert_gemm_epilogue_parity(gfx, olib, op, tokens, pair):
    """One K2 GEMM with its fused epilogue at T = 4096 / 8192 (the persistent
    CTAs run 1-6 tiles each, cycling both TMEM accumulators) against numpy:
    y = bf16(x . W^T + b [GELU] [+ resid]) with W, b from the parameter stream.
    Ops 4 / 5 add the post-LN LayerNorm (fp64 statistics of the bf16-rounded
    residual sum, as the oracle's layernorm_rows): fused into the GEMM's
    epilogue through the 3-CTA cluster at 256 / 4096 tokens, the residual GEMM
    + layernorm_kernel fallback at 8192 (more row blocks than resident clusters)."""
    from scipy.special import erf
    layer, seqs = 3, tokens // SEQ
    idx = 73
    seed = gfx.model_seed("bert-gemm-epilogues")
    desc = gfx.models.bert_desc(4, seqs, seed)
    gfx.check(gfx._ffi.gfx_model_register(idx, C.byref(desc)))
    pages = C.c_int32()
    gfx.check(gfx._ffi.gfx_model_pages(idx, C.byref(pages)))
    K, N = {0: (D, 3 * D), 1: (D, D), 2: (D, 3072), 3: (3072, D), 4: (D, D), 5: (3072, D)}[op]
    wt, bt = {0: (0, 1), 1: (2, 3), 2: (6, 7), 3: (8, 9), 4: (2, 3), 5: (8, 9)}[op]
    rng = np.random.default_rng(100 + op)
    x = bf16_round(rng.standard_normal((tokens, K)).astype(np.float32))
    r = bf16_round(rng.standard_normal((tokens, N)).astype(np.float32))
    w = np.zeros(N * K, np.float32)
    olib.orc_fill_params(seed, 16 * layer + wt, w.size, np.float32(1.0 / np.sqrt(K)), w.ctypes.data)
    w = bf16_round(w).reshape(N, K)
    b = np.zeros(N, np.float32)
    olib.orc_fill_params(seed, 16 * layer + bt, N, np.float32(0.02), b.ctypes.data)
    v = x.astype(np.float64) @ w.T.astype(np.float64) + b
    if op == 2:
        v = 0.5 * v * (1.0 + erf(v / np.sqrt(2.0)))
    if op in (1, 3, 4, 5):
        v = v + r
    want = bf16_round(v.astype(np.float32))
    if op in (4, 5):
        gt, bet = (4, 5) if op == 4 else (10, 11)
        g = np.zeros(N, np.float32)
        be = np.zeros(N, np.float32)
        olib.orc_fill_params(seed, 16 * layer + gt, N, np.float32(0.1), g.ctypes.data)
        olib.orc_fill_params(seed, 16 * layer + bet, N, np.float32(0.1), be.ctypes.data)
        g = g + np.float32(1.0)
        t1 = want.astype(np.float64)
        mean = t1.mean(axis=1, keepdims=True)
        var = ((t1 - mean) ** 2).mean(axis=1, keepdims=True)
        want = bf16_round(((t1 - mean) / np.sqrt(var + 1e-12) * g + be).astype(np.float32))
    a = C.c_void_p()
    gfx.check(gfx._ffi.gfx_arena_create(0, (pages.value + 2) << 21, C.byref(a)))
    try:
        gfx.check(gfx._ffi.gfx_arena_set_option(a, gfx._ffi.GFX_OPT_GEMM_PAIR, int(pair)))
        gfx.check(gfx._ffi.gfx_load_h2d(a, idx, None))
        xd, rd, yd = C.c_void_p(), C.c_void_p(), C.c_void_p()
        for p, n in ((xd, x.size), (rd, r.size), (yd, r.size)):
            gfx.check(gfx._ffi.gfx_device_alloc(a, 2 * n, C.byref(p)))
        xb, rb = bf16_bits(x), bf16_bits(r)
        gfx.check(gfx._ffi.gfx_memcpy_h2d(a, xd, xb.ctypes.data, xb.nbytes))
        gfx.check(gfx._ffi.gfx_memcpy_h2d(a, rd, rb.ctypes.data, rb.nbytes))
        gfx.check(gfx._ffi.gfx_bert_gemm(a, idx, layer, op, xd, rd, yd, tokens))
        got = np.zeros(tokens * N, np.uint16)
        gfx.check(gfx._ffi.gfx_memcpy_d2h(a, got.ctypes.data, yd, got.nbytes))
        for p in (xd, rd, yd):
            gfx.check(gfx._ffi.gfx_device_free(a, p))
    finally:
        gfx._ffi.gfx_arena_destroy(a)
    got = bf16_to_f32(got).reshape(tokens, N)
    err = rel(got, want)
    flips = float(np.mean(got != want))
    assert err <= TOL, f"op {op} T {tokens}: {err:.3e}"
    assert flips < 0.01, f"op {op}: {flips:.4f} of outputs differ from the bf16-rounded reference"
