"""Pin the inference oracle (oracle/infer_oracle.c) to third-party implementations.

The reference has no inference code (its inference is the profiled constant
infer_time_us, proj/src/cluster.cpp:161,167), so the oracle's model definitions
cannot be pinned to the reference. They are pinned here to the standard
implementations instead, on CPU, with the oracle's own parameters:

  * C2/C3 MLP: torch fp64 ``nn.Linear`` + ReLU + softmax. The
    oracle accumulates in fp64 and rounds each layer output to fp32, so the two
    agree to fp32 resolution.
  * C5 BERT-base encoder layer and pooler: Hugging Face ``transformers``
    ``BertLayer`` (post-LN, erf GELU, 1/sqrt(d_head) scaling, eps 1e-12) and
    ``BertPooler`` (tanh on the [CLS] token) in fp64 with the oracle's weights.
    The oracle rounds every stored activation to bf16 (the product's rounding
    points) and HF does not, so the tolerance covers bf16 rounding noise (a
    normwise 3e-3) while a structural difference (pre-LN, a missing residual,
    the wrong softmax scale, head split) lands far outside it — checked by the
    negative control below. (The tanh GELU approximation is NOT separable from
    erf at bf16 resolution; the product's GELU is checked against erf directly
    in tests/test_gpu_bert.py's per-epilogue parity.)
Test infrastructure only: nothing here is on the product path.
"""
import ctypes as C

import numpy as np
import pytest

import simabi

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")


@pytest.fixture(scope="module")
def olib():
    lib = C.CDLL(simabi.ORACLE_SO)
    lib.orc_fill_params.restype = None
    lib.orc_fill_params.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_float, C.c_void_p]
    lib.orc_mlp_forward.restype = C.c_int
    lib.orc_mlp_forward.argtypes = [C.c_uint64, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_int]
    lib.orc_bert_layer.restype = C.c_int
    lib.orc_bert_layer.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_int]
    lib.orc_bert_layer_masked.restype = C.c_int
    lib.orc_bert_layer_masked.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
    lib.orc_bert_pool.restype = C.c_int
    lib.orc_bert_pool.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    return lib


def params(olib, seed, tensor, n, scale):
    out = np.zeros(n, np.float32)
    olib.orc_fill_params(seed, tensor, n, np.float32(scale), out.ctypes.data)
    return out


def bf16_round(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint32) << 16
    return u.view(np.float32)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("dims", [(1024, 1344, 1344, 1344, 1000), (64, 96, 10), (300, 17, 33, 5)])
def test_mlp_oracle_matches_torch_linear(olib, dims):
    """The oracle's MLP = torch fp64 Linear/ReLU stack + softmax (parameters from
    the shared parameter stream: tensor 2l = W_l [N x K], 2l + 1 = b_l, scale 1/sqrt(K))."""
    seed, batch = 0x5EED0000 + len(dims), 32
    x = params(olib, 0xC0FFEE0000000000 + 3, 0xFFFFFFFF, batch * dims[0], 1.0).reshape(batch, dims[0])
    nl = len(dims) - 1
    d32 = np.asarray(dims, np.int32)
    logits = np.zeros((batch, dims[-1]), np.float32)
    probs = np.zeros_like(logits)
    assert olib.orc_mlp_forward(seed, nl, d32.ctypes.data, batch, x.ctypes.data, logits.ctypes.data,
                                probs.ctypes.data, 4) == 0
    layers = []
    for l in range(nl):
        K, N = dims[l], dims[l + 1]
        lin = torch.nn.Linear(K, N, dtype=torch.float64)
        with torch.no_grad():
            lin.weight.copy_(torch.from_numpy(params(olib, seed, 2 * l, N * K, 1.0 / np.sqrt(K)).reshape(N, K)))
            lin.bias.copy_(torch.from_numpy(params(olib, seed, 2 * l + 1, N, 1.0 / np.sqrt(K))))
        layers.append(lin)
        if l + 1 < nl:
            layers.append(torch.nn.ReLU())
    with torch.no_grad():
        want = torch.nn.Sequential(*layers)(torch.from_numpy(x).double())
        want_p = torch.softmax(want, dim=-1)
    assert rel(logits, want.numpy()) < 1e-6
    assert rel(probs, want_p.numpy()) < 1e-6


D, HEADS, FFN, SEQ = 768, 12, 3072, 128


def hf_bert_layer(olib, seed, l):
    """transformers.BertLayer in fp64 carrying the oracle's layer-l parameters
    (tensor ids 16 l + {0 Wqkv, 1 bqkv, 2 Wo, 3 bo, 4 ln1_g, 5 ln1_b, 6 W1, 7 b1,
    8 W2, 9 b2, 10 ln2_g, 11 ln2_b}; matrices bf16-rounded, LN gammas 1 + 0.1 u)."""
    from transformers.models.bert.modeling_bert import BertLayer
    cfg = transformers.BertConfig(hidden_size=D, num_attention_heads=HEADS, intermediate_size=FFN,
                                  hidden_act="gelu", layer_norm_eps=1e-12, hidden_dropout_prob=0.0,
                                  attention_probs_dropout_prob=0.0)
    cfg._attn_implementation = "eager"
    layer = BertLayer(cfg).double().eval()
    t0 = 16 * l

    def mat(t, n, k):
        return torch.from_numpy(bf16_round(params(olib, seed, t0 + t, n * k, 1.0 / np.sqrt(k))).reshape(n, k)).double()

    def vec(t, n, scale, shift=0.0):
        return torch.from_numpy(params(olib, seed, t0 + t, n, scale) + np.float32(shift)).double()

    wqkv, bqkv = mat(0, 3 * D, D), vec(1, 3 * D, 0.02)
    sa, ao = layer.attention.self, layer.attention.output
    with torch.no_grad():
        for i, lin in enumerate((sa.query, sa.key, sa.value)):
            lin.weight.copy_(wqkv[i * D:(i + 1) * D])
            lin.bias.copy_(bqkv[i * D:(i + 1) * D])
        ao.dense.weight.copy_(mat(2, D, D))
        ao.dense.bias.copy_(vec(3, D, 0.02))
        ao.LayerNorm.weight.copy_(vec(4, D, 0.1, 1.0))
        ao.LayerNorm.bias.copy_(vec(5, D, 0.1))
        layer.intermediate.dense.weight.copy_(mat(6, FFN, D))
        layer.intermediate.dense.bias.copy_(vec(7, FFN, 0.02))
        layer.output.dense.weight.copy_(mat(8, D, FFN))
        layer.output.dense.bias.copy_(vec(9, D, 0.02))
        layer.output.LayerNorm.weight.copy_(vec(10, D, 0.1, 1.0))
        layer.output.LayerNorm.bias.copy_(vec(11, D, 0.1))
    return layer


def bert_input(olib, seqs):
    # The product's request input (tensor 0xFFFFFFFF of seed 0xC0FFEE.. + request), bf16.
    x = bf16_round(params(olib, 0xC0FFEE0000000000 + 11, 0xFFFFFFFF, seqs * SEQ * D, 1.0))
    return x, (x.view(np.uint32) >> 16).astype(np.uint16)


def test_bert_layer_oracle_matches_transformers(olib):
    seed, seqs, l = 0xB0B0 + 7, 2, 3
    x, xb = bert_input(olib, seqs)
    got = np.zeros_like(xb)
    assert olib.orc_bert_layer(seed, l, D, HEADS, FFN, SEQ, seqs, xb.ctypes.data, got.ctypes.data, 8) == 0
    got_f = (got.astype(np.uint32) << 16).view(np.float32)
    layer = hf_bert_layer(olib, seed, l)
    with torch.no_grad():
        want = layer(torch.from_numpy(x).double().reshape(seqs, SEQ, D))
        want = (want[0] if isinstance(want, tuple) else want).reshape(-1).numpy()
    err = rel(got_f, want)
    assert err < 5e-3, err  # the oracle's bf16 rounding points (measured 3.2e-3)
    # Negative control: the same layer without the 1/sqrt(d_head) score scaling is a
    # different model and lands ~10x outside the tolerance, so the bound can tell.
    layer.attention.self.scaling = 1.0
    with torch.no_grad():
        other = layer(torch.from_numpy(x).double().reshape(seqs, SEQ, D))
        other = (other[0] if isinstance(other, tuple) else other).reshape(-1).numpy()
    assert rel(got_f, other) > 5 * 5e-3


def test_bert_masked_layer_oracle_matches_transformers(olib):
    """Padding mask: the oracle's masked layer (keys j >= lengths[s] excluded) =
    transformers BertLayer with the additive -inf attention mask; query rows past
    a sequence's length are computed too (and compared)."""
    seed, seqs, l = 0xB0B0 + 21, 3, 1
    lengths = np.array([1, 77, 128], np.int32)
    x, xb = bert_input(olib, seqs)
    got = np.zeros_like(xb)
    assert olib.orc_bert_layer_masked(seed, l, D, HEADS, FFN, SEQ, seqs, lengths.ctypes.data, xb.ctypes.data,
                                      got.ctypes.data, 8) == 0
    got_f = (got.astype(np.uint32) << 16).view(np.float32)
    mask = torch.zeros(seqs, 1, 1, SEQ, dtype=torch.float64)
    for s_, n in enumerate(lengths):
        mask[s_, :, :, n:] = float("-inf")
    layer = hf_bert_layer(olib, seed, l)
    with torch.no_grad():
        want = layer(torch.from_numpy(x).double().reshape(seqs, SEQ, D), attention_mask=mask)
        want = (want[0] if isinstance(want, tuple) else want).reshape(-1).numpy()
        unmasked = layer(torch.from_numpy(x).double().reshape(seqs, SEQ, D))
        unmasked = (unmasked[0] if isinstance(unmasked, tuple) else unmasked).reshape(-1).numpy()
    assert rel(got_f, want) < 5e-3
    assert rel(got_f, unmasked) > 5 * 5e-3  # the mask matters at these lengths
    bad = np.array([0, 5, 5], np.int32)
    assert olib.orc_bert_layer_masked(seed, l, D, HEADS, FFN, SEQ, seqs, bad.ctypes.data, xb.ctypes.data,
                                      got.ctypes.data, 8) == -1


def test_bert_masked_layer_full_lengths_equals_unmasked(olib):
    """Consistency of the oracle's two entry points: lengths = seq everywhere is the
    unmasked layer, bit for bit."""
    seed, seqs, l = 0xB0B0 + 23, 2, 0
    x, xb = bert_input(olib, seqs)
    a = np.zeros_like(xb)
    b = np.zeros_like(xb)
    assert olib.orc_bert_layer(seed, l, D, HEADS, FFN, SEQ, seqs, xb.ctypes.data, a.ctypes.data, 8) == 0
    full = np.full(seqs, SEQ, np.int32)
    assert olib.orc_bert_layer_masked(seed, l, D, HEADS, FFN, SEQ, seqs, full.ctypes.data, xb.ctypes.data,
                                      b.ctypes.data, 8) == 0
    assert np.array_equal(a, b)


def test_bert_pooler_oracle_matches_transformers(olib):
    from transformers.models.bert.modeling_bert import BertPooler
    seed, seqs, L = 0xB0B0 + 9, 3, 12
    x, xb = bert_input(olib, seqs)
    got = np.zeros((seqs, D), np.float32)
    assert olib.orc_bert_pool(seed, L, D, SEQ, seqs, xb.ctypes.data, got.ctypes.data) == 0
    cfg = transformers.BertConfig(hidden_size=D)
    pool = BertPooler(cfg).double().eval()
    tp = 16 * L
    with torch.no_grad():
        pool.dense.weight.copy_(torch.from_numpy(bf16_round(params(olib, seed, tp, D * D, 1.0 / np.sqrt(D))).reshape(D, D)))
        pool.dense.bias.copy_(torch.from_numpy(params(olib, seed, tp + 1, D, 0.02)))
        want = pool(torch.from_numpy(x).double().reshape(seqs, SEQ, D)).numpy()
    assert rel(got, want) < 1e-6
