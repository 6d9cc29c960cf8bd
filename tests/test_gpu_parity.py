"""GPU parity tests (B200): the product path through the C-ABI against the oracle.

  * schedule: the replay's decision stream is bit-exact with the oracle's
    (same canonical digest, same per-request model assignment);
  * numerics: every checked inference output (logits and softmax) is within the
    north-star fp32 tolerance of the oracle's fp64-accumulated restatement:
    normwise relative error <= 1e-5;
  * cache data plane: H2D loads, evictions, page reuse, emulated NVLink peer
    fetches (two GPU managers on one device) and host-I/O replays all yield the
    same outputs; split-K reductions are deterministic run to run.
"""
import ctypes as C
import os

import numpy as np
import pytest

import simabi

pytestmark = pytest.mark.gpu

TOL = 1e-5  # north star: 1e-5 relative for fp32 (normwise, SURVEY.md §7 hard part 5)


@pytest.fixture(scope="module")
def gfx():
    import paper_2303_05601_b200 as g
    n = C.c_int(0)
    g.check(g._ffi.gfx_device_count(C.byref(n)))
    assert n.value >= 1, "no CUDA device: the B200 path has no CPU fallback"
    g.register_models(g.load_model_specs("mlp_c2"))
    return g


@pytest.fixture(scope="module")
def olib():
    lib = C.CDLL(simabi.ORACLE_SO)
    lib.orc_mlp_forward.restype = C.c_int
    lib.orc_mlp_forward.argtypes = [C.c_uint64, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_int]
    lib.orc_fill_params.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_float, C.c_void_p]
    return lib


def oracle_forward(olib, gfx, spec, rid):
    x = np.zeros((32, spec.dims[0]), np.float32)
    olib.orc_fill_params(gfx._ffi.gfx_input_seed(int(rid)), 0xFFFFFFFF, x.size, 1.0, x.ctypes.data)
    dims = (C.c_int32 * len(spec.dims))(*spec.dims)
    lo = np.zeros((32, spec.dims[-1]), np.float32)
    pr = np.zeros_like(lo)
    assert olib.orc_mlp_forward(spec.seed, len(spec.dims) - 1, C.cast(dims, C.c_void_p), 32, x.ctypes.data,
                                lo.ctypes.data, pr.ctypes.data, os.cpu_count() or 1) == 0
    return x, lo, pr


def rel(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b.astype(np.float64)))


@pytest.mark.parametrize("catalog,policy,gpus", [("mlp_c2", "lalbo3", 1), ("mlp_c2", "lb", 1),
                                                 ("mlp_c2_paper", "lalbo3", 1), ("mlp_c2_paper", "lb", 1),
                                                 ("mlp_c2_paper", "lalb", 3)])
def test_replay_schedule_bit_exact(gfx, catalog, policy, gpus):
    cat = gfx.catalog_text(catalog)
    cfg = gfx.sim_config(gpus=gpus, capacity_mb=204.0, policy=policy, minutes=2)
    rep = gfx.Replay(cat, cfg, n_devices=1)
    res = rep.run()
    models, _ = rep.request_info(int(res.n_requests))
    rep.close()
    o = simabi.load_oracle().run(cat, simabi.make_config(gpus=gpus, capacity_mb=204.0, policy=policy, minutes=2))
    assert int(res.decision_digest) == o.decision_digest
    assert np.array_equal(models, o.model_idx)
    c = o.counts()
    assert (res.hits, res.misses, res.false_misses, res.local_enqueues, res.evictions) == (
        c["hits"], c["misses"], c["false_misses"], c["local_enqueues"], c["evictions"])
    assert res.loads_h2d + res.loads_p2p == res.misses


def test_replay_rejects_models_registered_out_of_catalog_order(gfx):
    """Catalog row i must be the model registered at index i: a store holding
    another model there is refused at replay creation (domain error), instead
    of silently serving the wrong weights under the catalog's id."""
    specs = gfx.load_model_specs("mlp_c2")
    try:
        gfx.register_models(list(reversed(specs)))
        with pytest.raises(gfx._ffi.GfxError, match="not catalog row"):
            gfx.Replay(gfx.catalog_text("mlp_c2"), gfx.sim_config(gpus=1, capacity_mb=204.0, minutes=1))
    finally:
        gfx.register_models(specs)


def test_replay_outputs_match_oracle(gfx, olib):
    cat = gfx.catalog_text("mlp_c2")
    specs = gfx.load_model_specs("mlp_c2")
    rep = gfx.Replay(cat, gfx.sim_config(minutes=1), keep_outputs=True)
    res = rep.run()
    n = int(res.n_requests)
    out = rep.outputs(n)
    models, _ = rep.request_info(n)
    rep.close()
    for rid in np.linspace(0, n - 1, 6).astype(int):
        _, lo, pr = oracle_forward(olib, gfx, specs[int(models[rid])], rid)
        assert rel(out[rid, 0], lo) <= TOL
        assert rel(out[rid, 1], pr) <= TOL
        assert np.allclose(out[rid, 1].sum(axis=1), 1.0, atol=1e-5)


def test_every_model_shape(gfx, olib):
    """All 22 catalog models (hidden widths 1600..3136, the 1000-class tail tile)."""
    specs = gfx.load_model_specs("mlp_c2")
    a = C.c_void_p()
    gfx.check(gfx._ffi.gfx_arena_create(0, 204 << 20, C.byref(a)))
    try:
        x = C.c_void_p()
        y = C.c_void_p()
        gfx.check(gfx._ffi.gfx_device_alloc(a, 32 * 1024 * 4, C.byref(x)))
        gfx.check(gfx._ffi.gfx_device_alloc(a, 2 * 32 * 1000 * 4, C.byref(y)))
        for i, s in enumerate(specs):
            gfx.check(gfx._ffi.gfx_load_h2d(a, i, None))
            gfx.check(gfx._ffi.gfx_fill_params(a, x, 32 * 1024, gfx._ffi.gfx_input_seed(1000 + i), 0xFFFFFFFF, 1.0))
            gfx.check(gfx._ffi.gfx_infer(a, i, x, y, 32, None))
            got = np.zeros((2, 32, 1000), np.float32)
            gfx.check(gfx._ffi.gfx_memcpy_d2h(a, got.ctypes.data, y, got.nbytes))
            _, lo, pr = oracle_forward(olib, gfx, s, 1000 + i)
            assert rel(got[0], lo) <= TOL, s.model_id
            assert rel(got[1], pr) <= TOL, s.model_id
            gfx.check(gfx._ffi.gfx_evict(a, i))
        free = C.c_int32()
        gfx.check(gfx._ffi.gfx_arena_free_pages(a, C.byref(free)))
        assert free.value == 102
        gfx.check(gfx._ffi.gfx_device_free(a, x))
        gfx.check(gfx._ffi.gfx_device_free(a, y))
    finally:
        gfx._ffi.gfx_arena_destroy(a)


def test_cache_ops_errors_and_page_accounting(gfx):
    a = C.c_void_p()
    pages21 = gfx.load_model_specs("mlp_c2")[21].pages  # vgg19, the largest model
    gfx.check(gfx._ffi.gfx_arena_create(0, pages21 << 21, C.byref(a)))  # exactly its pages
    try:
        free = C.c_int32()
        gfx.check(gfx._ffi.gfx_load_h2d(a, 21, None))
        gfx.check(gfx._ffi.gfx_arena_free_pages(a, C.byref(free)))
        assert free.value == 0
        rc = gfx._ffi.gfx_load_h2d(a, 0, None)  # no room: the control plane would have evicted
        assert rc == 2 and b"out of pages" in gfx._ffi.gfx_last_error()
        assert gfx._ffi.gfx_infer(a, 0, None, None, 32, None) == 2  # not resident
        assert gfx._ffi.gfx_evict(a, 3) == 2
        gfx.check(gfx._ffi.gfx_evict(a, 21))
        gfx.check(gfx._ffi.gfx_arena_free_pages(a, C.byref(free)))
        assert free.value == pages21
        ev = C.c_void_p()
        gfx.check(gfx._ffi.gfx_load_h2d(a, 0, C.byref(ev)))
        gfx.check(gfx._ffi.gfx_event_sync(ev))
        assert gfx._ffi.gfx_event_query(ev) == 0
        gfx.check(gfx._ffi.gfx_event_release(ev))
        res = C.c_int32()
        gfx.check(gfx._ffi.gfx_arena_resident(a, 0, C.byref(res)))
        assert res.value == 1
        assert gfx._ffi.gfx_arena_create(0, (2 << 20) + 1, C.byref(C.c_void_p())) == 1
    finally:
        gfx._ffi.gfx_arena_destroy(a)


def test_peer_fetch_emulated_and_deterministic(gfx, olib):
    """Two GPU managers on one device: false misses fetch from the peer arena
    (the NVLink path's logic; on one device it is a D2D copy). Outputs equal a
    replay without P2P bit for bit, and repeated runs are bit-identical."""
    cat = gfx.catalog_text("mlp_c2_paper")
    cfg = gfx.sim_config(gpus=2, capacity_mb=204.0, policy="lb", minutes=2)
    outs = []
    for p2p in (True, False, True):
        rep = gfx.Replay(cat, cfg, n_devices=1, use_p2p=p2p, keep_outputs=True)
        res = rep.run()
        if p2p:
            assert res.loads_p2p > 0 and res.loads_p2p <= res.false_misses
        else:
            assert res.loads_p2p == 0
        outs.append(rep.outputs(int(res.n_requests)))
        rep.close()
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], outs[2])


def test_host_io_replay_equals_device_resident(gfx):
    cat = gfx.catalog_text("mlp_c2")
    cfg = gfx.sim_config(minutes=1)
    rep = gfx.Replay(cat, cfg, keep_outputs=True)
    r1 = rep.run()
    n = int(r1.n_requests)
    dev_out = rep.outputs(n)
    rep.close()
    hin = np.zeros((n, 32 * 1024), np.float32)
    for i in range(n):
        gfx.check(gfx._ffi.gfx_host_fill_params(hin[i].ctypes.data, hin.shape[1], gfx._ffi.gfx_input_seed(i),
                                                0xFFFFFFFF, 1.0))
    hout = np.zeros((n, 2 * 32 * 1000), np.float32)
    rep = gfx.Replay(cat, cfg, host_io=True, host_inputs=hin, host_outputs=hout)
    r2 = rep.run()
    rep.close()
    assert r2.io_h2d_bytes == n * 32 * 1024 * 4 and r2.io_d2h_bytes == n * 2 * 32 * 1000 * 4
    assert np.array_equal(hout.reshape(dev_out.shape), dev_out)


@pytest.mark.parametrize("policy,gpus", [("lb", 3), ("lalbo3", 3), ("lalbo3", 1)])
def test_pipelined_replay(gfx, policy, gpus):
    """Pipelined-GPU extension on the device: the replay follows the oracle's
    pipelined schedule bit for bit (staged loads overlap the running inference
    on the copy stream), and every request's output equals the reference-mode
    replay's output for that request."""
    cat = gfx.catalog_text("mlp_c2_paper")
    outs, digests = {}, {}
    for pipe in (False, True):
        cfg = gfx.sim_config(gpus=gpus, capacity_mb=204.0, policy=policy, minutes=2, pipeline=pipe)
        rep = gfx.Replay(cat, cfg, n_devices=1, use_p2p=gpus > 1, keep_outputs=True)
        res = rep.run()
        outs[pipe] = rep.outputs(int(res.n_requests))
        digests[pipe] = int(res.decision_digest)
        rep.close()
    o = simabi.load_oracle().run(cat, simabi.make_config(gpus=gpus, capacity_mb=204.0, policy=policy, minutes=2,
                                                         pipeline=True))
    assert digests[True] == o.decision_digest
    assert np.array_equal(outs[True], outs[False])


@pytest.mark.parametrize("dims", [
    [1024, 1000],                      # one layer: no hidden activations, no dataflow boundary
    [32, 4],                           # smallest legal layer
    [1024, 64, 1000],                  # one-tile hidden layer, maximum split-K
    [96, 160, 352, 100],               # widths that are not multiples of 64 / 128
    [256] * 16 + [1000],               # the maximum of 16 layers
    [8192, 8192, 1000],                # the maximum width (282 MiB of weights)
    [1024, 8192, 8192, 8192, 1000],    # 604 MB, 289 arena pages (beyond round 1's 192-page table)
], ids=["L1", "min", "h64", "odd", "L16", "w8192", "p289"])
def test_mlp_edge_shapes(gfx, olib, dims):
    """Edge shapes of the one-launch forward against the oracle's fp64 forward."""
    import ctypes as C
    spec = gfx.ModelSpec("edge-" + "x".join(map(str, dims)), "mlp", dims, 0, 0)
    idx = 50
    gfx.check(gfx._ffi.gfx_model_register(idx, C.byref(spec.desc())))
    pages = C.c_int32()
    gfx.check(gfx._ffi.gfx_model_pages(idx, C.byref(pages)))
    a = C.c_void_p()
    gfx.check(gfx._ffi.gfx_arena_create(0, C.c_uint64((pages.value + 2) << 21), C.byref(a)))
    try:
        x, y = C.c_void_p(), C.c_void_p()
        gfx.check(gfx._ffi.gfx_device_alloc(a, 32 * dims[0] * 4, C.byref(x)))
        gfx.check(gfx._ffi.gfx_device_alloc(a, 2 * 32 * dims[-1] * 4, C.byref(y)))
        gfx.check(gfx._ffi.gfx_load_h2d(a, idx, None))
        rid = 7000 + len(dims)
        gfx.check(gfx._ffi.gfx_fill_params(a, x, 32 * dims[0], gfx._ffi.gfx_input_seed(rid), 0xFFFFFFFF, 1.0))
        for _ in range(2):  # the second launch runs on the other counter bank
            gfx.check(gfx._ffi.gfx_infer(a, idx, x, y, 32, None))
            got = np.zeros((2, 32, dims[-1]), np.float32)
            gfx.check(gfx._ffi.gfx_memcpy_d2h(a, got.ctypes.data, y, got.nbytes))
            _, lo, pr = oracle_forward(olib, gfx, spec, rid)
            assert rel(got[0], lo) <= TOL
            assert rel(got[1], pr) <= TOL
        gfx.check(gfx._ffi.gfx_evict(a, idx))
        gfx.check(gfx._ffi.gfx_device_free(a, x))
        gfx.check(gfx._ffi.gfx_device_free(a, y))
    finally:
        gfx._ffi.gfx_arena_destroy(a)


def test_mlp_random_shapes(gfx, olib):
    """Twelve seeded random MLPs (1-6 layers, widths 32-4096 in steps of 32, any
    number of classes divisible by 4): every tile / split / boundary pattern the
    one-launch forward derives from them matches the oracle's fp64 forward."""
    import ctypes as C
    rng = np.random.default_rng(2303)
    for case in range(12):
        L = int(rng.integers(1, 7))
        dims = [int(rng.integers(1, 129)) * 32 for _ in range(L)] + [int(rng.integers(1, 513)) * 4]
        spec = gfx.ModelSpec(f"rand-{case}-" + "x".join(map(str, dims)), "mlp", dims, 0, 0)
        idx = 51
        gfx.check(gfx._ffi.gfx_model_register(idx, C.byref(spec.desc())))
        pages = C.c_int32()
        gfx.check(gfx._ffi.gfx_model_pages(idx, C.byref(pages)))
        a = C.c_void_p()
        gfx.check(gfx._ffi.gfx_arena_create(0, C.c_uint64((pages.value + 2) << 21), C.byref(a)))
        try:
            x, y = C.c_void_p(), C.c_void_p()
            gfx.check(gfx._ffi.gfx_device_alloc(a, 32 * dims[0] * 4, C.byref(x)))
            gfx.check(gfx._ffi.gfx_device_alloc(a, 2 * 32 * dims[-1] * 4, C.byref(y)))
            gfx.check(gfx._ffi.gfx_load_h2d(a, idx, None))
            rid = 9000 + case
            gfx.check(gfx._ffi.gfx_fill_params(a, x, 32 * dims[0], gfx._ffi.gfx_input_seed(rid), 0xFFFFFFFF, 1.0))
            gfx.check(gfx._ffi.gfx_infer(a, idx, x, y, 32, None))
            got = np.zeros((2, 32, dims[-1]), np.float32)
            gfx.check(gfx._ffi.gfx_memcpy_d2h(a, got.ctypes.data, y, got.nbytes))
            _, lo, pr = oracle_forward(olib, gfx, spec, rid)
            assert rel(got[0], lo) <= TOL, dims
            assert rel(got[1], pr) <= TOL, dims
        finally:
            gfx._ffi.gfx_arena_destroy(a)
