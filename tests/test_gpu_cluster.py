"""N1 on the B200: one gfx_managerd process per GPU fed by the global cache
manager over shared memory (paper_2303_05601_b200/csrc/capi/cluster.cu).

On one device the GPUs are emulated (every daemon on device 0, peer fetches
cross processes through CUDA IPC as D2D copies); with more devices the same
test places the daemons on distinct devices.

  * run(): the reference's deterministic schedule executed by the daemons —
    decision digest equal to the oracle's, false misses served by cross-process
    peer fetches, outputs within 1e-5 of the oracle and identical run to run;
  * run_live(): live closed-loop serving with one process per GPU (the mode
    that needed every GPU in one process before N1) — every request served once,
    outputs within 1e-5 of the oracle.
"""
import ctypes as C
import os

import numpy as np
import pytest

import simabi

pytestmark = pytest.mark.gpu


def _oracle():
    lib = C.CDLL(simabi.ORACLE_SO)
    lib.orc_mlp_forward.restype = C.c_int
    lib.orc_mlp_forward.argtypes = [C.c_uint64, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_int]
    lib.orc_fill_params.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_float, C.c_void_p]
    return lib


def _check_outputs(gfx, cl, specs, models, rids, olib):
    worst = 0.0
    for rid in rids:
        s = specs[int(models[rid])]
        x = np.zeros((32, s.dims[0]), np.float32)
        olib.orc_fill_params(gfx._ffi.gfx_input_seed(int(rid)), 0xFFFFFFFF, x.size, 1.0, x.ctypes.data)
        dims = (C.c_int32 * len(s.dims))(*s.dims)
        lo = np.zeros((32, s.dims[-1]), np.float32)
        pr = np.zeros_like(lo)
        assert olib.orc_mlp_forward(s.seed, len(s.dims) - 1, C.cast(dims, C.c_void_p), 32, x.ctypes.data,
                                    lo.ctypes.data, pr.ctypes.data, os.cpu_count() or 1) == 0
        got = cl.output(int(rid))
        for g, w in ((got[0], lo), (got[1], pr)):
            worst = max(worst, float(np.linalg.norm(g.astype(np.float64) - w) / np.linalg.norm(w)))
    assert worst <= 1e-5, f"normwise error {worst:.3e}"
    return worst


def _devices(gfx, G):
    n = C.c_int(0)
    gfx.check(gfx._ffi.gfx_device_count(C.byref(n)))
    return [g % n.value for g in range(G)] if n.value >= G else [0] * G


@pytest.mark.parametrize("gpus,policy", [(2, "lalb"), (3, "lalbo3"), (1, "lb")])
def test_cluster_replay_bit_exact_and_outputs(gpus, policy):
    import paper_2303_05601_b200 as gfx
    specs = gfx.load_model_specs("mlp_c2")
    cat = gfx.catalog_text("mlp_c2_paper")
    cfg = gfx.sim_config(gpus=gpus, capacity_mb=204.0, policy=policy, minutes=2)
    cl = gfx.Cluster(cat, cfg, specs, devices=_devices(gfx, gpus))
    try:
        res = cl.run()
        o = simabi.load_oracle().run(cat, simabi.make_config(gpus=gpus, capacity_mb=204.0, policy=policy, minutes=2))
        assert int(res.decision_digest) == o.decision_digest
        n = int(res.n_requests)
        assert n == len(o.arrival) and int(res.hits + res.misses) == n
        if gpus > 1:
            assert res.loads_p2p > 0, "no false miss became a cross-process peer fetch"
        assert res.loads_h2d + res.loads_p2p == res.misses
        rids = np.linspace(0, n - 1, 10).astype(int)
        olib = _oracle()
        _check_outputs(gfx, cl, specs, o.model_idx, rids, olib)
        first = [cl.output(int(r)) for r in rids]
        res2 = cl.run()  # second run: cumulative cross-process counters, arenas reset
        assert int(res2.decision_digest) == o.decision_digest and res2.loads_p2p == res.loads_p2p
        for r, f in zip(rids, first):
            assert np.array_equal(cl.output(int(r)), f), "outputs differ between runs"
    finally:
        cl.close()


def test_cluster_live_one_process_per_gpu():
    import paper_2303_05601_b200 as gfx
    specs = gfx.load_model_specs("mlp_c2")
    cat = gfx.catalog_text("mlp_c2_paper")
    cfg = gfx.sim_config(gpus=3, capacity_mb=204.0, policy="lalbo3", minutes=1)
    cl = gfx.Cluster(cat, cfg, specs, devices=_devices(gfx, 3))
    try:
        base = cl.run()
        n = int(base.n_requests)
        scale = 60.0 / max(2 * base.device_ms / 1e3, 1e-3)
        live = cl.run_live(scale, 0.3)
        assert int(live.n_requests) == n and int(live.hits + live.misses) == n
        assert 0 < live.sim_p50_s <= live.sim_p99_s
        o = simabi.load_oracle().run(cat, simabi.make_config(gpus=3, capacity_mb=204.0, policy="lalbo3", minutes=1))
        served = [cl.request_gpu(r) for r in range(n)]
        assert min(served) >= 0 and len(set(served)) > 1
        _check_outputs(gfx, cl, specs, o.model_idx, np.linspace(0, n - 1, 12).astype(int), _oracle())
    finally:
        cl.close()
