"""Live closed-loop serving on the B200 (extension): the
trace's arrivals are released in real time, each GPU's completion is observed
on the device and fed back to the scheduler. The schedule then follows the
device, so decisions are not bit-exact with the replay; what must hold is that
every request is served once and its output is bit-for-bit the output the
deterministic replay produced for it (an output depends only on the model and
the request's input, never on the schedule, the cache state or the load path),
and a sample of live outputs is checked against the oracle's fp64 forward
directly (north-star fp32 tolerance 1e-5, normwise).
"""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _digests(outs):
    return [hashlib.sha1(o.tobytes()).hexdigest() for o in outs]


@pytest.mark.parametrize("gpus,policy,ema,pipe", [(1, "lalbo3", 0.0, False), (3, "lb", 0.0, False),
                                                   (3, "lalbo3", 0.0, False), (3, "lalbo3", 0.3, False),
                                                   (3, "lalbo3", 0.3, True), (1, "lb", 0.0, True)])
def test_live_outputs_match_replay(gpus, policy, ema, pipe):
    import paper_2303_05601_b200 as gfx
    gfx.register_models(gfx.load_model_specs("mlp_c2"))
    cat = gfx.catalog_text("mlp_c2_paper")
    cfg = gfx.sim_config(gpus=gpus, capacity_mb=204.0, policy=policy, minutes=1, pipeline=pipe)
    rep = gfx.Replay(cat, cfg, n_devices=1, use_p2p=gpus > 1, keep_outputs=True)
    base = rep.run()
    n = int(base.n_requests)
    want = _digests(rep.outputs(n))
    span_s = 60.0
    # Compress one minute of arrivals into ~2x the replay's device time: queues form but drain.
    scale = span_s / max(2 * base.device_ms / 1e3, 1e-3)
    for _ in range(2):
        live = rep.run_live(scale, ema)
        assert int(live.n_requests) == n
        assert int(live.hits + live.misses) == n
        got = _digests(rep.outputs(n))
        assert got == want, "live outputs differ from the deterministic replay"
        assert live.sim_p50_s > 0 and live.sim_p99_s >= live.sim_p50_s
    rep.close()


def test_live_outputs_match_oracle():
    """Live-mode outputs against the oracle itself (not only the product's replay)."""
    import ctypes as C
    import os

    import paper_2303_05601_b200 as gfx
    import simabi
    specs = gfx.load_model_specs("mlp_c2")
    gfx.register_models(specs)
    olib = C.CDLL(simabi.ORACLE_SO)
    olib.orc_mlp_forward.restype = C.c_int
    olib.orc_mlp_forward.argtypes = [C.c_uint64, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_int]
    olib.orc_fill_params.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_float, C.c_void_p]
    cat = gfx.catalog_text("mlp_c2_paper")
    rep = gfx.Replay(cat, gfx.sim_config(gpus=3, capacity_mb=204.0, policy="lalbo3", minutes=1), n_devices=1,
                     use_p2p=True, keep_outputs=True)
    base = rep.run()
    n = int(base.n_requests)
    live = rep.run_live(60.0 / max(2 * base.device_ms / 1e3, 1e-3), 0.3)
    assert int(live.n_requests) == n
    outs = rep.outputs(n)
    models, _ = rep.request_info(n)
    rep.close()
    worst = 0.0
    for rid in np.linspace(0, n - 1, 12).astype(int):
        s = specs[int(models[rid])]
        x = np.zeros((32, s.dims[0]), np.float32)
        olib.orc_fill_params(gfx._ffi.gfx_input_seed(int(rid)), 0xFFFFFFFF, x.size, 1.0, x.ctypes.data)
        dims = (C.c_int32 * len(s.dims))(*s.dims)
        lo = np.zeros((32, s.dims[-1]), np.float32)
        pr = np.zeros_like(lo)
        assert olib.orc_mlp_forward(s.seed, len(s.dims) - 1, C.cast(dims, C.c_void_p), 32, x.ctypes.data,
                                    lo.ctypes.data, pr.ctypes.data, os.cpu_count() or 1) == 0
        for got, want in ((outs[rid, 0], lo), (outs[rid, 1], pr)):
            err = float(np.linalg.norm(got.astype(np.float64) - want) / np.linalg.norm(want))
            worst = max(worst, err)
    assert worst <= 1e-5, f"live output normwise error {worst:.3e}"


def test_live_mode_rejects_bad_args():
    import paper_2303_05601_b200 as gfx
    gfx.register_models(gfx.load_model_specs("mlp_c2"))
    cat = gfx.catalog_text("mlp_c2_paper")
    rep = gfx.Replay(cat, gfx.sim_config(gpus=1, capacity_mb=204.0, policy="lb", minutes=1))
    with pytest.raises(Exception, match="time_scale"):
        rep.run_live(0.0)
    rep.close()
