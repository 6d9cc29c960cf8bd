"""configs[2] (C3) and configs[3] (C4) on the B200, with the fleet's GPU
managers emulated on the one device (n_devices=1; every manager has its own
paged arena, streams and page tables; a peer fetch is a D2D copy standing in
for NVLink).

  * C3: 8 GPUs x 128 MiB arenas, 20 MLP models of 25-100 MB (1294 MB, more
    than the 1 GiB aggregate cache), working set 20: the schedule is bit-exact
    with the oracle and sampled outputs are within the fp32 tolerance of the
    oracle's forward;
  * C4: Zipf 1.0/1.2 at 2/4/8 GPUs, the same decision stream replayed with
    false misses served by peer fetch vs by pinned-host reload: identical
    decisions, bit-identical outputs, every peer fetch replacing one H2D load.
"""
import numpy as np
import pytest

import simabi
from test_gpu_parity import TOL, olib, oracle_forward, rel  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gfx():
    import paper_2303_05601_b200 as g
    g.register_models(g.load_model_specs("mlp_c3"))
    return g


def _oracle(gfx, cfg_kw):
    return simabi.load_oracle().run(gfx.catalog_text("mlp_c3"), simabi.make_config(**cfg_kw))


@pytest.mark.parametrize("policy", ["lb", "lalbo3"])
def test_c3_fleet_bit_exact_and_outputs(gfx, olib, policy):  # noqa: F811
    G = 8
    cfg = gfx.c3_config(gpus=G, policy=policy)
    rep = gfx.Replay(gfx.catalog_text("mlp_c3"), cfg, n_devices=1, use_p2p=True, keep_outputs=True)
    res = rep.run()
    n = int(res.n_requests)
    out = rep.outputs(n)
    models, _ = rep.request_info(n)
    rep.close()
    o = _oracle(gfx, dict(gpus=G, capacity_mb=gfx.C3_ARENA_MB, policy=policy, working_set=20,
                          rpm=gfx.c3_rpm(G), minutes=6))
    assert int(res.decision_digest) == o.decision_digest
    assert np.array_equal(models, o.model_idx)
    c = o.counts()
    assert (res.hits, res.misses, res.false_misses, res.evictions) == (
        c["hits"], c["misses"], c["false_misses"], c["evictions"])
    assert res.loads_p2p > 0 and res.loads_h2d + res.loads_p2p == res.misses
    specs = gfx.load_model_specs("mlp_c3")
    for rid in np.linspace(0, n - 1, 5).astype(int):
        _, lo, pr = oracle_forward(olib, gfx, specs[int(models[rid])], rid)
        assert rel(out[rid, 0], lo) <= TOL
        assert rel(out[rid, 1], pr) <= TOL


@pytest.mark.parametrize("gpus,zipf", [(2, 1.2), (4, 1.0), (8, 1.2)])
def test_c4_peer_fetch_vs_host_reload(gfx, olib, gpus, zipf):  # noqa: F811
    cfg = gfx.c3_config(gpus=gpus, policy="lalbo3", zipf=zipf)
    got = {}
    for p2p in (True, False):
        rep = gfx.Replay(gfx.catalog_text("mlp_c3"), cfg, n_devices=1, use_p2p=p2p, keep_outputs=True)
        res = rep.run()
        got[p2p] = (res, rep.outputs(int(res.n_requests)), rep.request_info(int(res.n_requests))[0])
        rep.close()
    a, b = got[True][0], got[False][0]
    assert int(a.decision_digest) == int(b.decision_digest)
    assert a.loads_p2p > 0 and b.loads_p2p == 0
    assert a.loads_p2p + a.loads_h2d == b.loads_h2d == a.misses
    assert a.h2d_bytes + a.p2p_bytes == b.h2d_bytes
    assert np.array_equal(got[True][1], got[False][1])
    # ... and the peer-fetch replay's outputs are the oracle's (not only the reload replay's).
    n, models = int(a.n_requests), got[True][2]
    specs = gfx.load_model_specs("mlp_c3")
    for rid in np.linspace(0, n - 1, 4).astype(int):
        _, lo, pr = oracle_forward(olib, gfx, specs[int(models[rid])], rid)
        assert rel(got[True][1][rid, 0], lo) <= TOL
        assert rel(got[True][1][rid, 1], pr) <= TOL
