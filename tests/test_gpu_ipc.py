"""Cross-process NVLink peer fetch (one process per GPU, the bench.py --gpus N
layout) on one B200: two ranks, each executing only its own GPU's decisions,
exchange CUDA IPC blobs of their arenas and flag words over gloo; a false miss
fetches the model out of the holder's arena with device-side ordering
(cuStreamWaitValue32 on the holder's load counter, a write back when the read
is done). On one device the "peer" copy is D2D; the ordering, page-table
shadowing and counters are the same code as across NVLink.

Checks: peer fetches happen on both runs, every request's output is bit-for-
bit the output of the single-process replay (two managers, in-process peer
path) on the same schedule, and sampled outputs of that replay — requests
served after peer fetches included — are within the fp32 tolerance of the
oracle's forward."""
import hashlib
import os
import socket

import numpy as np
import pytest

from test_gpu_parity import TOL, olib, oracle_forward, rel  # noqa: F401

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(gfx):
    return gfx.sim_config(gpus=WORLD, capacity_mb=204.0, policy="lb", minutes=2)


def _digests(outs):
    """Per-request sha1 of the output bytes; None for rows this process did not serve (all zero)."""
    d = []
    for o in outs:
        d.append(None if not o.any() else hashlib.sha1(o.tobytes()).hexdigest())
    return d


def _worker(rank, port, q, distinct_devices=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2303_05601_b200 as gfx
        gfx.register_models(gfx.load_model_specs("mlp_c2"))
        cat = gfx.catalog_text("mlp_c2_paper")
        rep = gfx.Replay(cat, _cfg(gfx), n_devices=1, first_device=rank if distinct_devices else 0, only_gpu=rank,
                         use_p2p=True, keep_outputs=True)
        rep.connect_peers()
        runs = []
        for _ in range(2):  # the second run exercises the cumulative cross-process counters
            res = rep.run()
            n = int(res.n_requests)
            dist.barrier()
            runs.append((int(res.loads_p2p), int(res.loads_h2d), int(res.false_misses),
                         _digests(rep.outputs(n))))
        rep.close()
        q.put((rank, runs))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_cross_process_peer_fetch_matches_single_process(olib):  # noqa: F811
    run_cross_process(distinct_devices=False, olib=olib)


def run_cross_process(distinct_devices, olib=None):
    import torch.multiprocessing as mp

    import paper_2303_05601_b200 as gfx
    gfx.register_models(gfx.load_model_specs("mlp_c2"))
    cat = gfx.catalog_text("mlp_c2_paper")
    ref = gfx.Replay(cat, _cfg(gfx), n_devices=1, use_p2p=True, keep_outputs=True)
    rres = ref.run()
    n = int(rres.n_requests)
    outs = ref.outputs(n)
    want = _digests(outs)
    models, _ = ref.request_info(n)
    ref.close()
    assert rres.loads_p2p > 0
    if olib is not None:
        specs = gfx.load_model_specs("mlp_c2")
        for rid in np.linspace(0, n - 1, 6).astype(int):
            _, lo, pr = oracle_forward(olib, gfx, specs[int(models[rid])], rid)
            assert rel(outs[rid, 0], lo) <= TOL
            assert rel(outs[rid, 1], pr) <= TOL

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, distinct_devices)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for run in range(2):
        p2p = sum(got[r][run][0] for r in range(WORLD))
        assert p2p == rres.loads_p2p, f"run {run}: {p2p} cross-process fetches, single process {rres.loads_p2p}"
        served = [None] * n
        for r in range(WORLD):
            for i, d in enumerate(got[r][run][3]):
                if d is not None:
                    assert served[i] is None, f"request {i} served twice"
                    served[i] = d
        assert served == want, f"run {run}: outputs differ from the single-process replay"
