"""The C-ABI boundary: the product library loads on a CPU-only host and exports
every entry point include/gpufaas_b200.h declares (no compute calls here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

import simabi

HDR = os.path.join(simabi.ROOT, "include", "gpufaas_b200.h")


def declared_functions():
    text = open(HDR).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s+\**\s*(gfx_[a-z0-9_]+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_cache_and_replay_surface():
    names = declared_functions()
    for n in ("gfx_arena_create", "gfx_load_h2d", "gfx_fetch_p2p", "gfx_evict", "gfx_infer", "gfx_event_query",
              "gfx_event_sync", "gfx_last_error", "gfx_replay", "gfx_sim_run", "gfx_sim_run_stream"):
        assert n in names
    assert len(names) >= 40


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(simabi.PRODUCT_SO)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", simabi.PRODUCT_SO], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gfx_[a-z0-9_]+)", out))
    assert set(declared_functions()) <= exported


def test_package_import_and_status_codes_without_gpu():
    import paper_2303_05601_b200 as gfx
    n = C.c_int(-1)
    rc = gfx._ffi.gfx_device_count(C.byref(n))
    if rc != 0:  # no GPU here: a loud CUDA-class error, never a silent fallback
        assert rc == 3 and gfx._ffi.gfx_last_error()
        with pytest.raises(gfx.GfxError):
            gfx.check(rc)


def test_host_param_stream_matches_oracle():
    import numpy as np
    import paper_2303_05601_b200 as gfx
    olib = C.CDLL(simabi.ORACLE_SO)
    olib.orc_fill_params.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_float, C.c_void_p]
    for seed, tensor, scale in ((1, 0, 1.0), (gfx.model_seed("vgg19"), 5, 0.03125), (2 ** 63 + 7, 0xFFFFFFFF, 0.5)):
        a = np.zeros(4096, np.float32)
        b = np.zeros(4096, np.float32)
        gfx.check(gfx._ffi.gfx_host_fill_params(a.ctypes.data, a.size, seed, tensor, scale))
        olib.orc_fill_params(seed, tensor, b.size, scale, b.ctypes.data)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_model_catalog_charges_cover_arena_pages():
    """occupation_mb = 2 MiB x pages, so the reference's sum-of-sizes capacity
    model and the paged arena agree exactly."""
    import paper_2303_05601_b200 as gfx
    import csv
    for name in ("mlp_c2", "mlp_c2_paper"):
        specs = {s.model_id: s for s in gfx.load_model_specs(name)}
        rows = list(csv.DictReader(open(os.path.join(gfx.DATA_DIR, f"{name}_catalog.csv"))))
        assert len(rows) == 22
        for r in rows:
            s = specs[r["model_id"]]
            assert float(r["occupation_mb"]) == 2 * s.pages
            assert s.pages == -(-s.bytes // (2 << 20))


def test_model_registration_limits_without_gpu():
    """Shapes the inference path cannot take are refused at registration, with
    the reason (no GPU needed): width > 8192, more than 16 layers, layer inputs
    not a multiple of 32, outputs not a multiple of 4, unknown family."""
    import ctypes as C

    import paper_2303_05601_b200 as gfx
    from paper_2303_05601_b200 import _ffi

    def reg(dims, n_layers=None, family=None):
        d = gfx.ModelSpec("edge", "mlp", dims, 0, 0).desc()
        if n_layers is not None:
            d.n_layers = n_layers
        if family is not None:
            d.family = family
        rc = _ffi.gfx_model_register(60, C.byref(d))
        return rc, _ffi.gfx_last_error().decode()

    assert reg([1024, 8224, 1000])[1] == "bad layer width"
    assert reg([1024] * 16 + [1000], n_layers=17)[1] == "bad layer count"
    assert "multiples of 32" in reg([1000, 1024])[1]
    assert "multiples of 32" in reg([1024, 1001])[1]
    assert "family" in reg([1024, 1000], family=7)[1]
    # 16 layers of 8192 x 8192 fp32 = 4.3 GB: beyond the 1024-page (2 GiB) page table
    assert "page-table limit" in reg([8192] * 16 + [1000], n_layers=16)[1]


def test_sim_rejects_unknown_policy_values():
    """A policy id outside 0..2 is a caller error through the C-ABI, not a silent LALBO3."""
    import pytest
    import simabi
    lib = simabi.load_product()
    for bad in (3, -1, 17):
        cfg = simabi.make_config(gpus=1, capacity_mb=204.0, policy=bad, minutes=1)
        with pytest.raises(simabi.SimError, match="policy"):
            lib.run(simabi.table1_catalog(), cfg)


def test_cluster_command_ring_across_processes():
    """N1's shared-memory SPSC command ring: 200k commands from a forked producer
    arrive in order and untorn (the daemon/coordinator transport, no device)."""
    import paper_2303_05601_b200 as gfx
    rc = gfx._ffi.gfx_cluster_ring_selftest(200_000)
    assert rc == 0, gfx._ffi.gfx_cluster_last_error()


def test_cluster_without_device_fails_loudly():
    """The manager daemons start, fail on the missing device, and the coordinator
    raises the daemon's CUDA error (no hang, no CPU fallback, segment removed)."""
    import ctypes as C
    import os

    import pytest

    import paper_2303_05601_b200 as gfx
    n = C.c_int(0)
    if gfx._ffi.gfx_device_count(C.byref(n)) == 0 and n.value > 0:
        pytest.skip("a GPU is present (covered by tests/test_gpu_cluster.py)")
    with pytest.raises(gfx.ClusterError) as ei:
        gfx.Cluster(gfx.catalog_text("mlp_c2_paper"), gfx.sim_config(gpus=2, capacity_mb=204.0, minutes=1),
                    gfx.load_model_specs("mlp_c2"))
    assert ei.value.code == 3 and "gfx_managerd" in str(ei.value)
    assert not [f for f in os.listdir("/dev/shm") if f.startswith(f"gfx_cluster_{os.getpid()}_")]
