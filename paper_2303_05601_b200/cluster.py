"""The GPU Manager as one daemon process per GPU (N1) through the product C-ABI
(gfx_cluster_* / gfx_managerd): this process runs the global cache manager
(the reference control plane) and feeds every daemon over shared memory."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _ffi
from .replay import ReplayResult


class ClusterError(_ffi.GfxError):
    pass


def _check(rc: int):
    if rc != 0:
        raise ClusterError(rc, _ffi.gfx_cluster_last_error().decode(errors="replace"))


class Cluster:
    """G gfx_managerd processes (one per GPU) plus the coordinator in this process.
    devices: CUDA device per GPU (default: all on device 0 = emulated peers)."""

    def __init__(self, catalog_csv: str, cfg: _ffi.SimConfig, specs, devices=None, use_p2p=True,
                 spawn=True, shm_name: str | None = None, trace_csv: str | None = None):
        G = cfg.gpu_count
        self._cat = catalog_csv.encode()
        self._trace = trace_csv.encode() if trace_csv else None
        self._models = (_ffi.ModelDesc * len(specs))(*[s.desc() for s in specs])
        self._devices = (C.c_int32 * G)(*(devices if devices is not None else [0] * G))
        self._name = shm_name.encode() if shm_name else None
        a = _ffi.ClusterArgs()
        a.catalog_csv = self._cat
        a.trace_csv = self._trace
        a.cfg = cfg
        a.models = self._models
        a.n_models = len(specs)
        a.use_p2p = int(use_p2p)
        a.devices = self._devices
        a.spawn = int(spawn)
        a.shm_name = self._name
        self.h = C.c_void_p()
        _check(_ffi.gfx_cluster_create(C.byref(a), C.byref(self.h)))

    def _result(self, r) -> ReplayResult:
        return ReplayResult({k: getattr(r, k) for k, _ in r._fields_})

    def run(self) -> ReplayResult:
        """The deterministic schedule (run_stream, bit-exact with the reference) executed by the daemons."""
        r = _ffi.ReplayResultC()
        _check(_ffi.gfx_cluster_run(self.h, C.byref(r)))
        return self._result(r)

    def run_live(self, time_scale: float, ema_alpha: float = 0.0) -> ReplayResult:
        """Live closed-loop serving with one process per GPU; sim_* latency fields hold real seconds."""
        r = _ffi.ReplayResultC()
        _check(_ffi.gfx_cluster_run_live(self.h, float(time_scale), float(ema_alpha), C.byref(r)))
        return self._result(r)

    def output(self, request_id: int, shape=(2, 32, 1000)) -> np.ndarray:
        out = np.zeros(shape, np.float32)
        _check(_ffi.gfx_cluster_output(self.h, int(request_id), out.ctypes.data, out.nbytes))
        return out

    def request_gpu(self, request_id: int) -> int:
        g = C.c_int32()
        _check(_ffi.gfx_cluster_request_gpu(self.h, int(request_id), C.byref(g)))
        return g.value

    def close(self):
        if self.h:
            _check(_ffi.gfx_cluster_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
