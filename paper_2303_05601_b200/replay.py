"""Trace replay through the product C-ABI (gfx_replay_*)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _ffi

POLICIES = {"lb": 0, "lalb": 1, "lalbo3": 2}


def sim_config(gpus=1, capacity_mb=204.0, policy="lalbo3", o3_limit=25, working_set=15, rpm=325,
               minutes=6, seed=1, syn_functions=60, syn_minutes=6, syn_draws=3000, syn_zipf=0.7063,
               syn_seed=91, pipeline=False) -> _ffi.SimConfig:
    """Reference SimConfig (proj/include/gpufaas/engine.hpp:20-32) with the C2 arena.
    pipeline=True: the pipelined-GPU extension (SchedulerConfig::pipeline; not the
    reference's semantics, checked against the oracle's restatement of it)."""
    c = _ffi.SimConfig()
    c.gpu_count = gpus
    c.policy = POLICIES[policy] if isinstance(policy, str) else int(policy)
    c.o3_limit = o3_limit
    c.working_set = working_set
    c.per_minute_total = rpm
    c.duration_minutes = minutes
    c.use_synthetic_trace = 1
    c.syn_function_count = syn_functions
    c.syn_minutes = syn_minutes
    c.syn_draws_per_minute = syn_draws
    c.syn_zipf_exponent = syn_zipf
    c.syn_seed = syn_seed
    c.capacity_mb = capacity_mb
    c.seed = seed
    c.pipeline = 1 if pipeline else 0
    return c


def azure_trace_to_csv(in_path: str, out_path: str, top_k: int = 1000, max_minutes: int = 0) -> tuple[int, int]:
    """Azure Functions 2019 invocation file -> trace CSV of its top_k functions
    (extension; streaming, C++). Returns (rows read, rows kept);
    the output feeds Replay(trace_csv=...) / the simulator like the bundled trace."""
    read, kept = C.c_int64(), C.c_int64()
    if _ffi.gfx_sim_azure_convert(in_path.encode(), out_path.encode(), int(top_k), int(max_minutes),
                                  C.byref(read), C.byref(kept)) != 0:
        raise _ffi.GfxError(-1, _ffi.gfx_sim_last_error().decode(errors="replace"))
    return read.value, kept.value


C3_ARENA_MB = 128.0  # per GPU: 8 x 128 MiB < 1294 MB of C3 weights (working set > aggregate cache)


def c3_rpm(gpus: int, mean_infer_s: float = 1.315, rho: float = 0.59) -> int:
    """Request rate putting the fleet at rho_infer = rpm/60 * mean(infer)/G (the
    reference regime, Appendix B.5). 1.315 s = mean infer_time_s of the mlp_c3 catalog."""
    return int(round(rho * 60.0 * gpus / mean_infer_s))


def c3_config(gpus=8, policy="lalbo3", zipf=0.7063, seed=1, o3_limit=25) -> _ffi.SimConfig:
    """configs[2] (C3) / configs[3] (C4, zipf in {0.7063, 1.0, 1.2}, G in {2, 4, 8}): the
    mlp_c3 catalog (20 models, 25-100 MB), working set 20, 6 minutes, synthetic
    Azure-shaped trace (60 functions, 3000 draws/min, seed 91) at the given Zipf exponent."""
    return sim_config(gpus=gpus, capacity_mb=C3_ARENA_MB, policy=policy, o3_limit=o3_limit, working_set=20,
                      rpm=c3_rpm(gpus), minutes=6, seed=seed, syn_zipf=zipf)


@dataclass
class ReplayResult:
    raw: dict

    def __getattr__(self, k):
        try:
            return self.raw[k]
        except KeyError as e:
            raise AttributeError(k) from e


class Replay:
    """One replay context (GPU managers, device buffers, events) reused across runs."""

    def __init__(self, catalog_csv: str, cfg: _ffi.SimConfig, n_devices=1, first_device=0, only_gpu=-1,
                 use_p2p=False, host_io=False, record_kernels=False, record_requests=False,
                 keep_outputs=False, host_inputs: np.ndarray | None = None,
                 host_outputs: np.ndarray | None = None):
        self._cat = catalog_csv.encode()
        a = _ffi.ReplayArgs()
        a.catalog_csv = self._cat
        a.trace_csv = None
        a.cfg = cfg
        a.n_devices = n_devices
        a.first_device = first_device
        a.only_gpu = only_gpu
        a.use_p2p = int(use_p2p)
        a.host_io = int(host_io)
        a.record_kernels = int(record_kernels)
        a.record_requests = int(record_requests)
        a.keep_outputs = int(keep_outputs)
        self._in = host_inputs
        self._out = host_outputs
        a.host_inputs = host_inputs.ctypes.data if host_inputs is not None else None
        a.host_outputs = host_outputs.ctypes.data if host_outputs is not None else None
        self.args = a
        self.h = C.c_void_p()
        _ffi.check(_ffi.gfx_replay_create(C.byref(a), C.byref(self.h)))

    def run(self) -> ReplayResult:
        r = _ffi.ReplayResultC()
        _ffi.check(_ffi.gfx_replay_run(self.h, C.byref(r)))
        return ReplayResult({k: getattr(r, k) for k, _ in r._fields_})

    def run_live(self, time_scale: float, ema_alpha: float = 0.0) -> ReplayResult:
        """Live closed-loop serving of the same trace (extension):
        arrivals compressed by ``time_scale`` and released in real time, every
        completion observed on the device and fed back to the scheduler; with
        ``ema_alpha`` > 0 the planned load/infer times follow the event-measured
        device durations. The sim_* latency fields hold real seconds; the
        schedule is not reproducible run to run (it follows the device)."""
        r = _ffi.ReplayResultC()
        _ffi.check(_ffi.gfx_replay_run_live(self.h, float(time_scale), float(ema_alpha), C.byref(r)))
        return ReplayResult({k: getattr(r, k) for k, _ in r._fields_})

    def outputs(self, n_requests: int, shape=(2, 32, 1000)) -> np.ndarray:
        """Per-request fp32 outputs of the last run (MLP: logits + softmax;
        BERT: pass shape=(sequences, 768) for the pooled output)."""
        out = np.zeros((n_requests,) + tuple(shape), dtype=np.float32)
        _ffi.check(_ffi.gfx_replay_outputs(self.h, out.ctypes.data, out.nbytes))
        return out

    def request_info(self, n_requests: int):
        mi = np.zeros(n_requests, np.int32)
        svc = np.zeros(n_requests, np.float64)
        _ffi.check(_ffi.gfx_replay_requests(self.h, mi.ctypes.data, svc.ctypes.data, n_requests))
        return mi, svc

    def ipc_export(self) -> bytes:
        """This rank's CUDA IPC blob (arena + flag words) for cross-process peer fetch."""
        n = int(_ffi.gfx_replay_ipc_blob_bytes())
        buf = (C.c_char * n)()
        _ffi.check(_ffi.gfx_replay_ipc_export(self.h, buf, n))
        return bytes(buf)

    def ipc_import(self, blobs: list[bytes]):
        """Map every rank's blob (index = GPU id) before the first run."""
        n = int(_ffi.gfx_replay_ipc_blob_bytes())
        if any(len(b) != n for b in blobs):
            raise ValueError("ipc blobs of the wrong size")
        buf = C.create_string_buffer(b"".join(blobs), n * len(blobs))
        _ffi.check(_ffi.gfx_replay_ipc_import(self.h, buf, len(blobs)))

    def connect_peers(self, group=None):
        """All-gather the IPC blobs over torch.distributed (one process per GPU) and import them."""
        import torch.distributed as dist
        blobs = [None] * dist.get_world_size(group)
        dist.all_gather_object(blobs, self.ipc_export(), group=group)
        self.ipc_import(blobs)

    def close(self):
        if self.h:
            _ffi.check(_ffi.gfx_replay_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
