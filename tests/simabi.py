"""Uniform ctypes view of the three control-plane implementations.

  * ``ref``     — the UNMODIFIED reference simulator compiled in place
                  (oracle/_ref/libgpufaas_ref.so, prefix ``ref_sim_``);
  * ``oracle``  — our plain-C restatement (oracle/_build/liboracle.so, ``orc_sim_``);
  * ``product`` — the B200 build's C++ control plane
                  (paper_2303_05601_b200/_lib/libgpufaas_b200.so, ``gfx_sim_``).

All three export the same C ABI (see oracle/gpufaas_oracle.h for the struct
layout and the canonical FNV-1a digests) so parity is checked field by field.
Test infrastructure only.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libgpufaas_ref.so")
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
PRODUCT_SO = os.path.join(ROOT, "paper_2303_05601_b200", "_lib", "libgpufaas_b200.so")
GOLDEN = os.path.join(ROOT, "tests", "golden")

POLICIES = {"lb": 0, "lalb": 1, "lalbo3": 2}
KINDS = ["hit_idle", "miss_idle", "enqueue_local"]


class SimConfig(C.Structure):
    _fields_ = [
        ("gpu_count", C.c_int32),
        ("policy", C.c_int32),
        ("o3_limit", C.c_int32),
        ("working_set", C.c_int32),
        ("per_minute_total", C.c_int32),
        ("duration_minutes", C.c_int32),
        ("use_synthetic_trace", C.c_int32),
        ("syn_function_count", C.c_int32),
        ("syn_minutes", C.c_int32),
        ("syn_draws_per_minute", C.c_int32),
        ("debug_checks", C.c_int32),
        ("log_events", C.c_int32),
        ("use_reference_scheduler", C.c_int32),
        ("pipeline", C.c_int32),
        ("capacity_mb", C.c_double),
        ("syn_zipf_exponent", C.c_double),
        ("seed", C.c_uint64),
        ("syn_seed", C.c_uint64),
    ]


def make_config(gpus=12, capacity_mb=8192.0, policy="lalbo3", o3_limit=25, working_set=15,
                rpm=325, minutes=6, seed=1, synthetic=True, syn_functions=60, syn_minutes=6,
                syn_draws=3000, syn_zipf=0.7063, syn_seed=91, debug_checks=False, log_events=0,
                reference_scheduler=False, pipeline=False) -> SimConfig:
    """Defaults = the reference SimConfig defaults (proj/include/gpufaas/engine.hpp:20-32)."""
    c = SimConfig()
    c.gpu_count = gpus
    c.policy = POLICIES[policy] if isinstance(policy, str) else policy
    c.o3_limit = o3_limit
    c.working_set = working_set
    c.per_minute_total = rpm
    c.duration_minutes = minutes
    c.use_synthetic_trace = 1 if synthetic else 0
    c.syn_function_count = syn_functions
    c.syn_minutes = syn_minutes
    c.syn_draws_per_minute = syn_draws
    c.syn_zipf_exponent = syn_zipf
    c.syn_seed = syn_seed
    c.debug_checks = 1 if debug_checks else 0
    c.log_events = log_events
    c.use_reference_scheduler = 1 if reference_scheduler else 0
    c.pipeline = 1 if pipeline else 0
    c.capacity_mb = capacity_mb
    c.seed = seed
    return c


class OrcReport(C.Structure):
    _fields_ = [
        ("request_count", C.c_int64), ("total_sim_time_s", C.c_double),
        ("has_latency", C.c_int32), ("has_ratios", C.c_int32), ("has_time", C.c_int32),
        ("max_skip_count", C.c_int32),
        ("avg_latency_s", C.c_double), ("latency_variance_s2", C.c_double),
        ("cache_miss_ratio", C.c_double), ("false_miss_ratio", C.c_double),
        ("avg_top_model_duplicates", C.c_double), ("utilization_busy", C.c_double),
        ("utilization_infer_only", C.c_double),
        ("hits", C.c_int64), ("misses", C.c_int64), ("false_misses", C.c_int64),
        ("local_enqueues", C.c_int64), ("evictions", C.c_int64),
        ("top_model_idx", C.c_int32), ("pad_", C.c_int32),
    ]

    def as_dict(self, model_ids=None) -> dict:
        """Same keys as report_to_json (proj/src/metrics.cpp:109-141), minus per_model."""
        d = {"request_count": self.request_count, "total_sim_time_s": self.total_sim_time_s}
        for k in ("avg_latency_s", "latency_variance_s2"):
            d[k] = getattr(self, k) if self.has_latency else None
        for k in ("cache_miss_ratio", "false_miss_ratio"):
            d[k] = getattr(self, k) if self.has_ratios else None
        for k in ("avg_top_model_duplicates", "utilization_busy", "utilization_infer_only"):
            d[k] = getattr(self, k) if self.has_time else None
        for k in ("hits", "misses", "false_misses", "local_enqueues", "evictions", "max_skip_count"):
            d[k] = getattr(self, k)
        d["top_model"] = (model_ids[self.top_model_idx] if model_ids and self.top_model_idx >= 0
                          else self.top_model_idx)
        return d


@dataclass
class SimResult:
    ints: np.ndarray            # [n, 7] kind, request, gpu, from_local, false_miss, skip, n_evicted
    times: np.ndarray           # [n, 3] completion, load, infer
    model_idx: np.ndarray
    arrival: np.ndarray
    dispatched: np.ndarray
    completed: np.ndarray
    skip: np.ndarray
    decision_digest: int
    request_digest: int
    log_digest: int
    log: str
    run_ns: float
    report: dict = field(default_factory=dict)

    @property
    def latency_us(self) -> np.ndarray:
        return self.completed - self.arrival

    def percentile_s(self, q: float) -> float:
        """Nearest-rank percentile of completed - arrival."""
        lat = np.sort(self.latency_us)
        if lat.size == 0:
            return float("nan")
        rank = int(np.ceil(q / 100.0 * lat.size))
        return float(lat[max(rank, 1) - 1]) / 1e6

    def counts(self) -> dict:
        k = self.ints[:, 0]
        disp = k != 2
        return {
            "decisions": int(len(k)),
            "hits": int((k == 0).sum()),
            "misses": int((k == 1).sum()),
            "false_misses": int(((k == 1) & (self.ints[:, 4] == 1)).sum()),
            "local_enqueues": int((k == 2).sum()),
            "evictions": int(self.ints[disp, 6].sum()),
            "max_skip": int(self.ints[:, 5].max()) if len(k) else 0,
        }


class SimError(RuntimeError):
    pass


class SimLib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        L = self.lib
        p = prefix

        def fn(name, res, args):
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = args
            return f

        self._last_error = fn("last_error", C.c_char_p, [])
        self._run = fn("run", C.c_void_p, [C.c_char_p, C.c_char_p, C.POINTER(SimConfig)])
        self._run_stream = fn("run_stream", C.c_void_p,
                              [C.c_char_p, C.POINTER(SimConfig), C.c_int, C.POINTER(C.c_int32),
                               C.POINTER(C.c_int64)])
        self._nd = fn("num_decisions", C.c_int64, [C.c_void_p])
        self._nr = fn("num_requests", C.c_int64, [C.c_void_p])
        self._run_ns = fn("run_ns", C.c_double, [C.c_void_p])
        self._get_dec = fn("get_decisions", None, [C.c_void_p, C.c_void_p, C.c_void_p])
        self._get_req = fn("get_requests", None, [C.c_void_p] + [C.c_void_p] * 5)
        self._dd = fn("decision_digest", C.c_uint64, [C.c_void_p])
        self._rd = fn("request_digest", C.c_uint64, [C.c_void_p])
        self._ld = fn("log_digest", C.c_uint64, [C.c_void_p])
        self._log = fn("log", C.c_char_p, [C.c_void_p])
        self._free = fn("free", None, [C.c_void_p])
        self._report_json = getattr(L, p + "report_json", None)
        if self._report_json is not None:
            self._report_json.restype = C.c_char_p
            self._report_json.argtypes = [C.c_void_p]
        self._get_report = getattr(L, p + "get_report", None)
        if self._get_report is not None:
            self._get_report.restype = None
            self._get_report.argtypes = [C.c_void_p, C.POINTER(OrcReport)]

    def _collect(self, h) -> SimResult:
        if not h:
            raise SimError(self._last_error().decode())
        try:
            nd = self._nd(h)
            nr = self._nr(h)
            ints = np.zeros((nd, 7), dtype=np.int32)
            times = np.zeros((nd, 3), dtype=np.int64)
            if nd:
                self._get_dec(h, ints.ctypes.data, times.ctypes.data)
            mi = np.zeros(nr, np.int32)
            ar = np.zeros(nr, np.int64)
            di = np.zeros(nr, np.int64)
            co = np.zeros(nr, np.int64)
            sk = np.zeros(nr, np.int32)
            if nr:
                self._get_req(h, mi.ctypes.data, ar.ctypes.data, di.ctypes.data, co.ctypes.data,
                              sk.ctypes.data)
            rep = {}
            if self._report_json is not None:
                rep = json.loads(self._report_json(h).decode())
            elif self._get_report is not None:
                r = OrcReport()
                self._get_report(h, C.byref(r))
                rep = r.as_dict()
            return SimResult(ints, times, mi, ar, di, co, sk, int(self._dd(h)), int(self._rd(h)),
                             int(self._ld(h)), self._log(h).decode(), float(self._run_ns(h)), rep)
        finally:
            self._free(h)

    def run(self, catalog_csv: str, cfg: SimConfig, trace_csv: str | None = None) -> SimResult:
        h = self._run(catalog_csv.encode(), trace_csv.encode() if trace_csv else None, C.byref(cfg))
        return self._collect(h)

    def run_stream(self, catalog_csv: str, cfg: SimConfig, model_idx, arrival_us) -> SimResult:
        mi = np.ascontiguousarray(model_idx, dtype=np.int32)
        ar = np.ascontiguousarray(arrival_us, dtype=np.int64)
        h = self._run_stream(catalog_csv.encode(), C.byref(cfg), len(mi),
                             mi.ctypes.data_as(C.POINTER(C.c_int32)),
                             ar.ctypes.data_as(C.POINTER(C.c_int64)))
        return self._collect(h)

    def run_live_timed(self, catalog_csv: str, cfg: SimConfig, time_scale: float, ema_alpha: float = 0.0,
                       trace_csv: str | None = None) -> SimResult:
        """Product only: run_live() against the timed stand-in device."""
        f = getattr(self.lib, self.prefix + "run_live_timed")
        f.restype = C.c_void_p
        f.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(SimConfig), C.c_double, C.c_double]
        h = f(catalog_csv.encode(), trace_csv.encode() if trace_csv else None, C.byref(cfg), time_scale, ema_alpha)
        return self._collect(h)


def load_ref() -> SimLib:
    return SimLib(REF_SO, "ref_sim_")


def load_oracle() -> SimLib:
    return SimLib(ORACLE_SO, "orc_sim_")


def load_product() -> SimLib:
    return SimLib(PRODUCT_SO, "gfx_sim_")


def table1_catalog() -> str:
    """Paper Table I catalog fixture (copied once from proj/data/models.csv by
    tests/golden/make_golden.py)."""
    with open(os.path.join(GOLDEN, "table1_models.csv")) as f:
        return f.read()


def assert_same(a: SimResult, b: SimResult, what: str = ""):
    """Decision-stream + per-request parity (Appendix C item 11)."""
    assert a.ints.shape == b.ints.shape, f"{what}: decision count {a.ints.shape} vs {b.ints.shape}"
    if not np.array_equal(a.ints, b.ints) or not np.array_equal(a.times, b.times):
        bad = np.nonzero((a.ints != b.ints).any(1) | (a.times != b.times).any(1))[0][0]
        raise AssertionError(f"{what}: first differing decision #{bad}: {a.ints[bad]} {a.times[bad]} "
                             f"vs {b.ints[bad]} {b.times[bad]}")
    assert a.decision_digest == b.decision_digest, f"{what}: decision digest (evicted lists differ)"
    assert np.array_equal(a.dispatched, b.dispatched), f"{what}: dispatched_at"
    assert np.array_equal(a.completed, b.completed), f"{what}: completed_at"
    assert np.array_equal(a.skip, b.skip), f"{what}: skip_count"
    assert a.request_digest == b.request_digest, what
