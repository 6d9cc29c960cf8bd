"""ctypes binding of include/gpufaas_b200.h (the product C-ABI)."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libgpufaas_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()). "
        "There is no CPU fallback for the B200 path.")

lib = C.CDLL(LIB_PATH)

GFX_MAX_LAYERS = 16


class GfxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[gfx {code}] {msg}")
        self.code = code


class SimConfig(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "gpu_count", "policy", "o3_limit", "working_set", "per_minute_total", "duration_minutes",
        "use_synthetic_trace", "syn_function_count", "syn_minutes", "syn_draws_per_minute",
        "debug_checks", "log_events", "use_reference_scheduler", "pipeline")] + [
        ("capacity_mb", C.c_double), ("syn_zipf_exponent", C.c_double),
        ("seed", C.c_uint64), ("syn_seed", C.c_uint64)]


class ModelDesc(C.Structure):
    _fields_ = [("family", C.c_int32), ("n_layers", C.c_int32),
                ("dims", C.c_int32 * (GFX_MAX_LAYERS + 1)), ("batch", C.c_int32), ("pad_", C.c_int32),
                ("seed", C.c_uint64)]


class ReplayArgs(C.Structure):
    _fields_ = [("catalog_csv", C.c_char_p), ("trace_csv", C.c_char_p), ("cfg", SimConfig),
                ("n_devices", C.c_int32), ("first_device", C.c_int32), ("only_gpu", C.c_int32),
                ("use_p2p", C.c_int32), ("host_io", C.c_int32), ("record_kernels", C.c_int32),
                ("record_requests", C.c_int32), ("keep_outputs", C.c_int32),
                ("host_inputs", C.c_void_p), ("host_outputs", C.c_void_p)]


class ReplayResultC(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "n_requests", "n_decisions", "hits", "misses", "false_misses", "local_enqueues", "evictions",
        "loads_h2d", "loads_p2p", "kernel_launches")] + [
        (n, C.c_uint64) for n in ("decision_digest", "h2d_bytes", "p2p_bytes", "io_h2d_bytes",
                                   "io_d2h_bytes")] + [
        (n, C.c_double) for n in ("device_ms", "host_ms", "sched_ms", "kernel_ms", "h2d_ms",
                                   "service_p50_ms", "service_p99_ms", "sim_p50_s", "sim_p99_s",
                                   "sim_avg_latency_s", "mlp_flops", "mlp_weight_bytes", "p2p_ms")]


class ClusterArgs(C.Structure):
    _fields_ = [("catalog_csv", C.c_char_p), ("trace_csv", C.c_char_p), ("cfg", SimConfig),
                ("models", C.POINTER(ModelDesc)), ("n_models", C.c_int32), ("use_p2p", C.c_int32),
                ("devices", C.POINTER(C.c_int32)), ("spawn", C.c_int32), ("pad_", C.c_int32),
                ("shm_name", C.c_char_p)]


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


_vp = C.c_void_p
gfx_last_error = _sig("gfx_last_error", C.c_char_p, [])
gfx_sim_last_error = _sig("gfx_sim_last_error", C.c_char_p, [])
gfx_sim_azure_convert = _sig("gfx_sim_azure_convert", C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.c_int,
                                                                C.POINTER(C.c_int64), C.POINTER(C.c_int64)])
gfx_device_count = _sig("gfx_device_count", C.c_int, [C.POINTER(C.c_int)])
gfx_device_init = _sig("gfx_device_init", C.c_int, [C.c_int, C.c_int])
gfx_model_register = _sig("gfx_model_register", C.c_int, [C.c_int, C.POINTER(ModelDesc)])
gfx_model_bytes = _sig("gfx_model_bytes", C.c_int, [C.c_int, C.POINTER(C.c_uint64)])
gfx_model_pages = _sig("gfx_model_pages", C.c_int, [C.c_int, C.POINTER(C.c_int32)])
gfx_models_clear = _sig("gfx_models_clear", C.c_int, [])
gfx_model_io_bytes = _sig("gfx_model_io_bytes", C.c_int, [C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)])
gfx_host_fill_input = _sig("gfx_host_fill_input", C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_uint64])
gfx_arena_create = _sig("gfx_arena_create", C.c_int, [C.c_int, C.c_uint64, C.POINTER(_vp)])
gfx_arena_destroy = _sig("gfx_arena_destroy", C.c_int, [_vp])
gfx_arena_reset = _sig("gfx_arena_reset", C.c_int, [_vp])
gfx_arena_free_pages = _sig("gfx_arena_free_pages", C.c_int, [_vp, C.POINTER(C.c_int32)])
gfx_arena_set_option = _sig("gfx_arena_set_option", C.c_int, [_vp, C.c_int32, C.c_int32])
GFX_OPT_GEMM_PAIR = 1
GFX_OPT_BERT_FLOW = 2
gfx_infer_sequence = _sig("gfx_infer_sequence", C.c_int, [_vp, _vp, C.c_int, _vp, C.c_uint64, _vp, C.c_uint64,
                                                          C.POINTER(C.c_double)])
gfx_bert_gemm = _sig("gfx_bert_gemm", C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int])
gfx_arena_resident = _sig("gfx_arena_resident", C.c_int, [_vp, C.c_int, C.POINTER(C.c_int32)])
gfx_load_h2d = _sig("gfx_load_h2d", C.c_int, [_vp, C.c_int, C.POINTER(_vp)])
gfx_fetch_p2p = _sig("gfx_fetch_p2p", C.c_int, [_vp, _vp, C.c_int, C.POINTER(_vp)])
gfx_evict = _sig("gfx_evict", C.c_int, [_vp, C.c_int])
gfx_infer = _sig("gfx_infer", C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int, C.POINTER(_vp)])
gfx_infer_debug = _sig("gfx_infer_debug", C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int, _vp])
gfx_infer_masked = _sig("gfx_infer_masked", C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int, _vp, _vp, C.POINTER(_vp)])
gfx_event_query = _sig("gfx_event_query", C.c_int, [_vp])
gfx_event_sync = _sig("gfx_event_sync", C.c_int, [_vp])
gfx_event_release = _sig("gfx_event_release", C.c_int, [_vp])
gfx_device_alloc = _sig("gfx_device_alloc", C.c_int, [_vp, C.c_uint64, C.POINTER(_vp)])
gfx_device_free = _sig("gfx_device_free", C.c_int, [_vp, _vp])
gfx_memcpy_h2d = _sig("gfx_memcpy_h2d", C.c_int, [_vp, _vp, _vp, C.c_uint64])
gfx_memcpy_d2h = _sig("gfx_memcpy_d2h", C.c_int, [_vp, _vp, _vp, C.c_uint64])
gfx_synchronize = _sig("gfx_synchronize", C.c_int, [_vp])
gfx_fill_params = _sig("gfx_fill_params", C.c_int, [_vp, _vp, C.c_uint64, C.c_uint64, C.c_uint32, C.c_float])
gfx_input_seed = _sig("gfx_input_seed", C.c_uint64, [C.c_int])
gfx_host_fill_params = _sig("gfx_host_fill_params", C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_uint32, C.c_float])
gfx_replay_create = _sig("gfx_replay_create", C.c_int, [C.POINTER(ReplayArgs), C.POINTER(_vp)])
gfx_replay_run = _sig("gfx_replay_run", C.c_int, [_vp, C.POINTER(ReplayResultC)])
gfx_replay_run_live = _sig("gfx_replay_run_live", C.c_int, [_vp, C.c_double, C.c_double,
                                                             C.POINTER(ReplayResultC)])
gfx_replay_outputs = _sig("gfx_replay_outputs", C.c_int, [_vp, _vp, C.c_uint64])
gfx_replay_requests = _sig("gfx_replay_requests", C.c_int, [_vp, _vp, _vp, C.c_int64])
gfx_replay_destroy = _sig("gfx_replay_destroy", C.c_int, [_vp])
gfx_replay_ipc_blob_bytes = _sig("gfx_replay_ipc_blob_bytes", C.c_uint64, [])
gfx_replay_ipc_export = _sig("gfx_replay_ipc_export", C.c_int, [_vp, _vp, C.c_uint64])
gfx_replay_ipc_import = _sig("gfx_replay_ipc_import", C.c_int, [_vp, _vp, C.c_int32])

gfx_cluster_last_error = _sig("gfx_cluster_last_error", C.c_char_p, [])
gfx_cluster_create = _sig("gfx_cluster_create", C.c_int, [C.POINTER(ClusterArgs), C.POINTER(_vp)])
gfx_cluster_run = _sig("gfx_cluster_run", C.c_int, [_vp, C.POINTER(ReplayResultC)])
gfx_cluster_run_live = _sig("gfx_cluster_run_live", C.c_int, [_vp, C.c_double, C.c_double, C.POINTER(ReplayResultC)])
gfx_cluster_output = _sig("gfx_cluster_output", C.c_int, [_vp, C.c_int32, _vp, C.c_uint64])
gfx_cluster_request_gpu = _sig("gfx_cluster_request_gpu", C.c_int, [_vp, C.c_int32, C.POINTER(C.c_int32)])
gfx_cluster_destroy = _sig("gfx_cluster_destroy", C.c_int, [_vp])
gfx_cluster_ring_selftest = _sig("gfx_cluster_ring_selftest", C.c_int, [C.c_int64])
gfx_managerd_serve = _sig("gfx_managerd_serve", C.c_int, [C.c_char_p, C.c_int32])


def check(rc: int):
    if rc != 0:
        raise GfxError(rc, gfx_last_error().decode(errors="replace"))
