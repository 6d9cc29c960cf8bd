"""B200-native GPU function-execution path of arXiv 2303.05601.

The product is the native library ``_lib/libgpufaas_b200.so`` (C++ control
plane + sm_100a CUDA data plane behind the C-ABI in include/gpufaas_b200.h).
This package is a thin ctypes binding over that C-ABI; there is no Python or
CPU fallback for any device operation — importing it without the built
library raises.
"""
from ._ffi import lib, GfxError, check  # noqa: F401
from .models import (ModelSpec, load_model_specs, register_models, model_seed, catalog_text,  # noqa: F401
                     DATA_DIR)
from .replay import (Replay, ReplayResult, sim_config, c3_config, c3_rpm, C3_ARENA_MB,  # noqa: F401
                     azure_trace_to_csv)
from .cluster import Cluster, ClusterError  # noqa: F401

__all__ = ["lib", "GfxError", "ModelSpec", "load_model_specs", "register_models", "model_seed",
           "catalog_text", "Replay", "ReplayResult", "sim_config", "c3_config", "c3_rpm", "C3_ARENA_MB", "azure_trace_to_csv",
           "DATA_DIR", "Cluster", "ClusterError"]
