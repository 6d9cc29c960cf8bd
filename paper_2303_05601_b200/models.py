"""Model catalog + model-store registration for the B200 path."""
from __future__ import annotations

import csv
import ctypes as C
import os
from dataclasses import dataclass

from . import _ffi

DATA_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")
GFX_MODEL_MLP = 1
GFX_MODEL_BERT = 2


def model_seed(model_id: str) -> int:
    """FNV-1a-64 of the model id: the model's parameter stream."""
    h = 14695981039346656037
    for b in model_id.encode():
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


@dataclass
class ModelSpec:
    model_id: str
    family: str
    dims: list
    bytes: int
    pages: int

    @property
    def seed(self) -> int:
        return model_seed(self.model_id)

    def desc(self) -> _ffi.ModelDesc:
        if self.family == "bert":  # dims = [layers, d_model, heads, ffn, seq, sequences]
            return bert_desc(self.dims[0], self.dims[5], self.seed, d=self.dims[1], heads=self.dims[2],
                             ffn=self.dims[3], seq=self.dims[4])
        d = _ffi.ModelDesc()
        d.family = GFX_MODEL_MLP
        d.n_layers = len(self.dims) - 1
        for i, v in enumerate(self.dims):
            d.dims[i] = v
        d.batch = 32
        d.seed = self.seed
        return d


def bert_desc(layers: int, sequences: int, seed: int, d=768, heads=12, ffn=3072, seq=128) -> _ffi.ModelDesc:
    """BERT-base-style encoder (C5): bf16, post-LN, tanh pooler."""
    m = _ffi.ModelDesc()
    m.family = GFX_MODEL_BERT
    m.n_layers = layers
    for i, v in enumerate((d, heads, ffn, seq)):
        m.dims[i] = v
    m.batch = sequences
    m.seed = seed
    return m


def load_model_specs(name: str = "mlp_c2") -> list[ModelSpec]:
    out = []
    with open(os.path.join(DATA_DIR, f"{name}_models.csv")) as f:
        for r in csv.DictReader(f):
            out.append(ModelSpec(r["model_id"], r["family"], [int(x) for x in r["dims"].split("x")],
                                 int(r["bytes"]), int(r["pages"])))
    return out


def catalog_text(name: str = "mlp_c2") -> str:
    with open(os.path.join(DATA_DIR, f"{name}_catalog.csv")) as f:
        return f.read()


def register_models(specs: list[ModelSpec]) -> None:
    """Builds every model's parameter blob in the pinned host model store; row i
    of the catalog is model index i."""
    for i, s in enumerate(specs):
        _ffi.check(_ffi.gfx_model_register(i, C.byref(s.desc())))
        nb = C.c_uint64()
        _ffi.check(_ffi.gfx_model_bytes(i, C.byref(nb)))
        if nb.value != s.bytes:
            raise RuntimeError(f"model {s.model_id}: blob {nb.value} B != spec {s.bytes} B")
