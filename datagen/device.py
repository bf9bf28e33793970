"""ctypes wrapper of the device generator (libradsort_datagen.so)."""
from __future__ import annotations

import ctypes
import os

from .host import CONFIGS, DISTS, PAYLOADS

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def _load():
    global _lib
    if _lib is None:
        p = os.path.join(_HERE, "libradsort_datagen.so")
        if not os.path.exists(p):
            raise RuntimeError(f"{p} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(p)
        L.datagen_fill.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                                   ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p]
        L.datagen_fill.restype = ctypes.c_int
        _lib = L
    return _lib


def fill(ptr: int, n: int, R: int, K: int, dist: str = "uniform", payload: str = "random", seed: int = 1,
         first: int = 0, stream_ptr: int = 0) -> None:
    rc = _load().datagen_fill(ctypes.c_void_p(ptr), n, first, R, K, DISTS[dist], PAYLOADS[payload], seed,
                              ctypes.c_void_p(stream_ptr))
    if rc:
        raise RuntimeError(f"datagen_fill failed: cudaError {rc}")


def generate_tensor(n: int, R: int, K: int, dist: str = "uniform", payload: str = "random", seed: int = 1,
                    first: int = 0, device: str = "cuda"):
    import torch

    t = torch.empty((n, R), dtype=torch.uint8, device=device)
    if n:
        fill(t.data_ptr(), n, R, K, dist, payload, seed, first, torch.cuda.current_stream().cuda_stream)
    return t


def generate_config(name: str, n: int | None = None, first: int = 0, device: str = "cuda"):
    c = CONFIGS[name]
    return generate_tensor(n if n is not None else c["n"], c["R"], c["K"], c["dist"], c["payload"], c["seed"],
                           first, device)
