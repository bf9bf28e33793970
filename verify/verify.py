from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def _load():
    global _lib
    if _lib is None:
        p = os.path.join(_HERE, "libradsort_verify.so")
        if not os.path.exists(p):
            raise RuntimeError(f"{p} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(p)
        L.verify_sorted.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p]
        L.verify_digest.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p]
        _lib = L
    return _lib


def sorted_check(ptr: int, n: int, R: int, K: int):
    out = (ctypes.c_ulonglong * 2)()
    rc = _load().verify_sorted(ptr, n, R, K, out)
    if rc:
        raise RuntimeError(f"verify_sorted failed: {rc}")
    return int(out[0]), int(out[1])


def digest(ptr: int, n: int, R: int):
    out = (ctypes.c_ulonglong * 2)()
    rc = _load().verify_digest(ptr, n, R, out)
    if rc:
        raise RuntimeError(f"verify_digest failed: {rc}")
    return int(out[0]), int(out[1])
