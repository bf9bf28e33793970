"""ctypes wrapper of the C++ oracle (oracle_sort.cpp).  Test infrastructure only."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle_sort.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def lib_path() -> str:
    return _LIB


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain g++ -O2; no tuning -- it is the checker)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-pthread", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, u64, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32
        L.oracle_sort.argtypes = [vp, vp, u64, u32, u32]
        L.oracle_sort.restype = ctypes.c_int
        L.oracle_sort_parallel.argtypes = [vp, vp, u64, u32, u32, u32]
        L.oracle_sort_parallel.restype = ctypes.c_int
        L.oracle_digit.argtypes = [vp, u32, u32]
        L.oracle_digit.restype = ctypes.c_int
        L.oracle_digit_hist.argtypes = [vp, u64, u32, u32, u32, vp]
        L.oracle_digit_hist.restype = ctypes.c_int
        L.oracle_key_compare.argtypes = [vp, vp, u32]
        L.oracle_key_compare.restype = ctypes.c_int
        L.oracle_rank_bounds.argtypes = [vp, u64, u32, u32, vp, vp, vp]
        L.oracle_rank_bounds.restype = ctypes.c_int
        L.oracle_compare.argtypes = [vp, vp, u64, u32, u32]
        L.oracle_compare.restype = ctypes.c_int64
        _lib = L
    return _lib


def _as_records(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    assert a.dtype == np.uint8 and a.ndim == 2, "records are an (n, R) uint8 array"
    return a


def sort(records: np.ndarray, K: int) -> np.ndarray:
    a = _as_records(records)
    n, R = a.shape
    out = np.empty_like(a)
    rc = _load().oracle_sort(a.ctypes.data, out.ctypes.data, n, R, K)
    if rc != 0:
        raise ValueError(f"oracle_sort: invalid R={R} K={K}")
    return out


def sort_parallel(records: np.ndarray, K: int, threads: int | None = None) -> np.ndarray:
    """sort() on `threads` host cores (chunked std::stable_sort + std::merge
    rounds): byte-identical to sort().  The benchmark's all-cores CPU baseline."""
    a = _as_records(records)
    n, R = a.shape
    out = np.empty_like(a)
    t = threads or os.cpu_count() or 1
    if _load().oracle_sort_parallel(a.ctypes.data, out.ctypes.data, n, R, K, t) != 0:
        raise ValueError(f"oracle_sort_parallel: invalid R={R} K={K}")
    return out


def digit(record: np.ndarray, K: int, d: int) -> int:
    r = np.ascontiguousarray(record, dtype=np.uint8).reshape(-1)
    v = _load().oracle_digit(r.ctypes.data, K, d)
    if v < 0:
        raise ValueError("digit depth out of range")
    return v


def digit_hist(records: np.ndarray, K: int, d: int) -> np.ndarray:
    a = _as_records(records)
    n, R = a.shape
    out = np.zeros(256, dtype=np.uint64)
    if _load().oracle_digit_hist(a.ctypes.data, n, R, K, d, out.ctypes.data) != 0:
        raise ValueError("bad digit/K")
    return out


def key_compare(a: np.ndarray, b: np.ndarray, K: int) -> int:
    x = np.ascontiguousarray(a, dtype=np.uint8).reshape(-1)
    y = np.ascontiguousarray(b, dtype=np.uint8).reshape(-1)
    return _load().oracle_key_compare(x.ctypes.data, y.ctypes.data, K)


def compare(got: np.ndarray, want: np.ndarray, K: int) -> int:
    g, w = _as_records(got), _as_records(want)
    assert g.shape == w.shape
    n, R = g.shape
    return int(_load().oracle_compare(g.ctypes.data, w.ctypes.data, n, R, K))


def rank_bounds(records: np.ndarray, K: int, key_record: np.ndarray):
    """(#keys < k, #keys <= k) over `records` for the key of `key_record`."""
    a = _as_records(records)
    n, R = a.shape
    k = np.ascontiguousarray(key_record, dtype=np.uint8).reshape(-1)
    lt = ctypes.c_uint64(0)
    le = ctypes.c_uint64(0)
    if _load().oracle_rank_bounds(a.ctypes.data, n, R, K, k.ctypes.data, ctypes.byref(lt), ctypes.byref(le)) != 0:
        raise ValueError("bad K/R")
    return int(lt.value), int(le.value)


def unique_count(sorted_records: np.ndarray, K: int):
    """Distinct keys of key-sorted records and their multiplicities, in key order
    -- the k-mer counting step the paper's sorter serves in KMC3 (PAPER.md:280-282
    §4.2).  Plain definition: a run of equal keys (bytes [0, K)) is one entry.
    Returns (keys: (U, K) uint8, counts: (U,) int64).  Test infrastructure only."""
    a = _as_records(sorted_records)
    n = a.shape[0]
    if n == 0:
        return np.zeros((0, K), dtype=np.uint8), np.zeros((0,), dtype=np.int64)
    keys = a[:, :K]
    head = np.ones(n, dtype=bool)
    head[1:] = np.any(keys[1:] != keys[:-1], axis=1)
    starts = np.flatnonzero(head)
    counts = np.diff(np.append(starts, n))
    return np.ascontiguousarray(keys[starts]), counts.astype(np.int64)
