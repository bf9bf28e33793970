"""Thin Python binding of libradsort.so (include/radsort.h).

Argument marshalling only: every step of the sort runs in the library's CUDA
kernels.  torch is used for device memory, streams and process groups.  There
is no CPU fallback -- if the extension is missing, importing this module
raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RADSORT_LIB_PATH") or os.path.join(_HERE, "libradsort.so")

OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_NOT_INITIALIZED, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_CAPACITY = range(8)
KERNEL_CLASSES = ["sample", "hist", "plan", "scatter", "children", "local", "multi", "gather"]

# every symbol include/radsort.h declares
EXPORTS = ["radsort_init", "radsort_sort", "radsort_sort_host", "radsort_sort_host_stream", "radsort_sort_multi", "radsort_locate_bucket",
           "radsort_set_timing", "radsort_last_stats", "radsort_error_string", "radsort_finalize",
           "radsort_version", "radsort_loopback_create", "radsort_loopback_destroy", "radsort_sort_multi_loopback",
           "radsort_plan_quotas", "radsort_plan_digit", "radsort_plan_equal_split", "radsort_tinybench",
           "radsort_unique_count", "radsort_comm_get_unique_id", "radsort_comm_init", "radsort_comm_destroy",
           "radsort_tinysort", "radsort_plan_fused"]


class Stats(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64), ("rec_size", ctypes.c_uint32), ("key_size", ctypes.c_uint32),
        ("levels", ctypes.c_uint32), ("scatter_passes", ctypes.c_uint32),
        ("constant_digits_skipped", ctypes.c_uint32), ("first_digit", ctypes.c_uint32),
        ("records_scattered", ctypes.c_uint64), ("records_hist", ctypes.c_uint64),
        ("records_local", ctypes.c_uint64), ("records_tiny", ctypes.c_uint64),
        ("records_copied", ctypes.c_uint64),
        ("bins_large", ctypes.c_uint64), ("bins_local", ctypes.c_uint64), ("bins_tiny", ctypes.c_uint64),
        ("bins_final", ctypes.c_uint64),
        ("nvlink_bytes_sent", ctypes.c_uint64), ("nvlink_bytes_recv", ctypes.c_uint64),
        ("kernel_launches", ctypes.c_uint32 * 8), ("kernel_ms", ctypes.c_float * 8),
        ("kernel_bytes", ctypes.c_uint64 * 8),
        ("bins_split", ctypes.c_uint64), ("records_split", ctypes.c_uint64),
        ("exchange", ctypes.c_uint32), ("key_index", ctypes.c_uint32), ("wide_levels", ctypes.c_uint32),
    ]


class RadsortError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"radsort status {status}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                          "(radsort has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    vp, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
    L.radsort_init.argtypes = [i32]
    L.radsort_sort.argtypes = [vp, vp, u64, u32, u32, vp]
    L.radsort_sort_host.argtypes = [vp, u64, u32, u32, vp]
    L.radsort_sort_host_stream.argtypes = [vp, vp, u32, u64, u32, u32, vp, u32, vp, vp]
    L.radsort_sort_multi.argtypes = [vp, vp, u64, u64, ctypes.POINTER(u64), u32, u32, vp, vp]
    L.radsort_locate_bucket.argtypes = [vp, u64, ctypes.POINTER(u32), ctypes.POINTER(u64)]
    L.radsort_set_timing.argtypes = [i32]
    L.radsort_last_stats.argtypes = [ctypes.POINTER(Stats)]
    L.radsort_error_string.argtypes = [i32]
    L.radsort_error_string.restype = ctypes.c_char_p
    L.radsort_finalize.argtypes = []
    L.radsort_finalize.restype = None
    L.radsort_version.restype = ctypes.c_char_p
    L.radsort_loopback_create.argtypes = [i32, ctypes.POINTER(vp)]
    L.radsort_loopback_destroy.argtypes = [vp]
    L.radsort_sort_multi_loopback.argtypes = [vp, i32, vp, vp, u64, u64, ctypes.POINTER(u64), u32, u32, vp]
    L.radsort_plan_quotas.argtypes = [u64, i32, vp]
    L.radsort_plan_digit.argtypes = [vp, u64, ctypes.POINTER(u32)]
    L.radsort_plan_equal_split.argtypes = [vp, i32, u64, u64, vp]
    L.radsort_plan_fused.argtypes = [vp, i32, i32, u32, vp, vp, vp, vp]
    L.radsort_tinybench.argtypes = [u32, u32, u32, u32, u64, ctypes.POINTER(ctypes.c_double)]
    L.radsort_unique_count.argtypes = [vp, u64, u32, u32, vp, vp, ctypes.POINTER(u64), vp]
    L.radsort_tinysort.argtypes = [u32, u32, u32, u32, vp, vp, u64, vp]
    L.radsort_comm_get_unique_id.argtypes = [vp]
    L.radsort_comm_init.argtypes = [vp, i32, i32, i32, ctypes.POINTER(vp)]
    L.radsort_comm_destroy.argtypes = [vp]
    for f in ("radsort_plan_fused", "radsort_tinysort", "radsort_comm_get_unique_id", "radsort_comm_init", "radsort_comm_destroy", "radsort_init", "radsort_sort", "radsort_sort_host", "radsort_sort_host_stream", "radsort_sort_multi",
              "radsort_locate_bucket", "radsort_set_timing", "radsort_last_stats", "radsort_loopback_create", "radsort_loopback_destroy",
              "radsort_sort_multi_loopback", "radsort_plan_quotas", "radsort_plan_digit", "radsort_plan_equal_split",
              "radsort_tinybench", "radsort_unique_count"):
        getattr(L, f).restype = i32
    return L


lib = _load()


def _check(rc: int):
    if rc != OK:
        raise RadsortError(rc, lib.radsort_error_string(rc).decode())


def version() -> str:
    return lib.radsort_version().decode()


def init(device: int | None = None) -> None:
    import torch

    if device is None:
        device = torch.cuda.current_device()
    _check(lib.radsort_init(int(device)))


def _stream_ptr(stream):
    import torch

    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def sort(records, tmp, key_size: int, stream=None, n: int | None = None) -> None:
    """Sort records (a CUDA uint8 tensor of shape [n, R], contiguous) in place.
    tmp: CUDA scratch tensor of >= n*R bytes (contents undefined afterwards)."""
    assert records.is_cuda and tmp.is_cuda and records.is_contiguous() and tmp.is_contiguous()
    R = records.shape[1] if records.dim() == 2 else int(records.numel() // (n or 1))
    n = records.shape[0] if n is None else n
    assert tmp.numel() * tmp.element_size() >= n * R, "tmp too small"
    init(records.device.index)
    _check(lib.radsort_sort(ctypes.c_void_p(records.data_ptr()), ctypes.c_void_p(tmp.data_ptr()), n, R, key_size,
                            _stream_ptr(stream)))


def sort_ptr(records_ptr: int, tmp_ptr: int, n: int, rec_size: int, key_size: int, stream_ptr: int = 0) -> None:
    _check(lib.radsort_sort(ctypes.c_void_p(records_ptr), ctypes.c_void_p(tmp_ptr), n, rec_size, key_size,
                            ctypes.c_void_p(stream_ptr)))


def sort_host(records, key_size: int, stream=None) -> None:
    """End-to-end sort of a host (ideally pinned) uint8 tensor/array [n, R] in place."""
    import numpy as np

    if isinstance(records, np.ndarray):
        ptr, n, R = records.ctypes.data, records.shape[0], records.shape[1]
    else:
        ptr, n, R = records.data_ptr(), records.shape[0], records.shape[1]
    _check(lib.radsort_sort_host(ctypes.c_void_p(ptr), n, R, key_size, _stream_ptr(stream)))


def sort_host_stream(host_in, host_out, key_size: int, dev_bufs, dev_tmp, stream=None) -> None:
    """Pipelined end-to-end sort of a list of host batches (pinned uint8 tensors [n, R], all the
    same shape): host_out[k] = sorted(host_in[k]).  dev_bufs: >= 2 device tensors of the batch's
    size (3 overlap the sort with both copies), dev_tmp: one more.  radsort_sort_host_stream."""
    assert len(host_in) == len(host_out) and len(host_in) > 0 and len(dev_bufs) >= 2
    n, R = host_in[0].shape
    for t in list(host_in) + list(host_out) + list(dev_bufs) + [dev_tmp]:
        assert tuple(t.shape) == (n, R), "every batch and buffer must have the same [n, R] shape"
    arr = ctypes.c_void_p * len(host_in)
    hin = arr(*[t.data_ptr() for t in host_in])
    hout = arr(*[t.data_ptr() for t in host_out])
    bufs = (ctypes.c_void_p * len(dev_bufs))(*[t.data_ptr() for t in dev_bufs])
    _check(lib.radsort_sort_host_stream(hin, hout, len(host_in), n, R, key_size, bufs, len(dev_bufs),
                                        ctypes.c_void_p(dev_tmp.data_ptr()), _stream_ptr(stream)))


def sort_multi(records, tmp, n_local: int, key_size: int, group=None, stream=None) -> int:
    """Collective multi-GPU sort (one process per GPU); returns this rank's n_out."""
    import torch
    import torch.distributed as dist

    group = group or dist.group.WORLD
    backend = group._get_backend(torch.device("cuda"))
    comm = backend._comm_ptr()
    R = records.shape[1]
    cap = min(records.shape[0], tmp.numel() * tmp.element_size() // R)
    n_out = ctypes.c_uint64(0)
    init(records.device.index)
    _check(lib.radsort_sort_multi(ctypes.c_void_p(records.data_ptr()), ctypes.c_void_p(tmp.data_ptr()), n_local, cap,
                                  ctypes.byref(n_out), R, key_size, ctypes.c_void_p(comm), _stream_ptr(stream)))
    return int(n_out.value)


def comm_unique_id() -> bytes:
    """A new 128-byte NCCL unique id (call on one rank, broadcast to the others)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib.radsort_comm_get_unique_id(buf))
    return buf.raw


def comm_init(unique_id: bytes, nranks: int, rank: int, max_ctas: int = 0) -> int:
    """A library-owned NCCL communicator (ncclComm_t as int) with NCCL's CTAs capped at max_ctas."""
    assert len(unique_id) == 128
    c = ctypes.c_void_p()
    _check(lib.radsort_comm_init(ctypes.create_string_buffer(unique_id, 128), nranks, rank, max_ctas,
                                 ctypes.byref(c)))
    return int(c.value)


def comm_destroy(comm: int) -> None:
    _check(lib.radsort_comm_destroy(ctypes.c_void_p(comm)))


def sort_multi_comm(records, tmp, n_local: int, key_size: int, comm: int, stream=None) -> int:
    """radsort_sort_multi on a communicator from comm_init; returns this rank's n_out."""
    R = records.shape[1]
    cap = min(records.shape[0], tmp.numel() * tmp.element_size() // R)
    n_out = ctypes.c_uint64(0)
    init(records.device.index)
    _check(lib.radsort_sort_multi(ctypes.c_void_p(records.data_ptr()), ctypes.c_void_p(tmp.data_ptr()), n_local, cap,
                                  ctypes.byref(n_out), R, key_size, ctypes.c_void_p(comm), _stream_ptr(stream)))
    return int(n_out.value)


class LoopbackGroup:
    """G in-process ranks on one GPU (host threads), same algorithm as NCCL."""

    def __init__(self, nranks: int):
        self.handle = ctypes.c_void_p()
        _check(lib.radsort_loopback_create(nranks, ctypes.byref(self.handle)))
        self.nranks = nranks

    def sort(self, rank: int, records, tmp, n_local: int, key_size: int, stream=None) -> int:
        R = records.shape[1]
        cap = min(records.shape[0], tmp.numel() * tmp.element_size() // R)
        n_out = ctypes.c_uint64(0)
        _check(lib.radsort_sort_multi_loopback(self.handle, rank, ctypes.c_void_p(records.data_ptr()),
                                               ctypes.c_void_p(tmp.data_ptr()), n_local, cap, ctypes.byref(n_out), R,
                                               key_size, _stream_ptr(stream)))
        return int(n_out.value)

    def close(self):
        if self.handle:
            lib.radsort_loopback_destroy(self.handle)
            self.handle = ctypes.c_void_p()


def plan_quotas(N: int, G: int):
    import numpy as np

    q = np.zeros(G, dtype=np.uint64)
    _check(lib.radsort_plan_quotas(N, G, ctypes.c_void_p(q.ctypes.data)))
    return q


def plan_digit(count_lt256, q: int) -> int:
    import numpy as np

    c = np.ascontiguousarray(count_lt256, dtype=np.uint64)
    d = ctypes.c_uint32(0)
    _check(lib.radsort_plan_digit(ctypes.c_void_p(c.ctypes.data), q, ctypes.byref(d)))
    return int(d.value)


def plan_equal_split(e, L: int, Q: int):
    import numpy as np

    e = np.ascontiguousarray(e, dtype=np.uint64)
    below = np.zeros_like(e)
    _check(lib.radsort_plan_equal_split(ctypes.c_void_p(e.ctypes.data), len(e), L, Q,
                                        ctypes.c_void_p(below.ctypes.data)))
    return below


def plan_fused(all_tables, me: int, piece_dst, piece_bucket):
    """Fused-exchange plan (radsort_plan_fused): all_tables = every rank's dense
    piece histogram table, uint32 [G, G, 256, 256] (sender, receiver, d0 bucket,
    digit d0+1).  Returns (piece_base [npieces, 256], recv_off [65537])."""
    import numpy as np

    t = np.ascontiguousarray(all_tables, dtype=np.uint32)
    G = t.shape[0]
    pd = np.ascontiguousarray(piece_dst, dtype=np.uint32)
    pb = np.ascontiguousarray(piece_bucket, dtype=np.uint32)
    base = np.zeros((len(pd), 256), dtype=np.uint32)
    recv = np.zeros(65537, dtype=np.uint64)
    _check(lib.radsort_plan_fused(ctypes.c_void_p(t.ctypes.data), G, me, len(pd), ctypes.c_void_p(pd.ctypes.data),
                                  ctypes.c_void_p(pb.ctypes.data), ctypes.c_void_p(base.ctypes.data),
                                  ctypes.c_void_p(recv.ctypes.data)))
    return base, recv


def locate_bucket(hist256, q: int):
    import numpy as np

    h = np.ascontiguousarray(hist256, dtype=np.uint64)
    assert h.shape == (256,)
    b = ctypes.c_uint32(0)
    before = ctypes.c_uint64(0)
    _check(lib.radsort_locate_bucket(ctypes.c_void_p(h.ctypes.data), q, ctypes.byref(b), ctypes.byref(before)))
    return int(b.value), int(before.value)


def set_timing(on: bool) -> None:
    _check(lib.radsort_set_timing(1 if on else 0))


def last_stats() -> dict:
    s = Stats()
    _check(lib.radsort_last_stats(ctypes.byref(s)))
    d = {k: getattr(s, k) for k, _ in Stats._fields_ if k not in ("kernel_launches", "kernel_ms", "kernel_bytes")}
    d["kernel_launches"] = {c: int(s.kernel_launches[i]) for i, c in enumerate(KERNEL_CLASSES)}
    d["kernel_ms"] = {c: float(s.kernel_ms[i]) for i, c in enumerate(KERNEL_CLASSES)}
    d["kernel_bytes"] = {c: int(s.kernel_bytes[i]) for i, c in enumerate(KERNEL_CLASSES)}
    return d


def finalize() -> None:
    lib.radsort_finalize()


TINY_ALGOS = {0: "enumeration sort (lane per record)", 1: "warp bitonic network", 2: "warp tail sorter",
              3: "insertion sort (thread per array)"}


def tinybench(rec_size: int, key_size: int, n: int, algo: int, bins: int = 1 << 18) -> float:
    """ns per record of tiny-sorter `algo` on `bins` arrays of n records (radsort_tinybench)."""
    out = ctypes.c_double(0.0)
    _check(lib.radsort_tinybench(rec_size, key_size, n, algo, bins, ctypes.byref(out)))
    return out.value


def unique_count(records, key_size: int, stream=None):
    """Distinct keys and their counts of a sorted (n, R) uint8 CUDA tensor:
    returns (keys: (U, key_size) uint8 tensor, counts: (U,) int32 tensor)."""
    import torch

    n, R = records.shape
    keys = torch.empty((max(n, 1), key_size), dtype=torch.uint8, device=records.device)
    counts = torch.empty((max(n, 1),), dtype=torch.int32, device=records.device)
    out = ctypes.c_uint64(0)
    st = (stream or torch.cuda.current_stream()).cuda_stream
    _check(lib.radsort_unique_count(records.data_ptr(), n, R, key_size, keys.data_ptr(), counts.data_ptr(),
                                    ctypes.byref(out), st))
    return keys[:out.value], counts[:out.value]


def tinysort(records, n: int, algo: int, key_size: int, stream=None):
    """Sort consecutive arrays of n records (a CUDA uint8 tensor [bins * n, R],
    keys of an array sharing their top byte) with tiny sorter `algo`; returns
    the sorted copy (radsort_tinysort)."""
    import torch

    R = records.shape[1]
    out = torch.empty_like(records)
    bins = records.shape[0] // n
    _check(lib.radsort_tinysort(R, key_size, n, algo, ctypes.c_void_p(records.data_ptr()),
                                ctypes.c_void_p(out.data_ptr()), bins, _stream_ptr(stream)))
    return out
