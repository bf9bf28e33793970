"""radsort -- B200-native MSD radix sort of fixed-size records (RADULS2,
arXiv 1703.00687, hot path).  The Python surface is a thin ctypes binding of
libradsort.so; see include/radsort.h for the C ABI and DESIGN.md."""
from .radsort import (  # noqa: F401
    EXPORTS, LIB_PATH, LoopbackGroup, RadsortError, finalize, init, last_stats, lib, locate_bucket, plan_digit,
    plan_equal_split, plan_quotas, set_timing, sort, sort_host, sort_host_stream, sort_multi, sort_ptr, version, TINY_ALGOS, tinybench,
    unique_count, comm_unique_id, comm_init, comm_destroy, sort_multi_comm, tinysort, plan_fused,
)
