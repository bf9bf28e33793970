"""CPU oracle for radsort -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_1703_00687_b200``) never does; it shares no code with it.

Functions (each documented in oracle_sort.cpp with the PAPER.md / SPEC.md
passage it follows):

- ``sort(records, K)``            stable comparison sort on the K-byte key
- ``sort_parallel(records, K, T)``  the same on T host cores (chunks + merge rounds; the all-cores CPU baseline)
- ``digit(record, K, d)``         digit d (0 = most significant byte)
- ``digit_hist(records, K, d)``   256-bin histogram of digit d
- ``key_compare(a, b, K)``        -1 / 0 / +1
- ``compare(got, want, K)``       canonical parity check (-1 = equal)
- ``rank_bounds(records, K, key)`` (#keys < k, #keys <= k): sampled full-size checks
- ``unique_count(sorted, K)``     distinct keys + counts (the KMC3 consumer)

Pins: tests/test_oracle.py (brute force, numpy/lexsort special cases, SPEC
worked examples in tests/golden/).  Parity pinned for every function above.
"""
from .oracle import sort, sort_parallel, digit, digit_hist, key_compare, compare, rank_bounds, unique_count, lib_path, build  # noqa: F401
