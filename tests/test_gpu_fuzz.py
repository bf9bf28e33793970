"""Seeded random sweep of (layout, n, distribution, knobs) against the oracle.

Each case draws a record layout, a size (log-uniform up to 3 M records, so
that every size class and level structure occurs), a key distribution, a
payload kind and the optional paths (cluster local sort forced on/off, local
size classes on/off), sorts through the C ABI and compares with the CPU
oracle (identical key sequence, identical multiset inside every equal-key run)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from datagen import host as dg  # noqa: E402
from test_gpu_sort import LAYOUTS, run_gpu_sort  # noqa: E402

DISTS = ["uniform", "uniform40", "zipf", "equal", "sorted", "reverse", "few", "consttop", "bytes", "kmer"]
CASES = 128


def _case(i):
    rng = np.random.default_rng(1703_00687 + i)
    R, K = LAYOUTS[int(rng.integers(len(LAYOUTS)))]
    n = int(np.exp(rng.uniform(0.0, np.log(3_000_000))))
    dist = DISTS[int(rng.integers(len(DISTS)))]
    payload = "index" if R > K and rng.random() < 0.5 else "random"
    cluster = str(int(rng.integers(2)))
    split = str(int(rng.integers(2)))
    return R, K, n, dist, payload, cluster, split, int(rng.integers(1 << 30))


@pytest.fixture(scope="module", autouse=True)
def _init():
    import paper_1703_00687_b200 as rs

    rs.init(0)


@pytest.mark.parametrize("i", range(CASES))
def test_fuzz_case(i, monkeypatch):
    R, K, n, dist, payload, cluster, split, seed = _case(i)
    monkeypatch.setenv("RADSORT_CLUSTER", cluster)
    monkeypatch.setenv("RADSORT_LOCAL_SPLIT", split)
    a = dg.generate(n, R, K, dist, payload=payload, seed=seed)
    got = run_gpu_sort(a, K)
    bad = oracle.compare(got, oracle.sort(a, K), K)
    assert bad == -1, f"case {i}: R={R} K={K} n={n} {dist} {payload} cluster={cluster} split={split}: record {bad}"
