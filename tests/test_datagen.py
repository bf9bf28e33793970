"""Pins for the seeded input generator (host mirror; the device twin is
checked bit-for-bit against it in tests/test_gpu_datagen.py)."""
import numpy as np
import pytest
import scipy.special as sp

from datagen import host as dg


def test_splitmix64_published_sequence():
    # u(seed=0, i=0, w) with W = 8 is the splitmix64 stream seeded with 0
    # (Vigna's reference generator: e220a8397b1dcdaf 6e789e6aa1b965f4 06c45d188009454f)
    i = np.zeros(1, dtype=np.uint64)
    assert int(dg.u(0, i, 0)[0]) == 0xE220A8397B1DCDAF
    assert int(dg.u(0, i, 1)[0]) == 0x6E789E6AA1B965F4
    assert int(dg.u(0, i, 2)[0]) == 0x06C45D188009454F


def test_shard_invariance():
    a = dg.generate(1000, 32, 16, "uniform", seed=77)
    b = np.concatenate([dg.generate(300, 32, 16, "uniform", seed=77, first=0),
                        dg.generate(700, 32, 16, "uniform", seed=77, first=300)])
    assert np.array_equal(a, b)


def test_c2_recipe():
    c = dg.CONFIGS["c2"]
    a = dg.generate_config("c2", n=50000)
    w = a.view(np.uint64).reshape(-1, 2)
    assert np.all(w[:, 0] < (1 << 40))                       # top 3 key bytes zero
    assert np.array_equal(w[:, 1], np.arange(50000, dtype=np.uint64))  # payload = index
    assert c["R"] == 16 and c["K"] == 8


def test_c4_recipe_layout():
    a = dg.generate_config("c4", n=100)
    w = a.view(np.uint64).reshape(-1, 4)
    idx = np.arange(100, dtype=np.uint64)
    seed = dg.CONFIGS["c4"]["seed"]
    assert np.array_equal(w[:, 1], dg.u(seed, idx, 0))  # high word at +8
    assert np.array_equal(w[:, 0], dg.u(seed, idx, 1))  # low word at +0
    assert np.array_equal(w[:, 2], dg.u(seed, idx, 2))


def test_zipf_frequencies_match_closed_form():
    # P(rank k) = k^-s / H(N, s), H(2^32, 1.1) = zeta(1.1) - zeta(1.1, 2^32 + 1) = 9.496260
    H = sp.zeta(1.1) - sp.zeta(1.1, 2.0**32 + 1)
    assert abs(H - 9.496260) < 1e-5
    n = 400000
    r = dg.zipf_ranks(dg.CONFIGS["c3"]["seed"], np.arange(n, dtype=np.uint64))
    assert r.min() >= 1 and r.max() <= 2**32
    for k in (1, 2, 3, 10):
        p = k ** -1.1 / H
        sigma = np.sqrt(p * (1 - p) / n)
        assert abs((r == k).mean() - p) < 5 * sigma, k
    # top-256 mass 0.509893
    p256 = sum(k ** -1.1 for k in range(1, 257)) / H
    assert abs(p256 - 0.509893) < 1e-5
    assert abs((r <= 256).mean() - p256) < 5 * np.sqrt(p256 * (1 - p256) / n)


@pytest.mark.parametrize("dist", list(dg.DISTS))
def test_every_distribution_generates(dist):
    for K, R in ((8, 8), (8, 16), (16, 32)):
        a = dg.generate(257, R, K, dist, seed=1)
        assert a.shape == (257, R)
