"""Pins for the CPU oracle (no GPU).  The oracle is checked against things
other than itself: the SPEC/PAPER worked examples (tests/golden/), numpy's
sort and lexsort (library special cases), brute force over every ordering of
tiny inputs, and the invariants sortedness / permutation / stability."""
import itertools
import os

import numpy as np
import pytest

import oracle
from datagen import host as dg


def rec_from_hex(h: str, K: int, R: int | None = None) -> np.ndarray:
    R = R or K
    v = int(h, 16)
    b = v.to_bytes(K, "little") + bytes(R - K)
    return np.frombuffer(b, dtype=np.uint8).copy()


def key_int(rec: np.ndarray, K: int) -> int:
    return int.from_bytes(bytes(rec[:K]), "little")


def load_golden(golden_dir):
    rows = []
    with open(os.path.join(golden_dir, "spec_examples.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line.split())
    return rows


def test_golden_examples(golden_dir):
    rows = load_golden(golden_dir)
    assert len(rows) >= 10
    for r in rows:
        kind, K = r[0], int(r[1])
        if kind == "digit":
            assert oracle.digit(rec_from_hex(r[2], K), K, int(r[3])) == int(r[4], 16), r
        elif kind == "cmp":
            assert oracle.key_compare(rec_from_hex(r[2], K), rec_from_hex(r[3], K), K) == int(r[4]), r
        elif kind == "hist":
            recs = np.stack([rec_from_hex(h, K) for h in r[2].split(",")])
            h = oracle.digit_hist(recs, K, int(r[3]))
            want = np.zeros(256, dtype=np.uint64)
            for kv in r[4].split(","):
                k, v = kv.split(":")
                want[int(k, 16)] = int(v)
            assert np.array_equal(h, want), r
        elif kind == "sort":
            recs = np.stack([rec_from_hex(h, K) for h in r[2].split(",")])
            want = np.stack([rec_from_hex(h, K) for h in r[4].split(",")])
            assert np.array_equal(oracle.sort(recs, K), want), r
        else:
            raise AssertionError(kind)


def test_identical_keys_different_payload_compare_equal():
    # payload never participates in the comparison
    a = rec_from_hex("0000000000000007", 8, 16)
    b = a.copy()
    b[8:] = 0xAB
    assert oracle.key_compare(a, b, 8) == 0


@pytest.mark.parametrize("dist", ["uniform", "bytes", "few", "sorted", "reverse", "equal", "uniform40"])
def test_matches_numpy_sort_r8(dist):
    # R = K = 8: the key sequence must equal numpy.sort of the uint64 keys
    a = dg.generate(5000, 8, 8, dist, seed=11)
    out = oracle.sort(a, 8)
    keys = a.view(np.uint64).reshape(-1)
    assert np.array_equal(out.view(np.uint64).reshape(-1), np.sort(keys))


@pytest.mark.parametrize("dist", ["uniform", "bytes", "few", "zipf"])
def test_matches_lexsort_k16(dist):
    # K = 16: high word at +8 decides, then the low word (np.lexsort: last key primary)
    a = dg.generate(3000, 32, 16, dist, seed=5)
    out = oracle.sort(a, 16)
    w = a.view(np.uint64).reshape(-1, 4)
    order = np.lexsort((w[:, 0], w[:, 1]))
    o = out.view(np.uint64).reshape(-1, 4)
    assert np.array_equal(o[:, :2], w[order][:, :2])
    # permutation: same multiset of full records
    assert sorted(map(bytes, out)) == sorted(map(bytes, a))


def test_stability_and_permutation_c2_like():
    # payload = original index (C2 recipe): strictly increasing inside equal-key runs
    a = dg.generate(20000, 16, 8, "few", payload="index", seed=3)
    out = oracle.sort(a, 8)
    w = out.view(np.uint64).reshape(-1, 2)
    k, p = w[:, 0], w[:, 1]
    assert np.all(k[1:] >= k[:-1])
    same = k[1:] == k[:-1]
    assert np.all(p[1:][same] > p[:-1][same])
    assert np.array_equal(np.sort(p), np.arange(20000, dtype=np.uint64))


ALPHABETS = {
    8: [0, 1, 2**63, 2**64 - 1, 0x0100000000000000, 0x00000000000000FF],
    16: [0, 1, 2**64, 2**64 + 1, (2**64 - 1), 2**127, 2**128 - 1],
}


@pytest.mark.parametrize("K,R", [(8, 8), (8, 16), (16, 16), (16, 32)])
def test_brute_force_all_orderings(K, R):
    rng = np.random.default_rng(7 + K + R)
    for n in range(0, 7):
        for trial in range(4 if n > 1 else 1):
            alpha = ALPHABETS[K]
            keys = [alpha[int(rng.integers(len(alpha)))] for _ in range(n)]
            recs = []
            for j, kv in enumerate(keys):
                b = kv.to_bytes(K, "little") + bytes([j + 1]) * (R - K)
                recs.append(np.frombuffer(b, dtype=np.uint8))
            base = np.stack(recs) if n else np.zeros((0, R), dtype=np.uint8)
            # brute force: all orderings whose key sequence is non-decreasing
            valid = set()
            for perm in itertools.permutations(range(n)):
                ks = [keys[i] for i in perm]
                if all(ks[i] <= ks[i + 1] for i in range(n - 1)):
                    valid.add(tuple(bytes(base[i]) for i in perm))
            assert valid
            want_keys = sorted(keys)
            for perm in itertools.permutations(range(n)):
                x = base[list(perm)] if n else base
                out = oracle.sort(x, K)
                assert [key_int(r, K) for r in out] == want_keys
                assert tuple(bytes(r) for r in out) in valid
                if R == K:
                    continue
                # stable: equal keys keep their input order
                pos = {bytes(x[i]): i for i in range(n)}
                for i in range(n - 1):
                    if key_int(out[i], K) == key_int(out[i + 1], K):
                        assert pos[bytes(out[i])] < pos[bytes(out[i + 1])]


def test_edge_sizes():
    for n in (0, 1, 2):
        a = dg.generate(n, 16, 8, "uniform", seed=2)
        out = oracle.sort(a, 8)
        assert out.shape == a.shape
        if n == 2:
            k = a.view(np.uint64).reshape(-1, 2)[:, 0]
            assert out.view(np.uint64).reshape(-1, 2)[0, 0] == k.min()


@pytest.mark.parametrize("K", [8, 16])
def test_digit_hist_closed_form(K):
    a = dg.generate(4000, 32, K, "bytes", seed=9)
    w = a.view(np.uint64).reshape(-1, 4)
    for d in range(K):
        word = w[:, (K - 1 - d) // 8]
        shift = 8 * ((K - 1 - d) % 8)
        want = np.bincount(((word >> np.uint64(shift)) & np.uint64(255)).astype(np.int64), minlength=256)
        assert np.array_equal(oracle.digit_hist(a, K, d), want.astype(np.uint64))


def test_constant_top_digits_c2_recipe():
    # C2: keys < 2^40 so digits 0..2 are constant (hist[d][0] == n)
    a = dg.generate(10000, 16, 8, "uniform40", payload="index", seed=dg.CONFIGS["c2"]["seed"])
    for d in range(3):
        h = oracle.digit_hist(a, 8, d)
        assert h[0] == 10000
    assert oracle.digit_hist(a, 8, 3).max() < 10000


def test_compare_canonical():
    a = dg.generate(3000, 16, 8, "few", payload="index", seed=4)
    want = oracle.sort(a, 8)
    assert oracle.compare(want, want, 8) == -1
    # permuting records inside an equal-key run is still a correct result
    got = want.copy()
    k = got.view(np.uint64).reshape(-1, 2)[:, 0]
    i = int(np.argmax(k[1:] == k[:-1]))
    got[[i, i + 1]] = got[[i + 1, i]]
    assert oracle.compare(got, want, 8) == -1
    # a corrupted payload inside a run is caught
    bad = got.copy()
    bad[i, 12] ^= 1
    assert oracle.compare(bad, want, 8) >= 0
    # swapping two different keys is caught at the first differing position
    j = int(np.argmax(k[1:] != k[:-1]))
    bad2 = want.copy()
    bad2[[j, j + 1]] = bad2[[j + 1, j]]
    assert oracle.compare(bad2, want, 8) == j


def test_rank_bounds_against_sorted_positions():
    a = dg.generate(5000, 16, 8, "few", payload="index", seed=8)
    s = oracle.sort(a, 8)
    keys = s.view(np.uint64).reshape(-1, 2)[:, 0]
    for i in (0, 1, 77, 2500, 4999):
        lt, le = oracle.rank_bounds(a, 8, s[i])
        assert lt == int(np.searchsorted(keys, keys[i], "left"))
        assert le == int(np.searchsorted(keys, keys[i], "right"))
        assert lt <= i < le


def test_unique_count_pinned_to_counter():
    # pinned to an independent method: collections.Counter over key bytes, on
    # oracle-sorted tie-heavy inputs (every run found, counts exact, key order)
    import collections

    for K, R in ((8, 8), (8, 16), (16, 32)):
        a = dg.generate(5000, R, K, "few" if K == 8 else "bytes", seed=5)
        s = oracle.sort(a, K)
        keys, counts = oracle.unique_count(s, K)
        c = collections.Counter(bytes(r[:K]) for r in a)
        assert len(keys) == len(c) and int(counts.sum()) == 5000
        for k, m in zip(keys, counts):
            assert c[bytes(k)] == m
        # keys strictly increasing as K-byte little-endian integers
        vals = [int.from_bytes(bytes(k), "little") for k in keys]
        assert all(x < y for x, y in zip(vals, vals[1:]))
    z = oracle.unique_count(np.zeros((0, 8), dtype=np.uint8), 8)
    assert z[0].shape == (0, 8) and z[1].shape == (0,)


def _kmer_reference(seed, idx, K):
    # independent pure-Python restatement of the k-mer recipe (datagen "kmer")
    mask = (1 << 64) - 1

    def mix(z):
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9 & mask
        z = (z ^ (z >> 27)) * 0x94D049BB133111EB & mask
        return z ^ (z >> 31)

    def uw(i, w):
        return mix((seed + (8 * i + w + 1) * 0x9E3779B97F4A7C15) & mask)

    k = 55 if K == 16 else 31
    L = 1 << 22
    p, e = uw(idx, 0) % L, uw(idx, 1)
    bases = [mix((seed + 0x9E3779B97F4A7C15 * ((p + j) % L + (1 << 32))) & mask) & 3 for j in range(k)]
    if e & 63 == 0:
        j = (e >> 8) % k
        bases[j] = (bases[j] + 1 + ((e >> 16) % 3)) & 3
    v = 0
    for b in bases:
        v = (v << 2) | b
    return v


def test_kmer_stream_matches_its_definition():
    # the k-mer generator (KMC3 stand-in) against a pure-Python restatement:
    # 2 bits per base, first base most significant, 1/64 records with one error
    for K in (8, 16):
        a = dg.generate(300, 16 if K == 8 else 32, K, "kmer", seed=11)
        for i in (0, 1, 7, 63, 299):
            got = int.from_bytes(bytes(a[i, :K]), "little")
            assert got == _kmer_reference(11, i, K)
        # unique keys + counts of a small stream against a Counter over the
        # pure-Python keys (independent of the generator and of the oracle)
        import collections

        m = 1500
        b = dg.generate(m, K, K, "kmer", seed=12)
        want = collections.Counter(_kmer_reference(12, i, K) for i in range(m))
        keys, counts = oracle.unique_count(oracle.sort(b, K), K)
        got = {int.from_bytes(bytes(k), "little"): int(c) for k, c in zip(keys, counts)}
        assert got == dict(want)
        # overlapping reads of a 2^22-base reference: ~48 repeated read positions
        # among 20000 reads, so some k-mer occurs at least twice
        big = dg.generate(20000, K, K, "kmer", seed=12)
        _, counts = oracle.unique_count(oracle.sort(big, K), K)
        assert counts.max() >= 2 and counts.sum() == 20000


@pytest.mark.parametrize("R,K", [(8, 8), (16, 8), (32, 16)])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_parallel_sort_is_the_stable_sort(R, K, threads):
    # pinned to numpy's stable lexsort (key words, high first; ties by input
    # position): the stable order is unique, so the bytes must match exactly
    for dist, n in (("few", 20011), ("uniform", 50000), ("bytes", 7)):
        a = dg.generate(n, R, K, dist, payload="index" if R > K else "random", seed=n)
        w = a.view(np.uint64).reshape(n, R // 8)
        order = np.lexsort(tuple([np.arange(n)] + [w[:, j] for j in range(K // 8)]))
        got = oracle.sort_parallel(a, K, threads)
        assert np.array_equal(got, a[order])
