"""Seeded synthetic record generator -- host (numpy) mirror.

This module is shared test/bench infrastructure: it produces the *inputs* for
both the CUDA path and the CPU oracle and holds none of the sort's arithmetic.
The device twin is ``datagen/datagen.cu``; for every integer-only distribution
the two are bit-identical (pinned in ``tests/test_datagen.py``).  The Zipf
sampler uses double-precision log/exp on both sides, so a last-ulp libm
difference could in principle flip a sample; large Zipf inputs are therefore
always generated on the device and copied to the host ("Input
recipe").

Counter-based stream (reading R10):
    u(i, w) = mix64(seed + (W*i + w + 1) * GOLDEN)   (mod 2^64)
with mix64 the splitmix64 finalizer, W = 8 words per record for every
distribution except Zipf (W = 32: rejection-inversion attempt j uses word j).
Record i is a pure function of (seed, i), so any sharding generates the same
global array.

Record layout (reading R1, "MSD radix sort with 1 B
digits"): bytes [0, K) hold the key as a K-byte little-endian
unsigned integer (K = 16: low word at +0, high word at +8); bytes [K, R) are
payload.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
W_DEFAULT = 8
W_ZIPF = 32
ZIPF_N = 1 << 32
ZIPF_S = 1.1

# distribution ids (must match datagen.cu)
DISTS = {
    "uniform": 0,     # all key bits uniform
    "uniform40": 1,   # key = u >> 24  (keys < 2^40, top 3 bytes zero) -- config C2
    "zipf": 2,        # key = mix64(k), k ~ Zipf(s=1.1) over [1, 2^32] -- config C3
    "equal": 3,       # every key identical
    "sorted": 4,      # key = i
    "reverse": 5,     # key = 2^64-1-i
    "few": 6,         # 7 distinct keys
    "consttop": 7,    # top 3 bytes fixed non-zero, rest uniform
    "bytes": 8,       # every key byte drawn from {0x00, 0x01, 0xFF}: ties at every digit
    "kmer": 9,        # k-mers (k = 55 / 31) of a 2^22-base pseudo-random reference, 1/64 with one error
}
KMER_L = 1 << 22
PAYLOADS = {"random": 0, "index": 1}

# The five BASELINE.json configurations (seed = 170300687000 + config number).
CONFIGS = {
    "c1": dict(n=1_000_000, R=8, K=8, dist="uniform", payload="random", seed=170300687001),
    "c2": dict(n=200_000_000, R=16, K=8, dist="uniform40", payload="index", seed=170300687002),
    "c3": dict(n=1_000_000_000, R=8, K=8, dist="zipf", payload="random", seed=170300687003),
    "c4": dict(n=1_000_000_000, R=32, K=16, dist="uniform", payload="random", seed=170300687004),
    "c5": dict(n=1_000_000_000, R=8, K=8, dist="uniform", payload="random", seed=170300687005),
}
# The KMC3 consumer workload ("413 M 16 B-key
# records"): a synthetic k-mer stream (the KMC set is not available), sorted then
# run-length counted.  Not one of BASELINE.json's configs.
EXTRA_CONFIGS = {
    "kmc": dict(n=413_000_000, R=16, K=16, dist="kmer", payload="random", seed=170300687006),
}
CONFIGS.update(EXTRA_CONFIGS)


def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def u(seed: int, idx, w: int, W: int = W_DEFAULT):
    """Counter-based uniform 64-bit word w of record idx (idx: uint64 array)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        ctr = np.uint64(W) * idx + np.uint64(w + 1)
        return mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + ctr * GOLDEN)


# ---- Zipf (Hoermann & Derflinger rejection-inversion), double precision ----
# Source: W. Hoermann, G. Derflinger, "Rejection-inversion to generate variates
# from monotone discrete distributions", ACM TOMACS 6(3), 1996; the helper1 /
# helper2 Taylor fallbacks follow the form Apache Commons Math publishes
# (RejectionInversionZipfSampler).  Test/bench input generator only.
def _helper1(x):
    x = np.asarray(x, dtype=np.float64)
    small = np.abs(x) <= 1e-8
    xs = np.where(small, 1.0, x)
    return np.where(small, 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x)), np.log1p(xs) / xs)


def _helper2(x):
    x = np.asarray(x, dtype=np.float64)
    small = np.abs(x) <= 1e-8
    xs = np.where(small, 1.0, x)
    return np.where(small, 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x)), np.expm1(xs) / xs)


def _H(x, s=ZIPF_S):
    lx = np.log(x)
    return _helper2((1.0 - s) * lx) * lx


def _h(x, s=ZIPF_S):
    return np.exp(-s * np.log(x))


def _Hinv(x, s=ZIPF_S):
    t = x * (1.0 - s)
    t = np.maximum(t, -1.0)
    return np.exp(_helper1(t) * x)


def zipf_ranks(seed: int, idx, N: int = ZIPF_N, s: float = ZIPF_S):
    idx = np.asarray(idx, dtype=np.uint64)
    hx1 = float(_H(1.5, s)) - 1.0
    hN = float(_H(N + 0.5, s))
    sconst = 2.0 - float(_Hinv(float(_H(2.5, s)) - float(_h(2.0, s)), s))
    out = np.zeros(idx.shape, dtype=np.uint64)
    done = np.zeros(idx.shape, dtype=bool)
    for j in range(W_ZIPF):
        w = u(seed, idx, j, W_ZIPF)
        U = (w >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        uu = hN + U * (hx1 - hN)
        x = _Hinv(uu, s)
        k = np.floor(x + 0.5)
        k = np.clip(k, 1.0, float(N))
        accept = (k - x <= sconst) | (uu >= _H(k + 0.5, s) - _h(k, s))
        take = ~done & (accept | (j == W_ZIPF - 1))
        out[take] = k[take].astype(np.uint64)
        done |= take
        if done.all():
            break
    return out


def key_words(dist: str, seed: int, idx, K: int):
    """Return list of K/8 uint64 arrays: key word 0 (least significant) .. K/8-1."""
    idx = np.asarray(idx, dtype=np.uint64)
    nw = K // 8
    d = DISTS[dist]
    if d == 0:
        if nw == 1:
            return [u(seed, idx, 0)]
        return [u(seed, idx, 1), u(seed, idx, 0)]
    if d == 1:
        k = u(seed, idx, 0) >> np.uint64(24)
    elif d == 2:
        r = zipf_ranks(seed, idx)
        if nw == 1:
            return [mix64(r)]
        return [mix64(r + np.uint64(1 << 32)), mix64(r)]
    elif d == 3:
        k = np.full(idx.shape, 0x5555AAAA5555AAAA, dtype=np.uint64)
    elif d == 4:
        k = idx.copy()
    elif d == 5:
        k = ~idx
    elif d == 6:
        k = mix64(u(seed, idx, 0) % np.uint64(7))
    elif d == 7:
        k = np.uint64(0xABCDEF << 40) | (u(seed, idx, 0) >> np.uint64(24))
    elif d == 9:  # must match kmer_key in datagen.cu
        k = 55 if nw == 2 else 31
        p = u(seed, idx, 0) % np.uint64(KMER_L)
        e = u(seed, idx, 1)
        err = (e & np.uint64(63)) == 0
        epos = (e >> np.uint64(8)) % np.uint64(k)
        hi = np.zeros(idx.shape, dtype=np.uint64)
        lo = np.zeros(idx.shape, dtype=np.uint64)
        with np.errstate(over="ignore"):
            for j in range(k):
                x = (p + np.uint64(j)) % np.uint64(KMER_L)
                b = mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + GOLDEN * (x + np.uint64(1 << 32))) & np.uint64(3)
                sub = (b + np.uint64(1) + ((e >> np.uint64(16)) % np.uint64(3))) & np.uint64(3)
                b = np.where(err & (epos == np.uint64(j)), sub, b)
                hi = (hi << np.uint64(2)) | (lo >> np.uint64(62))
                lo = (lo << np.uint64(2)) | b
        return [lo] if nw == 1 else [lo, hi]
    elif d == 8:
        words = []
        for kw in range(nw):
            r = u(seed, idx, 4 + kw)
            acc = np.zeros(idx.shape, dtype=np.uint64)
            for b in range(8):
                sel = (r >> np.uint64(8 * b)) & np.uint64(255)
                # 0x00 (prob 86/256), 0x01 (85/256), 0xFF (85/256)
                v = np.where(sel < 86, 0, np.where(sel < 171, 1, 255)).astype(np.uint64)
                acc |= v << np.uint64(8 * b)
            words.append(acc)
        return words
    else:
        raise ValueError(dist)
    if nw == 1:
        return [k]
    # K = 16 for the 64-bit-valued distributions: high word carries the value,
    # low word is a second uniform word (except equal/sorted/reverse: low = value too)
    if d in (3, 4, 5, 6):
        return [k, k]
    return [u(seed, idx, 1), k]


def generate(n: int, R: int, K: int, dist: str = "uniform", payload: str = "random",
             seed: int = 1, first: int = 0) -> np.ndarray:
    """Records [first, first+n) as a (n, R) uint8 array."""
    assert R % 8 == 0 and K % 8 == 0 and 8 <= K <= R <= 64 and K in (8, 16)
    idx = np.arange(first, first + n, dtype=np.uint64)
    words = np.zeros((n, R // 8), dtype=np.uint64)
    kw = key_words(dist, seed, idx, K)
    for j, w in enumerate(kw):
        words[:, j] = w
    for w in range(K // 8, R // 8):
        if PAYLOADS[payload] == 1 and w == K // 8:
            words[:, w] = idx
        else:
            words[:, w] = u(seed, idx, w)
    return words.view(np.uint8).reshape(n, R)


def generate_config(name: str, n: int | None = None, first: int = 0) -> np.ndarray:
    c = CONFIGS[name]
    return generate(n if n is not None else c["n"], c["R"], c["K"], c["dist"], c["payload"], c["seed"], first)
