"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Every case: seeded synthetic input -> radsort_sort on cuda:0 -> copy back ->
oracle.compare(gpu, oracle.sort(input)) == -1 (identical key sequence and
identical record multiset inside every equal-key run).  Sizes span several
tiles, ragged tails, every size-class boundary (tiny <= 128, local capacity
C, tile T) and the degenerate distributions.  Red zones around both buffers
check write containment (SPEC.md:318/331 analog)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from datagen import host as dg  # noqa: E402

LAYOUTS = [(8, 8), (16, 8), (16, 16), (24, 8), (24, 16), (32, 8), (32, 16), (40, 16)]
GUARD = 4096
POISON = 0xA5


def C_of(R):
    return 131072 // R


def T_of(R):
    return (32768 // R) // 256 * 256  # default scatter tile (RADSORT_SCATTER_CFG=1): a multiple of 256 records


def run_gpu_sort(a: np.ndarray, K: int, guard=True):
    import paper_1703_00687_b200 as rs

    n, R = a.shape
    nb = n * R
    dev = torch.device("cuda", 0)
    big = torch.full((GUARD + max(nb, 16) + GUARD,), POISON, dtype=torch.uint8, device=dev)
    big2 = torch.full((GUARD + max(nb, 16) + GUARD,), POISON, dtype=torch.uint8, device=dev)
    rec = big[GUARD:GUARD + nb]
    tmp = big2[GUARD:GUARD + max(nb, 16)]
    if nb:
        rec.copy_(torch.from_numpy(a.reshape(-1)))
    rs.sort_ptr(rec.data_ptr(), tmp.data_ptr(), n, R, K, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    if guard:
        for b, size in ((big, nb), (big2, max(nb, 16))):
            assert bool((b[:GUARD] == POISON).all()), "write below buffer"
            assert bool((b[GUARD + size:] == POISON).all()), "write above buffer"
    return rec.cpu().numpy().reshape(n, R)


def check(a, K):
    got = run_gpu_sort(a, K)
    want = oracle.sort(a, K)
    bad = oracle.compare(got, want, K)
    assert bad == -1, f"mismatch at record {bad} (n={a.shape[0]}, R={a.shape[1]}, K={K})"


@pytest.fixture(scope="module", autouse=True)
def _init():
    import paper_1703_00687_b200 as rs

    rs.init(0)
    yield


@pytest.mark.parametrize("R,K", LAYOUTS)
@pytest.mark.parametrize("n", [0, 1, 2, 3, 31, 32, 33, 64, 65, 127, 128, 129, 255, 256, 257, 1000, 4097])
def test_small_sizes(R, K, n):
    check(dg.generate(n, R, K, "uniform", seed=1000 + n), K)


@pytest.mark.parametrize("R,K", LAYOUTS)
def test_capacity_and_tile_boundaries(R, K):
    C, T = C_of(R), T_of(R)
    for n in (C - 1, C, C + 1, T - 1, T + 1, 3 * T + 17, 2 * 65536 // R + 5):
        check(dg.generate(n, R, K, "uniform", seed=n), K)


@pytest.mark.parametrize("cfg", ["0", "2", "3", "4"])
def test_other_tile_configs(cfg, monkeypatch):
    # every scatter/histogram tile configuration and the look-back variant stay exact
    monkeypatch.setenv("RADSORT_SCATTER_CFG", cfg)
    for R, K in ((8, 8), (16, 8), (24, 8), (32, 16), (40, 16)):
        check(dg.generate(400_003, R, K, "uniform", seed=11), K)
        check(dg.generate(200_001, R, K, "few", payload="index" if R > K else "random", seed=12), K)
    monkeypatch.setenv("RADSORT_LOOKBACK", "1")
    for R, K in ((8, 8), (16, 8), (24, 16), (32, 16)):
        check(dg.generate(400_003, R, K, "zipf", seed=13), K)


@pytest.mark.parametrize("tma", ["0", "1", "2"])
def test_scatter_write_out_paths(tma, monkeypatch):
    # the radix pass's write-out: coalesced plain stores (0) or one bulk copy per digit run (1: R = 16, 32;
    # 2: every R); R = 8, 24, 40 stage each run at the parity of its HBM slot and store an odd head / tail
    # record by hand -- odd and even run starts / lengths everywhere in these inputs
    monkeypatch.setenv("RADSORT_SCATTER_TMA", tma)
    for R, K in LAYOUTS:
        for n, dist in ((400_003, "uniform"), (300_001, "zipf"), (250_001, "few"), (700_001, "bytes")):
            check(dg.generate(n, R, K, dist, payload="index" if R > K else "random", seed=n + R), K)


@pytest.mark.parametrize("R,K", LAYOUTS)
@pytest.mark.parametrize("dist", ["uniform", "uniform40", "zipf", "equal", "sorted", "reverse", "few", "consttop",
                                  "bytes"])
def test_distributions(R, K, dist):
    for n in (5000, 300_000):
        payload = "index" if R > K else "random"
        check(dg.generate(n, R, K, dist, payload=payload, seed=77), K)


@pytest.mark.parametrize("R,K", [(8, 8), (16, 8), (32, 16)])
def test_multi_level_large(R, K):
    # several Large levels, many tiles per segment, ragged tails everywhere
    n = 2_000_003 if R <= 16 else 1_000_003
    check(dg.generate(n, R, K, "uniform", seed=5), K)
    check(dg.generate(n // 2, R, K, "bytes", seed=6), K)


def test_c1_full_size_against_oracle():
    a = dg.generate_config("c1")
    check(a, 8)


def test_repeated_calls_and_streams():
    import paper_1703_00687_b200 as rs

    a = dg.generate(100_000, 16, 8, "few", payload="index", seed=3)
    want = oracle.sort(a, 8)
    s = torch.cuda.Stream()
    for _ in range(3):
        rec = torch.from_numpy(a.copy()).cuda()
        tmp = torch.empty_like(rec)
        with torch.cuda.stream(s):
            rs.sort(rec, tmp, 8)
        s.synchronize()
        assert oracle.compare(rec.cpu().numpy(), want, 8) == -1


def test_sort_host_end_to_end():
    import paper_1703_00687_b200 as rs

    a = dg.generate(300_000, 32, 16, "uniform", seed=9)
    h = torch.from_numpy(a.copy()).pin_memory()
    rs.sort_host(h, 16)
    assert oracle.compare(h.numpy(), oracle.sort(a, 16), 16) == -1


@pytest.mark.parametrize("nbuf", [2, 3])
@pytest.mark.parametrize("R,K,n", [(32, 16, 300_001), (8, 8, 1_000_003), (16, 8, 70_000), (24, 8, 5)])
def test_sort_host_stream_pipelined_batches(nbuf, R, K, n):
    # radsort_sort_host_stream: every batch a different input (distribution and seed),
    # batch k staged in buffer k % nbuf, copies overlapped with the sorts; each
    # output against the oracle, and the in-place form (host_out = host_in)
    import paper_1703_00687_b200 as rs

    dists = ["uniform", "zipf", "few", "sorted", "equal"]
    ins = [dg.generate(n, R, K, dists[k], seed=100 + k) for k in range(5)]
    h_in = [torch.from_numpy(a.copy()).pin_memory() for a in ins]
    h_out = [torch.empty_like(h).pin_memory() for h in h_in]
    dev = torch.device("cuda", 0)
    bufs = [torch.full((n, R), POISON, dtype=torch.uint8, device=dev) for _ in range(nbuf)]
    tmp = torch.empty((n, R), dtype=torch.uint8, device=dev)
    rs.sort_host_stream(h_in, h_out, K, bufs, tmp)
    for k, a in enumerate(ins):
        assert oracle.compare(h_out[k].numpy(), oracle.sort(a, K), K) == -1, f"batch {k}"
        assert np.array_equal(h_in[k].numpy(), a), "input batch modified"
    rs.sort_host_stream(h_in[:3], h_in[:3], K, bufs, tmp)  # in place
    for k in range(3):
        assert oracle.compare(h_in[k].numpy(), oracle.sort(ins[k], K), K) == -1, f"in-place batch {k}"


def test_sort_host_stream_rejects_bad_arguments():
    import paper_1703_00687_b200 as rs

    h = torch.zeros((100, 8), dtype=torch.uint8).pin_memory()
    d = torch.zeros((100, 8), dtype=torch.uint8, device="cuda")
    with pytest.raises(AssertionError):
        rs.sort_host_stream([h], [h], 8, [d], d)  # one device buffer
    with pytest.raises(rs.RadsortError):
        rs.sort_host_stream([h], [h], 3, [d, d.clone()], d.clone())  # K = 3


def test_device_datagen_matches_host_mirror():
    from datagen import device as dd

    for dist in ("uniform", "uniform40", "equal", "sorted", "reverse", "few", "consttop", "bytes"):
        for R, K in ((8, 8), (16, 8), (32, 16)):
            h = dg.generate(4099, R, K, dist, payload="index", seed=42, first=123)
            d = dd.generate_tensor(4099, R, K, dist, payload="index", seed=42, first=123).cpu().numpy()
            assert np.array_equal(h, d), (dist, R, K)
    # Zipf: double-precision log/exp on both sides; allow a vanishing ulp-level disagreement
    h = dg.generate(200_000, 8, 8, "zipf", seed=3)
    d = dd.generate_tensor(200_000, 8, 8, "zipf", seed=3).cpu().numpy()
    assert (h != d).any(axis=1).mean() < 1e-4


def test_stats_report_constant_digit_skip():
    import paper_1703_00687_b200 as rs

    a = dg.generate_config("c2", n=1_000_000)
    got = run_gpu_sort(a, 8, guard=False)
    st = rs.last_stats()
    assert st["first_digit"] == 3            # digits 0..2 constant (keys < 2^40)
    w = got.view(np.uint64).reshape(-1, 2)
    assert np.all(w[1:, 0] >= w[:-1, 0])
    assert np.array_equal(np.sort(w[:, 1]), np.arange(1_000_000, dtype=np.uint64))


def _dominate(a: np.ndarray, K: int, frac_num: int, frac_den: int, key_words, offset: int = 0):
    """Overwrite the key of frac_num out of every frac_den records (from `offset`) with key_words."""
    w = a.view(np.uint64).reshape(a.shape[0], -1)
    for j in range(frac_num):
        for k, kw in enumerate(key_words):
            w[offset + j::frac_den, k] = np.uint64(kw)
    return a


@pytest.mark.parametrize("R,K", LAYOUTS)
@pytest.mark.parametrize("n", [40_000, 300_001, 2_000_003])
def test_dominant_key_split(R, K, n):
    # a key holding 60 % of the records dominates the level-0 segment and its
    # level-1 bin; a second key with 25 % shares its top byte (nested split);
    # the rest uniform.  Exercises the three-way split with the equal run
    # written to `records` (segment in tmp) and skipped + filled (R == K,
    # segment in `records`), and the below/above remainders at the same depth.
    import paper_1703_00687_b200 as rs

    a = dg.generate(n, R, K, "uniform", payload="index" if R > K else "random", seed=n + R)
    top = [0x5A00_1234_5678_9ABC] if K == 8 else [0x0123_4567_89AB_CDEF, 0x5A00_1234_5678_9ABC]
    sec = [0x5A77_0000_0000_0001] if K == 8 else [0x0, 0x5A77_0000_0000_0001]
    _dominate(a, K, 3, 5, top)
    _dominate(a, K, 1, 8, sec, offset=3)
    check(a, K)
    st = rs.last_stats()
    if n >= 300_001:
        assert st["bins_split"] >= 1 and st["records_split"] > 0


def test_dominant_key_split_zipf_stats():
    # Zipf keys (c3 recipe): heavy keys are split off, and the result is exact
    import paper_1703_00687_b200 as rs

    a = dg.generate(3_000_000, 8, 8, "zipf", seed=99)
    check(a, 8)
    st = rs.last_stats()
    assert st["bins_split"] >= 1


@pytest.mark.parametrize("R,K", [(8, 8), (16, 8), (16, 16), (32, 8), (32, 16)])
@pytest.mark.parametrize("algo", [0, 1, 2, 3])
def test_tiny_sorters_match_oracle(R, K, algo):
    # each tiny sorter of the tail (ES, warp bitonic network, warp tail sorter,
    # insertion sort) against the oracle, array by array, on tie-heavy keys
    # sharing their top byte (the sorters' contract: a bin below the top level)
    import paper_1703_00687_b200 as rs

    for n in (2, 3, 5, 16, 17, 31, 32, 33, 64, 100, 128):
        if algo == 0 and n > 32:
            continue
        bins = 48
        for dist in ("bytes", "few", "uniform"):
            a = dg.generate(bins * n, R, K, dist, payload="index" if R > K else "random", seed=n * 7 + algo)
            w = a.view(np.uint64).reshape(bins * n, R // 8)
            hi = K // 8 - 1
            w[:, hi] = (w[:, hi] & np.uint64(0x00FF_FFFF_FFFF_FFFF)) | np.uint64(0x4200_0000_0000_0000)
            got = rs.tinysort(torch.from_numpy(a).cuda(), n, algo, K)
            torch.cuda.synchronize()
            g = got.cpu().numpy()
            for b in range(bins):
                seg = a[b * n:(b + 1) * n]
                bad = oracle.compare(g[b * n:(b + 1) * n], oracle.sort(seg, K), K)
                assert bad == -1, f"algo {algo} n {n} {dist} bin {b}: record {bad}"


@pytest.mark.parametrize("R,K", [(8, 8), (16, 8), (32, 16)])
def test_tinybench_sorters_are_correct(R, K):
    # every tiny sorter sorts every array (the device check inside raises otherwise)
    import paper_1703_00687_b200 as rs

    for n in (2, 3, 17, 32, 33, 64, 65, 100, 128):
        for algo in (0, 1, 2, 3):
            if algo == 0 and n > 32:
                continue
            assert rs.tinybench(R, K, n, algo, bins=4096) > 0.0


@pytest.mark.parametrize("R,K", [(16, 16), (24, 8), (32, 16), (8, 8)])
def test_kmer_sort_and_unique_count(R, K):
    # NEXT-4, the KMC3 consumer: sort a k-mer stream, then run-length count it
    # on the GPU; keys and counts must equal the oracle's
    import paper_1703_00687_b200 as rs

    for n in (1, 2, 4097, 300_001):
        a = dg.generate(n, R, K, "kmer", payload="index" if R > K else "random", seed=n)
        got = run_gpu_sort(a, K, guard=False)
        assert oracle.compare(got, oracle.sort(a, K), K) == -1
        t = torch.from_numpy(got.copy()).cuda()
        keys, counts = rs.unique_count(t, K)
        wk, wc = oracle.unique_count(got, K)
        assert np.array_equal(keys.cpu().numpy(), wk)
        assert np.array_equal(counts.cpu().numpy().astype(np.int64), wc)


def test_kmer_device_generator_matches_host():
    from datagen import device as dd

    for R, K in ((16, 16), (8, 8)):
        h = dg.generate(5000, R, K, "kmer", seed=3, first=77)
        d = dd.generate_tensor(5000, R, K, "kmer", seed=3, first=77).cpu().numpy()
        assert np.array_equal(h, d)


def _top_word(a: np.ndarray, K: int):
    w = a.view(np.uint64).reshape(a.shape[0], -1)
    return w, K // 8 - 1  # the most significant key word


@pytest.fixture
def force_cluster(monkeypatch):
    # the cluster local sort is on by default for R >= 24 only; force it for every layout
    monkeypatch.setenv("RADSORT_CLUSTER", "1")


@pytest.mark.parametrize("R,K", LAYOUTS)
def test_cluster_local_bins(R, K, force_cluster):
    # level-0 bins of ~2.8 C records (2.5 C <= len <= the cluster capacity): sorted
    # by the 4-CTA cluster local sort (k_local_cluster), with a ragged tail
    import paper_1703_00687_b200 as rs

    n = 256 * (C_of(R) * 14 // 5) + 77
    check(dg.generate(n, R, K, "uniform", payload="index" if R > K else "random", seed=R * 3 + K), K)
    assert rs.last_stats()["scatter_passes"] == 1  # every level-0 bin was sorted on chip


@pytest.mark.parametrize("R,K", [(16, 8), (32, 16)])
def test_cluster_off_matches(R, K, monkeypatch):
    monkeypatch.setenv("RADSORT_CLUSTER", "0")
    n = 256 * (C_of(R) * 14 // 5) + 77
    check(dg.generate(n, R, K, "uniform", payload="index" if R > K else "random", seed=R * 5 + K), K)


@pytest.mark.parametrize("R,K,dw", [(24, 8, "1"), (32, 16, "0"), (32, 8, "1"), (40, 16, "1")])
def test_cluster_direct_write_variants(R, K, dw, force_cluster, monkeypatch):
    # the direct-write cluster sort (records from registers straight to their
    # output slots, colliding buckets fixed up in global memory) and the staged
    # one, each on the layouts the other one is the default for
    monkeypatch.setenv("RADSORT_CLUSTER_DW", dw)
    n = 256 * (C_of(R) * 14 // 5) + 77
    for dist in ("uniform", "few", "bytes"):
        check(dg.generate(n, R, K, dist, payload="index" if R > K else "random", seed=R + K), K)


@pytest.mark.parametrize("R,K,dw", [(8, 8, "0"), (16, 16, "0"), (32, 16, "1"), (32, 16, "0"), (24, 8, "1")])
@pytest.mark.parametrize("mode", ["one_slice", "constant", "split_slices"])
def test_cluster_local_bins_handed_back(R, K, dw, mode, force_cluster, monkeypatch):
    # the same bin sizes with a skewed digit 1: "one_slice" (digit 1 < 16: every
    # record of a bin lands in one CTA's bucket slice) and "constant" (digits
    # 1-2 constant: the composite digit is constant) make the cluster sort hand
    # the bins back to the next level's Large list; "split_slices" (half the
    # records share digits 1-2 = 0x92 0x34, the rest digit 1 < 16) fits, leaving
    # one huge colliding bucket for the next Local level.  Exact in all cases.
    # (The direct-write variant, dw = 1, has no staging capacity: it sorts the
    # "one_slice" bins itself.)
    monkeypatch.setenv("RADSORT_CLUSTER_DW", dw)
    n = 256 * (C_of(R) * 14 // 5) + 5
    a = dg.generate(n, R, K, "uniform", payload="index" if R > K else "random", seed=11)
    w, t = _top_word(a, K)
    keep_top = np.uint64(0xFF00_00FF_FFFF_FFFF)
    if mode == "one_slice":
        w[:, t] &= np.uint64(0xFF0F_FFFF_FFFF_FFFF)
    elif mode == "constant":
        w[:, t] = (w[:, t] & keep_top) | np.uint64(0x0012_3400_0000_0000)
    else:
        w[::2, t] &= np.uint64(0xFF0F_FFFF_FFFF_FFFF)
        w[1::2, t] = (w[1::2, t] & keep_top) | np.uint64(0x0092_3400_0000_0000)
    check(a, K)


@pytest.mark.parametrize("R,K", [(8, 8), (16, 16), (32, 16), (24, 8)])
@pytest.mark.parametrize("per_bin", [20, 100, 128])
def test_tail_sorter_dominant_key_pivot(R, K, per_bin):
    # tiny bins (<= 128 records, the warp tail sorter) made of many copies of
    # one key plus a few keys that differ only in the last byte, above and
    # below it: the pivot three-way path of the tail sorter's ES
    n = 256 * per_bin
    a = dg.generate(n, R, K, "uniform", payload="index" if R > K else "random", seed=per_bin + R)
    w, t = _top_word(a, K)
    top = w[:, t] & np.uint64(0xFF00_0000_0000_0000)
    w[:, t] = top | np.uint64(0x0012_3456_789A_BC80)
    if K == 16:
        w[:, 0] = np.uint64(0x1111_2222_3333_4480)
    rng = np.random.default_rng(per_bin)
    odd = rng.random(n) < 0.08
    low = rng.integers(0, 256, n).astype(np.uint64)
    w[odd, 0] = (w[odd, 0] & ~np.uint64(0xFF)) | low[odd]
    check(a, K)


@pytest.mark.parametrize("R,K", [(8, 8), (16, 16), (32, 16)])
@pytest.mark.parametrize("split", ["1", "0"])
@pytest.mark.parametrize("mix", ["small", "medium"])
def test_local_size_classes(R, K, split, mix, monkeypatch):
    # level-0 bins of two size classes, 160 of the smaller (more than one per
    # SM) and 96 large ones (<= C): small (<= 64 x 256 B / R records) or medium
    # (<= 256 x ceil(C / 512)) bins are then sorted by a launch of their own
    # that the large configuration skips (RADSORT_LOCAL_SPLIT=0: one launch)
    monkeypatch.setenv("RADSORT_LOCAL_SPLIT", split)
    C = C_of(R)
    small = {8: 1024, 16: 1024, 32: 512}[R]
    med = 256 * ((C + 511) // 512)
    lo = small // 2 if mix == "small" else (small + med) // 2
    hi = (med + C) // 2 if mix == "medium" or R != 32 else (small + med) // 2
    sizes = [lo if b % 8 < 5 else hi for b in range(256)]
    n = int(sum(sizes))
    a = dg.generate(n, R, K, "uniform", payload="index" if R > K else "random", seed=R + 5)
    w, t = _top_word(a, K)
    top = np.repeat(np.arange(256, dtype=np.uint64), sizes)
    w[:, t] = (w[:, t] & np.uint64(0x00FF_FFFF_FFFF_FFFF)) | (top << np.uint64(56))
    check(a, K)
    import paper_1703_00687_b200 as rs

    launches = rs.last_stats()["kernel_launches"]["local"]
    assert launches == (2 if split == "1" else 1), launches


@pytest.mark.parametrize("R,K", [(8, 8), (16, 8), (16, 16), (32, 16)])
@pytest.mark.parametrize("dist", ["sorted", "reverse"])
def test_level0_digit_guess_too_deep(R, K, dist):
    """The level-0 digit is guessed from a strided sample (k_sample); when the
    sample misses the only records that differ in a higher digit, k_plan must
    re-histogram at the true first non-constant digit.  n = 2^16+1
    and 2^24+1 sorted/reverse keys are such inputs (sampled max 65520 < 65536)."""
    sizes = [65537, (1 << 24) + 1] if R == 8 else [65537]
    for n in sizes:
        check(dg.generate(n, R, K, dist, payload="index" if R > K else "random", seed=9), K)


@pytest.mark.parametrize("R,K", [(8, 8), (16, 8), (32, 16)])
def test_rare_wide_outliers(R, K):
    # 32-bit ids plus a few keys far above them at positions the sample never sees
    n = 1_000_003
    a = dg.generate(n, R, K, "uniform", payload="index" if R > K else "random", seed=21)
    w = a.view(np.uint64).reshape(n, R // 8)
    hi = K // 8 - 1
    w[:, hi] &= np.uint64(0xFFFFFFFF)
    for i in (1, 4097, 500_001, n - 2):  # the sample stride here is n // 4096 = 244
        w[i, hi] = np.uint64(1 << 63) | np.uint64(i)
    check(a, K)


@pytest.mark.parametrize("var", ["RADSORT_LOCAL_BIG=1", "RADSORT_LOCAL2=1", "RADSORT_LOCAL_EARLY=0", "RADSORT_LOCAL_PIPE=0",
                                 "RADSORT_LOCAL_PIPE256=1", "RADSORT_LOCAL_PIPE256=0"])
@pytest.mark.parametrize("R,K", [(8, 8), (16, 8), (16, 16), (32, 16), (24, 8), (40, 16)])
def test_opt_in_local_sorters(var, R, K, monkeypatch):
    # the opt-in local sorters (k_local_big: 1024-thread CTAs, ranks by a second
    # atomic pass; k_local2: two-phase partition through the scratch range; the
    # pipelined sort with a bin's fix-up beside the next bin's count; round 1's
    # unpipelined k_local; the 256-thread class pipelined or not) on bins of every size class, skewed and duplicate-heavy keys included
    name, val = var.split("=")
    monkeypatch.setenv(name, val)
    for dist, n in (("uniform", 2_000_003), ("zipf", 1_500_001), ("few", 300_007), ("bytes", 700_001),
                    ("uniform40", 1_000_003)):
        check(dg.generate(n, R, K, dist, payload="index" if R > K else "random", seed=n % 97), K)


@pytest.mark.parametrize("R,K", [(32, 8), (40, 16)])
@pytest.mark.parametrize("ki", ["1", "0"])
@pytest.mark.parametrize("dist", ["uniform", "zipf", "few", "equal", "bytes"])
def test_key_index_sort(R, K, ki, dist, monkeypatch):
    # NEXT-1: (key, index) records sorted by the radix sort, then one gather of
    # the full records (RADSORT_KEY_INDEX=1), against the direct sort (=0);
    # sizes below / at / above the CTA-local capacity and across several tiles
    import paper_1703_00687_b200 as rs

    monkeypatch.setenv("RADSORT_KEY_INDEX", ki)
    for n in (C_of(R) - 1, C_of(R) + 1, 3 * T_of(R) + 17, 700_001):
        a = dg.generate(n, R, K, dist, payload="random", seed=n + R)
        check(a, K)
        if n > C_of(R):
            assert rs.last_stats()["key_index"] == (1 if ki == "1" else 0)


# ---- wide levels (10-bit digit: digit d + the two leading bits of digit d+1)
def _wide_levels():
    import paper_1703_00687_b200 as rs

    return rs.last_stats()["wide_levels"]


@pytest.mark.parametrize("R,K", LAYOUTS)
@pytest.mark.parametrize("dist", ["uniform", "zipf", "sorted", "few", "consttop", "bytes", "uniform40"])
def test_wide_level_forced(R, K, dist, monkeypatch):
    # RADSORT_WIDE=2: every level whose segments average >= 2 K records scatters by 10 bits (the
    # next level then by 8); sizes span several 1024-digit tiles, ragged tails, children of every
    # class (tiny, local with the 2 shared bits, Large again)
    monkeypatch.setenv("RADSORT_WIDE", "2")
    payload = "index" if R > K else "random"
    for n in (2_500, 300_001, 1_500_007):
        a = dg.generate(n, R, K, dist, payload=payload, seed=4242 + n)
        check(a, K)
        if dist in ("uniform", "bytes") and n > C_of(R):
            assert _wide_levels() >= 1, "no wide level ran"


@pytest.mark.parametrize("R,K", [(8, 8), (16, 16), (32, 16), (24, 8), (40, 16)])
def test_wide_level_consecutive_and_split(R, K, monkeypatch):
    # RADSORT_WIDE=3: every level wide, so wide levels also run on segments whose digit already
    # shares two leading bits; and the dominant-key three-way split on a wide level
    monkeypatch.setenv("RADSORT_WIDE", "3")
    # uniform: level-0 children of ~1.3 C records are Large again -> a second wide level
    for n, dist in ((int(1.3 * C_of(R) * 1024) + 7, "uniform"), (400_001, "zipf"), (200_003, "bytes")):
        check(dg.generate(n, R, K, dist, payload="index" if R > K else "random", seed=99 + n), K)
        assert _wide_levels() >= (2 if dist == "uniform" else 1)
    monkeypatch.setenv("RADSORT_WIDE", "2")
    a = dg.generate(1_000_003, R, K, "uniform", seed=98)
    a[::3] = a[0]
    a[1::3] = a[0]  # two thirds of the records carry one key: split three ways on the wide level 0
    check(a, K)
    assert _wide_levels() >= 1


@pytest.mark.parametrize("R,K", [(32, 16), (32, 8)])
def test_wide_level_default_rule(R, K, monkeypatch):
    # the default rule takes a wide level where the 8-bit children would exceed the CTA-local
    # capacity C and the 10-bit ones fit: segments averaging (256 C, 0.95 * 1024 C] records;
    # one such segment at level 0 (n = 3.5 M for R = 32); default for R >= 24 only
    monkeypatch.delenv("RADSORT_WIDE", raising=False)
    n = 3_500_000
    check(dg.generate(n, R, K, "uniform", seed=7), K)
    assert _wide_levels() == 1
    monkeypatch.setenv("RADSORT_WIDE", "0")
    check(dg.generate(n, R, K, "uniform", seed=7), K)
    assert _wide_levels() == 0


@pytest.mark.parametrize("R,K,bins", [(16, 8, 300), (16, 16, 300), (8, 8, 300), (16, 8, 600)])
def test_wide_level_small_records_need_distinct_keys(R, K, bins, monkeypatch):
    # R < 24 takes the default rule's wide level only where the sampled keys hardly repeat
    # (k_dupest).  The rule's window is (256 C, 0.95 * 1024 C] records per segment:
    # with 600 C records the whole input is in it (level 0 is wide, decided before the pass);
    # with 1200 C only the two level-0 bins are (the leading key byte takes two values: level 1
    # is wide).  Repeated keys: no wide level
    monkeypatch.delenv("RADSORT_WIDE", raising=False)
    monkeypatch.delenv("RADSORT_WIDE_MIN_R", raising=False)
    n = int(2 * bins * C_of(R)) + 11
    a = dg.generate(n, R, K, "uniform", payload="index" if R > K else "random", seed=31)
    a[:, K - 1] &= 1
    check(a, K)
    assert _wide_levels() == 1
    b = a.copy()
    b[:, :K] = a[np.arange(n) % 50_021, :K]  # ~50 K distinct keys, ~100 copies each
    check(b, K)
    assert _wide_levels() == 0
    monkeypatch.setenv("RADSORT_WIDE_MIN_R", "8")  # the rule without the estimate
    check(b, K)
    assert _wide_levels() == 1


@pytest.mark.parametrize("R,K", [(8, 8), (16, 8), (32, 16), (40, 16)])
@pytest.mark.parametrize("cfg", ["1", "2"])
def test_wide_level_both_tile_shapes(R, K, cfg, monkeypatch):
    # RADSORT_WIDE_CFG: the wide pass as one 1024-thread CTA per SM (1, default for R < 24) or two
    # 512-thread CTAs (2, default for R >= 24): both shapes on both record-size classes
    monkeypatch.setenv("RADSORT_WIDE", "2")
    monkeypatch.setenv("RADSORT_WIDE_CFG", cfg)
    for n, dist in ((1_200_011, "uniform"), (300_007, "zipf")):
        check(dg.generate(n, R, K, dist, payload="index" if R > K else "random", seed=515 + n), K)
        assert _wide_levels() >= 1
