"""Host-side logic of the multi-GPU path on CPU with 2 real processes (gloo).

radsort_sort_multi's host plan -- quotas, boundary bucket, digit-by-digit
splitter refinement, exact split of an equal-key run across ranks -- is made
of the pure C functions radsort_plan_quotas / radsort_locate_bucket /
radsort_plan_digit / radsort_plan_equal_split.  Here two gloo ranks drive
exactly those functions over real collectives (numpy stands in for the device
histogram / binary-search kernels, which tests/test_gpu_multi.py covers on the
GPU), exchange their slices, and the rank-order concatenation is checked
against the oracle and the exact quotas.  With fused=True the exchange is the
fused one: radsort_plan_fused places every record of every piece in its
receiver's (d0, d0+1) bin, and the receivers' buffers must come out exactly
covered."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _digit(keys, d):
    return ((keys >> np.uint64(8 * (7 - d))) & np.uint64(255)).astype(np.int64)


def _set_digit(key, d, v):
    sh = 8 * (7 - d)
    return (key & ~(0xFF << sh)) | (v << sh)


def _allreduce(x):
    t = torch.from_numpy(np.asarray(x, dtype=np.uint64).view(np.int64).copy())
    dist.all_reduce(t)
    return t.numpy().view(np.uint64)


def _allgather(x):
    t = torch.from_numpy(np.asarray(x, dtype=np.uint64).view(np.int64).copy())
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return np.stack([o.numpy() for o in out]).view(np.uint64)


def _worker(rank, world, port, dist_name, result_q, fused=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1703_00687_b200 as rs
    from datagen import host as dg

    sizes = [30_000, 17_001]
    first = [0, sizes[0]]
    a = dg.generate(sizes[rank], 16, 8, dist_name, payload="index", seed=99, first=first[rank])
    keys = a.view(np.uint64).reshape(-1, 2)[:, 0].copy()
    G = world
    N = int(_allreduce([len(keys)])[0])
    q = rs.plan_quotas(N, G)
    Qb = np.concatenate([[0], np.cumsum(q)]).astype(np.uint64)
    # global first non-constant digit (AND/OR allgathered) and its histogram
    ao = _allgather(np.array([np.bitwise_and.reduce(keys) if len(keys) else ~np.uint64(0),
                              np.bitwise_or.reduce(keys) if len(keys) else np.uint64(0)], dtype=np.uint64))
    AND = int(np.bitwise_and.reduce(ao[:, 0])) & 0xFFFFFFFFFFFFFFFF
    OR = int(np.bitwise_or.reduce(ao[:, 1])) & 0xFFFFFFFFFFFFFFFF
    d0 = next((d for d in range(8) if ((AND ^ OR) >> (8 * (7 - d))) & 255), 0)
    h = np.bincount(_digit(keys, d0), minlength=256).astype(np.uint64)
    H = _allreduce(h)
    # local level-0 partition by d0 (numpy stands in for k_scatter)
    order = np.argsort(_digit(keys, d0), kind="stable")
    part = a[order]
    pkeys = keys[order]
    lbase = np.concatenate([[0], np.cumsum(h)]).astype(np.int64)
    Hbase = np.concatenate([[0], np.cumsum(H)]).astype(np.uint64)
    cuts = [0]
    for g in range(1, G):
        Qg = int(Qb[g])
        b, before = rs.locate_bucket(H, Qg)
        assert before == int(Hbase[b])
        lo, hi = int(lbase[b]), int(lbase[b + 1])
        # sort the straddling bucket locally (the device path uses radsort_sort here)
        o2 = np.argsort(pkeys[lo:hi], kind="stable")
        part[lo:hi] = part[lo:hi][o2]
        pkeys[lo:hi] = pkeys[lo:hi][o2]
        key = _set_digit(AND, d0, b)
        for d in range(d0 + 1, 8):
            if not (((AND ^ OR) >> (8 * (7 - d))) & 255):
                continue
            probes = np.array([_set_digit(key, d, v) & ~((1 << (8 * (7 - d))) - 1) for v in range(256)],
                              dtype=np.uint64)
            cnt = np.searchsorted(pkeys[lo:hi], probes, "left").astype(np.uint64)
            gl = _allreduce(cnt)
            key = _set_digit(key, d, rs.plan_digit(gl, Qg - int(Hbase[b])))
        k = np.uint64(key)
        lt = int(np.searchsorted(pkeys[lo:hi], k, "left"))
        le = int(np.searchsorted(pkeys[lo:hi], k, "right"))
        allv = _allgather([lt, le - lt])
        L = int(Hbase[b]) + int(allv[:, 0].sum())
        below = rs.plan_equal_split(allv[:, 1], L, Qg)
        cuts.append(lo + lt + int(below[rank]))
    cuts.append(len(keys))
    if not fused:
        # exchange (every rank's slice for every destination), then sort the received key range
        allp = [None] * G
        dist.all_gather_object(allp, [part[cuts[g]:cuts[g + 1]] for g in range(G)])
        mine = np.concatenate([allp[src][rank] for src in range(G)])
    else:
        # fused exchange (radsort_plan_fused): pieces = (receiver, d0 bucket) ranges of the
        # partitioned array, histogrammed by digit d0+1; every record is "stored" at
        # base[piece][v] + its rank among the piece's records with digit v (the k_scatter<PEER>
        # pass); the receiver's buffer must come out exactly covered, bin (b, v) by bin
        d1 = d0 + 1
        pdst, pbkt, prng = [], [], []
        for g in range(G):
            for b in range(256):
                lo, hi = max(cuts[g], int(lbase[b])), min(cuts[g + 1], int(lbase[b + 1]))
                if hi > lo:
                    pdst.append(g)
                    pbkt.append(b)
                    prng.append((lo, hi))
        tab = np.zeros((G, 256, 256), dtype=np.uint32)
        for g, b, (lo, hi) in zip(pdst, pbkt, prng):
            tab[g, b] = np.bincount(_digit(pkeys[lo:hi], d1), minlength=256)
        tabs = [None] * G
        dist.all_gather_object(tabs, tab)
        base, recv = rs.plan_fused(np.stack(tabs), rank, pdst, pbkt)
        sends = [[] for _ in range(G)]
        for i, (g, (lo, hi)) in enumerate(zip(pdst, prng)):
            dv = _digit(pkeys[lo:hi], d1)
            o = np.argsort(dv, kind="stable")
            rank_in = np.empty(hi - lo, dtype=np.int64)
            rank_in[o] = np.arange(hi - lo) - np.searchsorted(dv[o], dv[o], "left")
            sends[g].append((base[i][dv].astype(np.int64) + rank_in, part[lo:hi]))
        allsends = [None] * G
        dist.all_gather_object(allsends, sends)
        n_recv = int(recv[65536])
        mine = np.zeros((n_recv, a.shape[1]), dtype=a.dtype)
        hits = np.zeros(n_recv, dtype=np.int64)
        for src in range(G):
            for off, recs in allsends[src][rank]:
                mine[off] = recs
                np.add.at(hits, off, 1)
        assert (hits == 1).all(), "fused exchange plan left gaps or overlaps"
        mk0 = mine.view(np.uint64).reshape(-1, 2)[:, 0]
        bv = _digit(mk0, d0) * 256 + _digit(mk0, d1)
        assert (np.diff(bv) >= 0).all(), "records outside their (d0, d0+1) bin"
        assert (np.searchsorted(bv, np.arange(65536), "left") == recv[:65536].astype(np.int64)).all()
    assert mine.shape[0] == int(q[rank]), (mine.shape, q)
    mk = mine.view(np.uint64).reshape(-1, 2)[:, 0]
    mine = mine[np.argsort(mk, kind="stable")]
    shards = [None] * G
    dist.all_gather_object(shards, mine)
    full = [None] * G
    dist.all_gather_object(full, a)
    if rank == 0:
        import oracle

        got = np.concatenate(shards)
        want = oracle.sort(np.concatenate(full), 8)
        result_q.put(oracle.compare(got, want, 8))
    dist.destroy_process_group()


@pytest.mark.parametrize("dist_name", ["uniform40", "few", "equal", "bytes"])
@pytest.mark.parametrize("fused", [False, True])
def test_two_rank_plan_matches_oracle(dist_name, fused):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dist_name, q, fused)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) == -1


def test_planner_functions():
    import paper_1703_00687_b200 as rs

    assert list(rs.plan_quotas(10, 3)) == [4, 3, 3]
    assert list(rs.plan_quotas(2, 4)) == [1, 1, 0, 0]
    c = np.arange(256, dtype=np.uint64) * 10
    assert rs.plan_digit(c, 0) == 0
    assert rs.plan_digit(c, 15) == 1
    assert rs.plan_digit(c, 10_000) == 255
    assert list(rs.plan_equal_split([5, 0, 7], L=100, Q=108)) == [5, 0, 3]
    assert list(rs.plan_equal_split([5, 0, 7], L=100, Q=100)) == [0, 0, 0]
