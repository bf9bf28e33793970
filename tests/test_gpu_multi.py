"""Multi-GPU path (radsort_sort_multi) on one B200.

The pool gives one GPU per box, so the G-rank algorithm runs through the
in-process loopback transport: G host threads are the G ranks (own stream,
own buffers, same kernels, same host plan; collectives are host barriers and
the exchange is device-to-device copies).  The NCCL transport itself runs with
a 1-rank communicator.  Parity: the rank-order concatenation of the shards
equals the oracle sort of the concatenated inputs (canonical compare), and
every rank holds exactly its quota."""
import os
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from datagen import host as dg  # noqa: E402


def run_loopback(shards, K, slack=1024, stats=None):
    import paper_1703_00687_b200 as rs

    G = len(shards)
    N = sum(s.shape[0] for s in shards)
    R = shards[0].shape[1]
    q = rs.plan_quotas(N, G)
    grp = rs.LoopbackGroup(G)
    recs, tmps, outs, errs = [], [], [None] * G, [None] * G
    for g, s in enumerate(shards):
        cap = max(int(q[g]), s.shape[0]) + slack
        r = torch.empty((cap, R), dtype=torch.uint8, device="cuda")
        if s.shape[0]:
            r[: s.shape[0]].copy_(torch.from_numpy(s))
        recs.append(r)
        tmps.append(torch.empty_like(r))
    torch.cuda.synchronize()

    def work(g):
        try:
            st = torch.cuda.Stream()
            outs[g] = grp.sort(g, recs[g], tmps[g], shards[g].shape[0], K, stream=st)
            st.synchronize()
            if stats is not None:
                stats[g] = rs.last_stats()  # thread-local: this rank's call
        except Exception as e:  # noqa: BLE001
            errs[g] = e

    th = [threading.Thread(target=work, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    grp.close()
    for e in errs:
        if e is not None:
            raise e
    for g in range(G):
        assert outs[g] == int(q[g]), f"rank {g}: n_out {outs[g]} != quota {q[g]}"
    return [recs[g][: outs[g]].cpu().numpy() for g in range(G)]


@pytest.fixture(scope="module", autouse=True)
def _init():
    import paper_1703_00687_b200 as rs

    rs.init(0)


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("R,K,dist", [(8, 8, "uniform"), (16, 8, "uniform40"), (8, 8, "zipf"), (32, 16, "uniform"),
                                      (16, 16, "bytes"), (8, 8, "few"), (16, 8, "equal"), (24, 8, "uniform"),
                                      (40, 16, "zipf")])
@pytest.mark.parametrize("fused", [1, 0])
def test_loopback_multi(G, R, K, dist, fused, monkeypatch):
    # fused = 1: the product path (next-digit scatter straight into the peers'
    # buffers); 0: the send/recv exchange
    monkeypatch.setenv("RADSORT_MULTI_FUSED", str(fused))
    rng = np.random.default_rng(G * 100 + R)
    sizes = [int(x) for x in rng.integers(20_000, 120_000, G)]
    if G >= 3:
        sizes[1] = 0  # an empty rank
    first = np.concatenate([[0], np.cumsum(sizes)])
    payload = "index" if R > K else "random"
    shards = [dg.generate(sizes[g], R, K, dist, payload=payload, seed=31, first=int(first[g])) for g in range(G)]
    st = [None] * G
    out = run_loopback(shards, K, stats=st)
    got = np.concatenate(out)
    a = np.concatenate(shards)
    assert oracle.compare(got, oracle.sort(a, K), K) == -1
    assert all(s["exchange"] == (2 if fused else 1) for s in st), [s["exchange"] for s in st]


def test_loopback_heavy_key_straddles_boundaries():
    # one key holds 60 % of the records: it straddles several rank boundaries
    G, R, K = 4, 16, 8
    a = dg.generate(200_000, R, K, "uniform", payload="index", seed=3)
    w = a.view(np.uint64).reshape(-1, 2)
    w[::5, 0] = 12345
    w[1::5, 0] = 12345
    w[2::5, 0] = 12345
    shards = np.array_split(a, G)
    for fused in ("1", "0"):
        os.environ["RADSORT_MULTI_FUSED"] = fused
        try:
            out = run_loopback([np.ascontiguousarray(s) for s in shards], K)
        finally:
            os.environ.pop("RADSORT_MULTI_FUSED", None)
        assert oracle.compare(np.concatenate(out), oracle.sort(a, K), K) == -1


def test_nccl_single_rank():
    import torch.distributed as dist

    import paper_1703_00687_b200 as rs

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    created = False
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        created = True
    try:
        a = dg.generate(300_000, 16, 8, "uniform40", payload="index", seed=7)
        rec = torch.from_numpy(a.copy()).cuda()
        tmp = torch.empty_like(rec)
        dist.barrier()
        n_out = rs.sort_multi(rec, tmp, a.shape[0], 8)
        torch.cuda.synchronize()
        assert n_out == a.shape[0]
        assert rs.last_stats()["exchange"] == 2  # fused exchange: the buffer is exported by CUDA IPC
        assert oracle.compare(rec.cpu().numpy(), oracle.sort(a, 8), 8) == -1
    finally:
        if created:
            dist.destroy_process_group()


def test_library_communicator_single_rank():
    # radsort_comm_init (library-owned communicator, NCCL CTAs capped) drives
    # the same collective sort
    import paper_1703_00687_b200 as rs

    uid = rs.comm_unique_id()
    comm = rs.comm_init(uid, 1, 0, max_ctas=4)
    try:
        for R, K, dist in ((16, 8, "uniform40"), (8, 8, "zipf"), (32, 16, "uniform")):
            a = dg.generate(250_000, R, K, dist, payload="index" if R > K else "random", seed=8)
            rec = torch.from_numpy(a.copy()).cuda()
            tmp = torch.empty_like(rec)
            n_out = rs.sort_multi_comm(rec, tmp, a.shape[0], K, comm)
            torch.cuda.synchronize()
            assert n_out == a.shape[0]
            assert oracle.compare(rec.cpu().numpy(), oracle.sort(a, K), K) == -1
    finally:
        rs.comm_destroy(comm)
