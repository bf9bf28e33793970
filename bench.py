#!/usr/bin/env python3
"""radsort benchmark: sorted Mrecords/s and effective HBM GB/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl radsort|reference]

A step = one radsort_sort of the whole workload (every MSD level: histogram,
plan, look-back scatter, children/tiny, CTA-local sort) with the input already
resident in HBM.  Between steps the input is restored from a pristine device
copy (untimed; each step is bracketed by a barrier + cudaDeviceSynchronize and
timed with CUDA events on the sort's stream).  Inputs (>= 3.2 GB at the
default config) are larger than the 126 MB L2, so no L2 flush is needed.

N = 1 runs the largest single-GPU configuration of BASELINE.json (c4: 1 B
records of 32 B, 16-byte uniform keys, 16-byte payload; 32 GB) unless
--config says otherwise.  N > 1 (torchrun, one process per GPU, NCCL) runs
radsort_sort_multi: c3/c4 as BASELINE.json defines them, strong scaling (the
config's n records in total, n/N per GPU); c5 weak scaling (n per GPU); c1/c2
(single-GPU configs) weak.

--impl reference times the CPU oracle (std::stable_sort, test infrastructure)
on bounded samples of the same workload on the host cores; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sorted Mrecords/s and effective HBM GB/s vs ~8 TB/s peak at 1/2/4/8 B200"
UNIT = "Mrecords/s"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clock / throttle sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []  # (arrival time, csv line)
        self.t0 = self.t1 = None

    def start(self):
        """Start nvidia-smi early (it needs ~0.1-0.5 s before its first line)."""
        return self.__enter__()

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        """End of the timed region: short regions get the first sample after it."""
        self.t1 = time.time()
        deadline = self.t1 + 2.0
        while self.proc and time.time() < deadline and not any(t >= self.t0 for t, _ in self.lines):
            time.sleep(0.02)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inside = [ln for t, ln in self.lines if self.t0 is None or self.t0 <= t <= (self.t1 or t)]
        after = False
        if not inside and self.t0 is not None:  # region shorter than the sampling period
            later = [ln for t, ln in self.lines if t >= self.t0]
            inside, after = later[:1], bool(later)
        for ln in inside:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if after:
            out["note"] = "timed region shorter than the 100 ms sampling period: first sample after it"
        return out


def workload_desc(name, c, n):
    return (f"{name}: {n} records, R={c['R']} B, K={c['K']} B, keys {c['dist']}, payload {c['payload']}, "
            f"seed {c['seed']}")


def cpu_baseline(cfg_name, target_s=10.0, max_n=40_000_000):
    """The oracle as it stands on a bounded prefix sample of the workload, on
    the host cores: single-threaded std::stable_sort (oracle.sort), and its
    all-cores form (oracle.sort_parallel: nproc chunks + merge rounds, the same
    stable result).  Returns the cpu_baseline dict."""
    import oracle
    from datagen import host as dg

    c = dg.CONFIGS[cfg_name]
    nproc = os.cpu_count() or 1
    n = 1_000_000
    a = dg.generate_config(cfg_name, n=n)
    t0 = time.perf_counter()
    oracle.sort(a, c["K"])
    dt = time.perf_counter() - t0
    n2 = int(min(max_n, max(n, n * target_s / max(dt, 1e-6))))
    if n2 > n:
        a = dg.generate_config(cfg_name, n=n2)
        t0 = time.perf_counter()
        oracle.sort(a, c["K"])
        dt = time.perf_counter() - t0
        n = n2
    t0 = time.perf_counter()
    oracle.sort_parallel(a, c["K"], nproc)
    dtp = time.perf_counter() - t0
    sample = f"first {n} records of the {cfg_name} stream ({n * c['R'] / 1e9:.2f} GB)"
    return {"value": round(n / dt / 1e6, 3), "unit": UNIT, "cores": 1, "nproc": nproc, "kind": "oracle",
            "sample": f"{sample}, oracle std::stable_sort on 1 of {nproc} host cores, {dt:.2f} s",
            "all_cores": {"value": round(n / dtp / 1e6, 3), "unit": UNIT, "cores": nproc,
                          "kind": "oracle (all cores)",
                          "sample": f"{sample}, {nproc} std::stable_sort chunks + std::merge rounds, {dtp:.2f} s"}}


STRONG = ("c3", "c4")  # BASELINE.json: fixed total N over 1, 2, 4, 8 GPUs


def scaling_of(cfg, world):
    # the label is the config's, at every N (at N = 1 both give the same work),
    # so the driver's per-N lines of one config agree on how they scale
    del world
    return "strong" if cfg in STRONG else "weak"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from datagen import host as dg

    import oracle

    c = dg.CONFIGS[args.config]
    # bounded sample per step (~5 s of CPU work), the same recipe as the GPU arm
    n = args.ref_sample
    a = dg.generate_config(args.config, n=n)
    for _ in range(args.warmup):
        oracle.sort(a, c["K"])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.sort(a, c["K"])
        times.append(time.perf_counter() - t0)
    total = sum(times)
    v = args.steps * n / total / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 3),
        "higher_is_better": True, "scaling": scaling_of(args.config, args.gpus), "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": workload_desc(args.config, c, c["n"]), "sample_records_per_step": n},
        "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": 1, "nproc": os.cpu_count(), "kind": "oracle",
                         "sample": f"first {n} records of the {args.config} stream per step, std::stable_sort"},
        "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def host_sorted_sample(a, K, m=1 << 21):
    """Sanity check of a host output: a window of m records in the middle is
    non-decreasing by key (little-endian K-byte key, high word last)."""
    import numpy as np

    n = a.shape[0]
    lo = max(0, n // 2 - m // 2)
    w = np.ascontiguousarray(a[lo:lo + m, :K]).view(np.uint64)
    if K == 8:
        return bool((w[1:, 0] >= w[:-1, 0]).all())
    hi, l0 = w[:, 1], w[:, 0]
    return bool(((hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (l0[1:] >= l0[:-1]))).all())


def run_radsort(args):
    import torch
    import torch.distributed as dist

    import paper_1703_00687_b200 as rs
    from datagen import device as dd
    from datagen import host as dg
    import verify

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    rs.init(local_rank)
    c = dict(dg.CONFIGS[args.config])
    n_cfg = args.n or c["n"]
    R, K = c["R"], c["K"]
    stream = torch.cuda.current_stream()
    strong = scaling_of(args.config, world) == "strong"

    def barrier():
        if world > 1:
            dist.barrier()

    # input shard of this rank: strong scaling splits the config's n records
    # (global indices [first, first + n)); weak scaling gives every rank n
    if strong:
        first = n_cfg * rank // world
        n = n_cfg * (rank + 1) // world - first
    else:
        first, n = rank * n_cfg, n_cfg
    pristine = dd.generate_tensor(n, R, K, c["dist"], c["payload"], c["seed"], first=first)
    # exact-balance output quotas differ from n by at most one record; slack for unequal shards
    cap = n if world == 1 else n + world + 1024
    rec = torch.empty((cap, R), dtype=torch.uint8, device="cuda")
    tmp = torch.empty((cap, R), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    dig_in = verify.digest(pristine.data_ptr(), n, R)

    def restore():
        rec[:n].copy_(pristine)

    kmc = args.config == "kmc"  # the KMC3 consumer: sort, then run-length count (unique keys + counts)
    uc = {"ms": 0.0, "unique": 0}

    def one_sort():
        if world == 1:
            rs.sort_ptr(rec.data_ptr(), tmp.data_ptr(), n, R, K, stream.cuda_stream)
            if kmc:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                keys, _ = rs.unique_count(rec[:n], K, stream)
                e1.record(stream)
                e1.synchronize()
                uc["ms"] += e0.elapsed_time(e1)
                uc["unique"] = int(keys.shape[0])
            return n
        return rs.sort_multi(rec, tmp, n, K)

    clk = ClockSampler(local_rank).start()  # started early: nvidia-smi's first line takes a while
    # warm-up (the first one is also the verification run: sorted + same multiset)
    for w in range(max(args.warmup, 1)):
        restore()
        torch.cuda.synchronize()
        n_out = one_sort()
        torch.cuda.synchronize()
        if w == 0:
            bad, first = verify.sorted_check(rec.data_ptr(), n_out, R, K)
            if bad or (world == 1 and verify.digest(rec.data_ptr(), n, R) != dig_in):
                print(json.dumps({"error": f"verification failed: {bad} inversions (first at {first})"}), flush=True)
                clk.__exit__()
                return 1

    rs.set_timing(True)
    uc["ms"] = 0.0
    kern_ms = {}
    kern_bytes = {}
    launches = 0
    step_ms = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.mark_start()
    try:
        for _ in range(args.steps):
            restore()
            torch.cuda.synchronize()
            barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            one_sort()
            ev1.record(stream)
            torch.cuda.synchronize()
            barrier()
            step_ms.append(ev0.elapsed_time(ev1))
            st = rs.last_stats()
            for k, v in st["kernel_ms"].items():
                kern_ms[k] = kern_ms.get(k, 0.0) + v
            for k, v in st["kernel_bytes"].items():
                kern_bytes[k] = kern_bytes.get(k, 0) + v
            launches += sum(st["kernel_launches"].values()) + (4 if kmc else 0)
    finally:
        clk.mark_end()
        clk.__exit__()
    rs.set_timing(False)
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    stats = rs.last_stats()
    N_total = n_cfg if strong else n * world
    value = N_total * args.steps / (total_ms / 1e3) / 1e6
    passes_bytes = sum(kern_bytes.values()) / args.steps  # algorithmic bytes per step (read + write)
    eff_gbs = passes_bytes * world / (total_ms / args.steps / 1e3) / 1e9
    peak, peak_kind = measured_peaks()
    # roofline of the dominant HBM-bound kernel (largest time per step), with
    # the traffic ncu measured for it (profiles/traffic_<config>.json, bytes per launch)
    traffic_map = {}
    tp = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic_map = json.load(f)
    names = {"scatter": "k_scatter (radix pass: rank, smem staging, coalesced scatter)",
             "local": "k_local / k_local_pipe + k_local_cluster (on-chip sort of bins <= C records / of C < n <= ~4C records "
                      "in a 4-CTA cluster)",
             "hist": "k_hist_pre (digit histogram + per-tile prefix, read only)"}
    launches_per_step = {k: v for k, v in rs.last_stats()["kernel_launches"].items()}
    roof_all = {}
    for k in ("scatter", "local", "hist"):
        ms = kern_ms.get(k, 0.0)
        b = kern_bytes.get(k, 0)
        if ms <= 0 or b <= 0:
            continue
        ach = b / (ms / 1e3) / 1e9
        nl = max(1, launches_per_step.get(k, 1))
        tr = traffic_map.get(k)
        if tr is not None and traffic_map.get("_per") == "step":  # bytes per sort -> per launch, as `achieved`
            tr = round(tr / nl)
        roof_all[k] = {"bound": "hbm", "kernel": names[k], "achieved": round(ach, 1), "peak": peak,
                       "peak_kind": peak_kind, "unit": "GB/s", "frac": round(ach / peak, 4),
                       "traffic": tr, "bytes_per_launch": b / args.steps / nl, "launches_per_step": nl,
                       "ms_per_step": round(ms / args.steps, 4)}
    dom = max(roof_all, key=lambda k: roof_all[k]["ms_per_step"]) if roof_all else None
    roofline = dict(roof_all[dom]) if dom else None

    # end to end through the public C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if world > 1 and not args.no_e2e:
        # every rank: H2D of its pinned input shard, the collective sort, D2H of its output shard;
        # the step time is the max over ranks
        host_in = pristine.cpu().pin_memory()
        e2e_t, out_bytes = [], 0
        for i in range(args.e2e_steps + 1):
            host_out = torch.empty((cap, R), dtype=torch.uint8).pin_memory()
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            rec[:n].copy_(host_in, non_blocking=True)
            n_out = rs.sort_multi(rec, tmp, n, K)
            host_out[:n_out].copy_(rec[:n_out], non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if i > 0:
                e2e_t.append(float(t.item()))
            out_bytes = n_out * R
        e2e = {"value": round(N_total / statistics.median(e2e_t) / 1e6, 3), "unit": UNIT,
               "h2d_bytes_per_step": n * R, "d2h_bytes_per_step": out_bytes,
               "note": "per rank; max over ranks of the wall time"}
        del host_in, host_out
    if world == 1 and not args.no_e2e:
        host_pristine = pristine.cpu().pin_memory()
        host = torch.empty_like(host_pristine).pin_memory()
        # pipelined (radsort_sort_host_stream): a stream of B batches of this workload,
        # each copied in from pinned host memory, sorted and copied out; batch k+1's
        # copy-in and batch k-1's copy-out overlap batch k's sort.  Device buffers: the
        # bench's own rec / tmp / pristine (its copy is on the host now) + one more.
        # The timed region runs from the first copy-in to the last copy-out.
        extra = torch.empty((cap, R), dtype=torch.uint8, device="cuda")
        bufs = [rec[:n], pristine[:n], extra[:n]]
        B = max(args.e2e_batches, 2)
        rs.sort_host_stream([host_pristine] * 2, [host] * 2, K, bufs, tmp[:n])  # warm-up (streams, events)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rs.sort_host_stream([host_pristine] * B, [host] * B, K, bufs, tmp[:n])
        dt_pipe = time.perf_counter() - t0
        ok = host_sorted_sample(host.numpy(), K)
        del extra, bufs
        torch.cuda.empty_cache()
        # serial (radsort_sort_host): copy-in, sort, copy-out of one batch per call
        e2e_t = []
        for i in range(args.e2e_steps + 1):
            host.copy_(host_pristine)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rs.sort_host(host, K)
            dt = time.perf_counter() - t0
            if i > 0:
                e2e_t.append(dt)
        e2e = {"value": round(B * n / dt_pipe / 1e6, 3), "unit": UNIT,
               "h2d_bytes_per_step": n * R, "d2h_bytes_per_step": n * R,
               "mode": f"radsort_sort_host_stream: {B} batches pipelined over 3 device buffers, "
                       f"{dt_pipe:.3f} s wall from the first copy-in to the last copy-out (host output "
                       f"sample sorted: {ok})",
               "serial": {"value": round(n / statistics.median(e2e_t) / 1e6, 3), "unit": UNIT,
                          "mode": "radsort_sort_host: copy-in + sort + copy-out per call, median of "
                                  f"{args.e2e_steps}"}}
        del host, host_pristine

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
            "scaling": scaling_of(args.config, world), "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": workload_desc(args.config, c, N_total), "records_per_gpu": n, "rec_size": R,
                       "key_size": K, "parallelism": f"key-range sharding x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than the 126 MB L2; input restored from a pristine copy between steps"},
            "effective_hbm_gbs": round(eff_gbs, 1),
            "hbm_frac_of_8tbs": round(eff_gbs / 8000.0, 4),
            "roofline": roofline,
            "roofline_by_kernel": roof_all,
            "kernel_ms_per_step": {k: round(v / args.steps, 4) for k, v in kern_ms.items()},
            "kernel_bytes_per_step": {k: v // args.steps for k, v in kern_bytes.items()},
            "passes": {"levels": stats["levels"], "scatter_passes": stats["scatter_passes"],
                       "first_digit": stats["first_digit"]},
            "gpu_launches": launches // args.steps,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if world > 1:
            line["multi"] = {"exchange": {2: "fused (next-digit scatter into the peers' buffers over NVLink)",
                                          1: "NCCL send/recv"}.get(stats.get("exchange", 0), "none"),
                             "nvlink_bytes_sent_rank0": stats["nvlink_bytes_sent"],
                             "nvlink_bytes_recv_rank0": stats["nvlink_bytes_recv"]}
        if kmc:  # the step also run-length counts the sorted k-mers (inside the timed region)
            line["kmc"] = {"unique_keys": uc["unique"], "unique_count_ms_per_step": round(uc["ms"] / args.steps, 4),
                           "note": "value/ms_per_step include the unique-count kernels; e2e is the sort alone"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5", "kmc"])
    ap.add_argument("--n", type=int, default=0, help="override records per GPU")
    ap.add_argument("--impl", default="radsort", choices=["radsort", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-batches", type=int, default=6, help="batches of the pipelined e2e stream")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=4_000_000)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_radsort(args)


if __name__ == "__main__":
    sys.exit(main())
