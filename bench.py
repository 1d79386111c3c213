"""Benchmark: queries/sec at fixed Recall@100 of the derived two-pass PQ search.

Workload (BASELINE.json configs[1], the metric's single-GPU config):
PQ 4x16 + derived 4x8, N = 10M SIFT-like codes (seeded synthetic stand-in for
SIFT, data="synthetic"), queries batched 1024 per step, R(r2) = 1000,
k(r) = 100.  A step = one batch of 1024 queries through the whole derived
path (tables, guard, scan, threshold, refine + top-k).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  `value` is device-timed (CUDA events on the
search stream, inputs resident in HBM, L2 flushed between steps); `e2e`
times the public API FlatIndex.search with host numpy queries and results
(H2D + D2H inside).  `--impl reference` times the CPU oracle port of the
reference path on the host cores (rank 0 only).

N > 1 (torchrun): the database is split into N contiguous shards (strong
scaling of a fixed 10M database); each query batch runs the split API
(dpq_shard_*) with an NCCL all-reduce of the score histograms and an
all-gather of the per-shard top-k.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

M, B, BBAR, DSUB = 4, 16, 8, 32
D = M * DSUB


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", "--rows", dest="n", type=int, default=10_000_000)
    p.add_argument("--batch", type=int, default=1024)
    p.add_argument("--r", type=int, default=100)
    p.add_argument("--r2", type=int, default=1000)
    p.add_argument("--train", type=int, default=100_000)
    p.add_argument("--kmeans-iters", type=int, default=12)
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--cpu-seconds", type=float, default=20.0, help="CPU work budget of cpu_baseline")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--profile-once", action="store_true", help="one short step only (for ncu)")
    p.add_argument("--mode", default="replicas", choices=["replicas", "shard"],
                   help="N > 1: query-parallel replicas of the index (default: configs[1] fits one GPU) or "
                        "the database sharded across GPUs with the NCCL exchange (configs[2]-[4] layout)")
    return p.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ setup --

def build_workload(args, device, rank: int = 0, world: int = 1, shard: bool = True, comm_device=None):
    """Seeded data, GPU-trained 4x16/8 model, GPU-encoded codes, queries,
    exact ground truth.  With world > 1 every rank generates the same
    database (seeded Philox chunks) and encodes only its contiguous shard;
    rank 0 trains and broadcasts the codebooks and the global prefix."""
    import torch

    from paper_1905_06900_b200 import datagen, train

    t0 = time.time()
    st = datagen.seed_streams(args.seed)
    centres = datagen.sift_centres(st["centres"])
    cb_shape = (M, 1 << B, DSUB)
    der_shape = (M, 1 << BBAR, DSUB)
    if rank == 0:
        tr = torch.as_tensor(datagen.sift_like(st["train"], centres, args.train), device=device)
        codebooks, derived = train.train_pq(tr, M, B, BBAR, iters=args.kmeans_iters, seed=args.seed)
        del tr
    if world > 1:
        import torch.distributed as dist

        cd = comm_device if comm_device is not None else device
        cbt = torch.as_tensor(codebooks, device=cd) if rank == 0 else torch.empty(cb_shape, device=cd)
        dt = torch.as_tensor(derived, device=cd) if rank == 0 else torch.empty(der_shape, device=cd)
        dist.broadcast(cbt, 0)
        dist.broadcast(dt, 0)
        codebooks, derived = cbt.cpu().numpy(), dt.cpu().numpy()
    t1 = time.time()
    db = datagen.sift_like_torch(args.n, args.seed + 1, centres, device=device)
    lo, hi = (rank * args.n // world, (rank + 1) * args.n // world) if shard else (0, args.n)
    enc = train.make_encoder(codebooks, device=device, kind="tc")  # tcgen05 3xTF32 GEMM + argmin
    codes = enc(db[lo:hi]).cpu().numpy().astype(np.uint16)
    del enc
    prefix = None
    if world > 1 and shard:
        import torch.distributed as dist

        npre = min(args.n, args.r2)
        pt = (torch.as_tensor(codes[:npre].astype(np.int32), device=device) if rank == 0
              else torch.empty((npre, M), dtype=torch.int32, device=device))
        dist.broadcast(pt, 0)
        prefix = pt.cpu().numpy().astype(np.uint16)
    nq = (args.steps + args.warmup) * args.batch * (1 if shard else world)
    queries = datagen.sift_like_torch(nq, args.seed + 2, centres, device=device)
    if shard:
        truth = train.exact_nn_gpu(db, queries, depth=1) if rank == 0 else None
    else:  # replicas: ground truth only for this rank's batches (s * world + rank)
        Bq = args.batch
        mine = np.concatenate([np.arange((s * world + rank) * Bq, (s * world + rank + 1) * Bq)
                               for s in range(args.steps + args.warmup)])
        truth = np.full((nq, 1), -1, dtype=np.int64)
        truth[mine] = train.exact_nn_gpu(db, queries[torch.as_tensor(mine, device=device)], depth=1)
    del db
    torch.cuda.empty_cache()
    t2 = time.time()
    log(f"[rank {rank}] setup: train {t1 - t0:.1f}s, data+encode+truth {t2 - t1:.1f}s")
    return {"codebooks": codebooks, "derived": derived, "codes": codes, "row_base": lo, "prefix": prefix,
            "queries": queries.cpu().numpy(), "queries_dev": queries, "truth": truth,
            "setup_s": t2 - t0}


# ---------------------------------------------------------------- clocks --

class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: an NVML
    polling thread (~1 ms period) that has taken its first sample before the
    region starts and stops right after it (nvidia-smi's >= 100 ms period
    cannot see a ~10 ms region)."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40),
               ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.smax = None
        self._stop = None

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:  # no NVML: report no samples
            return self
        self._stop = threading.Event()
        first = threading.Event()

        def poll():
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, rs))
                except Exception:
                    pass
                first.set()
                time.sleep(0.001)

        self._thread = threading.Thread(target=poll, daemon=True)
        self._thread.start()
        first.wait(2.0)
        return self

    def __exit__(self, *exc):
        if self._stop is not None:
            self._stop.set()
            self._thread.join(2.0)

    def summary(self):
        sm = [a for a, _ in self.samples]
        reasons = sorted({nm for _, rs in self.samples for nm, bit in self.REASONS if rs & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                "reasons": reasons, "samples": len(sm), "source": "NVML, ~1 ms polling during the timed steps"}


# ------------------------------------------------------------------- CPU --

_W = {}


def _cpu_worker(qrange):
    from oracle import derived_search as O

    lo, hi = qrange
    w = _W
    out = []
    for qi in range(lo, hi):
        ids, ds, info = O.derived_one(w["codebooks"], w["derived"], O.identity_rotate, w["codes"],
                                      w["queries"][qi], w["r"], w["r2"])
        out.append((qi, ids, ds, info["ncand"]))
    return out


def cpu_oracle_run(wl, args, nq_sample, procs):
    """The oracle port of the reference path on `procs` forked host
    processes (index arrays shared copy-on-write), queries [0, nq_sample)."""
    import multiprocessing as mp

    _W.update(codebooks=wl["codebooks"], derived=wl["derived"], codes=wl["codes"],
              queries=wl["queries"], r=args.r, r2=args.r2)
    per = (nq_sample + procs - 1) // procs
    ranges = [(i, min(nq_sample, i + per)) for i in range(0, nq_sample, per)]
    t0 = time.perf_counter()
    if procs == 1:
        res = [_cpu_worker(rg) for rg in ranges]
    else:
        with mp.get_context("fork").Pool(len(ranges)) as pool:
            res = pool.map(_cpu_worker, ranges)
    wall = time.perf_counter() - t0
    flat = sorted([x for part in res for x in part], key=lambda t: t[0])
    return wall, flat


def cpu_baseline(wl, args):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    procs = os.cpu_count() or 1
    t1, _ = cpu_oracle_run(wl, args, 1, 1)  # calibrate one query
    nq = int(max(procs, min(1024, args.cpu_seconds / max(t1, 1e-3))))
    nq = max(procs, (nq // procs) * procs)
    wall, rows = cpu_oracle_run(wl, args, nq, procs)
    return {"value": nq / wall, "unit": "queries/s", "cores": procs, "kind": "port",
            "sample": f"first {nq} queries of the bench workload (N={args.n}, r2={args.r2}, r={args.r}), "
                      f"oracle/derived_search.py on {procs} forked processes, {wall:.1f} s wall"}, rows


# ----------------------------------------------------------------- ours --

def run_ours(args):
    import torch

    from paper_1905_06900_b200 import _lib
    from paper_1905_06900_b200.flat import FlatIndex

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        return run_sharded(args, rank, world, local) if args.mode == "shard" else run_replicas(args, rank, world, local)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    wl = build_workload(args, device)
    idx = FlatIndex.from_arrays(wl["codebooks"], wl["derived"], wl["codes"], device=local)
    h = idx._handle()
    stream = torch.cuda.Stream(device=device)
    h.set_stream(stream.cuda_stream)
    h.set_batch(args.batch)
    Bq, r, r2 = args.batch, args.r, args.r2
    qdev = wl["queries_dev"]
    out_d = torch.empty((Bq, r), dtype=torch.float64, device=device)
    out_i = torch.empty((Bq, r), dtype=torch.int64, device=device)
    all_ids = np.empty((qdev.shape[0], r), np.int64)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)  # > 126 MB L2
    L = _lib.lib()

    def step(s):
        q = qdev[s * Bq:(s + 1) * Bq]
        rc = L.dpq_flat_search_derived_dev(h.raw, _lib.ptr(q), Bq, r, r2, _lib.ptr(out_d), _lib.ptr(out_i))
        _lib.check(rc, "search")

    # timed steps run as a caller's would: no phase events, so batches replay
    # as a CUDA graph (the first warm-up call sizes buffers, the second captures)
    h.set_timing(False)
    for s in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        step(s)
        all_ids[s * Bq:(s + 1) * Bq] = out_i.cpu().numpy()
    c0 = h.counters()
    torch.cuda.synchronize()
    evs = []
    with ClockSampler(local) as clk:
        for s in range(args.warmup, args.warmup + args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            step(s)
            with torch.cuda.stream(stream):
                e1.record(stream)
            evs.append((e0, e1))
            all_ids[s * Bq:(s + 1) * Bq] = out_i.cpu().numpy()
        torch.cuda.synchronize()
    c1 = h.counters()
    # per-phase CUDA-event times (incl. the scan launch for the roofline) from
    # a separate instrumented pass over the first timed batches
    phase = []
    h.set_timing(True)
    for s in range(args.warmup, args.warmup + min(args.steps, 3)):
        with torch.cuda.stream(stream):
            flush.zero_()
        step(s)
        phase.append(h.phase_ms().copy())
    h.set_timing(False)
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    phase = np.array(phase)
    value = args.steps * Bq / (total_ms / 1e3)
    timed = slice(args.warmup * Bq, (args.warmup + args.steps) * Bq)
    recall = float((all_ids[timed, :r] == wl["truth"][timed, :1]).any(axis=1).mean())
    launches = c1["launches"] - c0["launches"]
    refined = c1["refined"] - c0["refined"]
    # dominant kernel: the first-pass scan (K2b) — timed by the library's
    # events around that launch on the same stream
    scan_ms = float(np.mean(phase[:, 2]))
    alg_bytes = float(args.n) * M * 2 * Bq  # N_scanned * m * 2 B per query
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
        else {"hbm_gbs": 6650.0}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = alg_bytes / (scan_ms / 1e3) / 1e9
    phases = {k: round(float(np.mean(phase[:, i])), 4) for i, k in
              enumerate(["tables", "guard", "scan", "threshold", "refine", "fallback", "batch"])}
    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        qh = wl["queries"]
        times = []
        h.set_timing(False)  # a caller's search has no phase events (return_timings=False)
        for s in range(args.warmup):  # untimed e2e warm-up (first-call imports, pinned staging, graph)
            idx.search(qh[s * Bq:(s + 1) * Bq], r, mode="derived", r2=r2)
        for s in range(args.warmup, args.warmup + args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            stream.synchronize()
            t0 = time.perf_counter()
            d, i = idx.search(qh[s * Bq:(s + 1) * Bq], r, mode="derived", r2=r2)
            times.append(time.perf_counter() - t0)
            assert np.array_equal(i, all_ids[s * Bq:(s + 1) * Bq]), "e2e results differ from device run"
        e2e = {"value": args.steps * Bq / sum(times), "unit": "queries/s",
               "h2d_bytes_per_step": Bq * D * 4, "d2h_bytes_per_step": Bq * r * 16,
               "step_ms": [round(1e3 * t, 3) for t in times],
               "api": "FlatIndex.search(Y_host, 100, mode='derived', r2=1000) -> libdpq C ABI"}
    # comparator: conventional 16-bit search (flat.py:82-93) on a query sample
    nconv = min(256, args.steps * Bq)
    sel = slice(args.warmup * Bq, args.warmup * Bq + nconv)
    _, ic = idx.search(wl["queries"][sel], r)
    recall_conv = float((ic[:, :r] == wl["truth"][sel, :1]).any(axis=1).mean())
    recall_der_same = float((all_ids[sel, :r] == wl["truth"][sel, :1]).any(axis=1).mean())
    cpu = None
    parity = None
    if not args.no_cpu_baseline:
        cpu, rows = cpu_baseline(wl, args)
        # parity on the sampled queries (same inputs, same codes)
        ok = 0
        for qi, ids, ds, _ in rows:
            got = all_ids[qi]
            ok += int(np.array_equal(got[: len(ids)], ids))
        parity = {"queries_checked": len(rows), "ids_identical": ok}
    clocks = clk.summary()
    result = {
        "metric": "queries/s at Recall@100 (flat derived search, PQ 4x16 + derived 4x8, N=10M, r2=1000, k=100)",
        "value": round(value, 1), "unit": "queries/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8/u16 scan, f32 tables, f64 distances",
        "data": "synthetic (seeded SIFT-like stand-in; GPU-trained 4x16/8 codebooks)",
        "config": {"workload": "BASELINE configs[1]: flat PQ4x16+derived4x8, N=10M, batch 1024, r2=1000, k=100",
                   "n": args.n, "batch": Bq, "r": r, "r2": r2, "recall_at_100": round(recall, 4),
                   "l2": "flushed (256 MB write) between timed steps", "train_vectors": args.train,
                   "parallelism": "single GPU"},
        "recall_at_100": round(recall, 4),
        "recall_vs_conventional": {"queries": nconv, "derived": round(recall_der_same, 4),
                                   "conventional_16bit": round(recall_conv, 4)},
        "phase_ms": phases,
        "roofline": {"bound": "hbm", "kernel": "k_scan_emit (first-pass scan)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 3), "traffic": scan_traffic(),
                     "note": "achieved = algorithmic bytes (SURVEY 8d: N*m*2 B of codes per query x 1024 queries "
                             "per launch) / CUDA-event time of the launch; frac > 1 because one pass over the "
                             "4 B/code plane serves a 128-query tile, runs of equal (g0, g1) share half the "
                             "gathers and the run filter skips ~88% of the rows (DESIGN.md 1, 4); traffic = "
                             "DRAM read + write bytes per launch from profiles/r1_ncu_full_metrics.json, "
                             "mostly the emitted candidate lists",
                     "per_launch_ms": round(scan_ms, 4),
                     "physical": physical_roofline(scan_ms, peak)},
        "cpu_baseline": cpu, "parity_sample": parity,
        "e2e": e2e, "gpu_launches": int(launches),
        "candidates_per_query": round(refined / max(1, args.steps * Bq), 1),
        "emitted_per_query": round((c1["emitted"] - c0["emitted"]) / max(1, args.steps * Bq), 1),
        "table_entries_per_query": round((c1["table_entries"] - c0["table_entries"]) / max(1, args.steps * Bq), 1),
        "clocks": clocks, "setup_s": round(wl["setup_s"], 1),
    }
    print(json.dumps(result), flush=True)


def physical_roofline(scan_ms, peak):
    """The scan against HBM with the bytes it really moves (ncu DRAM traffic
    per launch / the live launch time): how far below the HBM roof the
    shared-memory-gather / ALU-bound kernel runs."""
    t = scan_traffic()
    if not t or not scan_ms:
        return None
    gbs = t / (scan_ms * 1e-3) / 1e9
    return {"dram_bytes_per_launch": t, "achieved_gbs": round(gbs, 1), "frac_of_hbm": round(gbs / peak, 4),
            "limiter": "shared-memory LUT gathers + hit emission (ncu: issue active 74%, ALU pipe 66%)"}


def scan_traffic():
    """DRAM bytes (read + write) of one k_scan_emit launch, from the
    committed ncu --set full capture of the same command (profiles/)."""
    try:
        prof = json.loads((ROOT / "profiles" / "r1_ncu_full_metrics.json").read_text())
        for k in prof["kernels"]:
            if "k_scan_emit" in k["kernel"]:
                return int(k["traffic_bytes"])
    except (OSError, ValueError, KeyError):
        pass
    return None


def run_replicas(args, rank, world, local):
    """N > 1 for configs[1]: the 10M index fits one GPU, so queries are the
    unit of parallelism (tier rule: shard independent units, no data-path
    collective).  Every rank holds the whole index (codebooks trained on rank
    0 and broadcast) and searches its own 1024-query batches; the step time is
    the max over ranks, value = all ranks' queries / that time (weak scaling:
    per-GPU work is fixed)."""
    import torch
    import torch.distributed as dist

    from paper_1905_06900_b200 import _lib
    from paper_1905_06900_b200.flat import FlatIndex

    ngpu = max(1, torch.cuda.device_count())
    local = local % ngpu  # (functional runs with more ranks than GPUs use gloo)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    nccl = world <= ngpu
    if nccl:
        dist.init_process_group("nccl", device_id=device)
    else:
        dist.init_process_group("gloo")
    cdev = device if nccl else torch.device("cpu")
    wl = build_workload(args, device, rank, world, shard=False, comm_device=cdev)
    idx = FlatIndex.from_arrays(wl["codebooks"], wl["derived"], wl["codes"], device=local)
    h = idx._handle()
    stream = torch.cuda.Stream(device=device)
    h.set_stream(stream.cuda_stream)
    h.set_batch(args.batch)
    Bq, r, r2 = args.batch, args.r, args.r2
    qdev, qh = wl["queries_dev"], wl["queries"]
    out_d = torch.empty((Bq, r), dtype=torch.float64, device=device)
    out_i = torch.empty((Bq, r), dtype=torch.int64, device=device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    L = _lib.lib()
    mine = lambda s: slice((s * world + rank) * Bq, (s * world + rank + 1) * Bq)  # noqa: E731
    hits = 0

    def step(s):
        rc = L.dpq_flat_search_derived_dev(h.raw, _lib.ptr(qdev[mine(s)]), Bq, r, r2, _lib.ptr(out_d),
                                           _lib.ptr(out_i))
        _lib.check(rc, "search")

    for s in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        step(s)
    torch.cuda.synchronize()
    c0 = h.counters()
    evs = []
    with ClockSampler(local) as clk:
        for s in range(args.warmup, args.warmup + args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            stream.synchronize()
            dist.barrier()
            with torch.cuda.stream(stream):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            step(s)
            with torch.cuda.stream(stream):
                e1.record(stream)
            evs.append((e0, e1))
            stream.synchronize()
            ids = out_i.cpu().numpy()
            hits += int((ids == wl["truth"][mine(s), :1]).any(axis=1).sum())
    c1 = h.counters()
    dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    # e2e: the public API with host queries, same per-rank batches
    wall = 0.0
    if not args.no_e2e:
        for s in range(args.warmup):
            idx.search(qh[mine(s)], r, mode="derived", r2=r2)
        for s in range(args.warmup, args.warmup + args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            stream.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            idx.search(qh[mine(s)], r, mode="derived", r2=r2)
            wall += time.perf_counter() - t0
    tot = torch.tensor([dev_ms, wall, c1["launches"] - c0["launches"], hits], dtype=torch.float64, device=cdev)
    mx = tot.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = tot.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    clocks = clk.summary()
    if rank == 0:
        total_ms = float(mx[0])
        nq = world * args.steps * Bq
        recall = float(sm[3]) / nq
        result = {
            "metric": "queries/s at Recall@100 (flat derived search, PQ 4x16 + derived 4x8, N=10M, r2=1000, k=100)",
            "value": round(nq / (total_ms / 1e3), 1), "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8/u16 scan, f32 tables, f64 distances",
            "data": "synthetic (seeded SIFT-like stand-in; GPU-trained 4x16/8 codebooks)",
            "config": {"workload": "BASELINE configs[1] (N=10M fits one GPU): query-parallel replicas",
                       "n": args.n, "batch": Bq, "r": r, "r2": r2, "recall_at_100": round(recall, 4),
                       "l2": "flushed (256 MB write) before each timed step",
                       "parallelism": f"dp{world}: every GPU holds the index and searches its own 1024-query "
                                      "batches; step time = max over ranks"},
            "recall_at_100": round(recall, 4),
            "e2e": None if args.no_e2e else {
                "value": round(nq / float(mx[1]), 1), "unit": "queries/s",
                "h2d_bytes_per_step": world * Bq * D * 4, "d2h_bytes_per_step": world * Bq * r * 16,
                "api": "FlatIndex.search(Y_host, 100, mode='derived', r2=1000) per rank, max wall over ranks"},
            "gpu_launches": int(sm[2]), "clocks": clocks, "setup_s": round(wl["setup_s"], 1),
        }
        print(json.dumps(result), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def run_sharded(args, rank, world, local):
    """N > 1: the 10M database split into `world` contiguous shards (strong
    scaling of one database); each batch runs the split API with NCCL
    all-reduces of the score histograms and an all-gather of the per-shard
    top-r (paper_1905_06900_b200/shard.py)."""
    import torch
    import torch.distributed as dist

    from paper_1905_06900_b200.shard import GpuShardEngine, TorchComm, sharded_search

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=device)
    wl = build_workload(args, device, rank, world)
    eng = GpuShardEngine(wl["codebooks"], wl["derived"], wl["codes"], wl["row_base"], args.n, wl["prefix"],
                         device=local)
    stream = torch.cuda.current_stream(device)
    eng.handle.set_stream(stream.cuda_stream)
    comm = TorchComm(device=device)
    Bq, r, r2 = args.batch, args.r, args.r2
    qh = wl["queries"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    ids_all = np.empty((qh.shape[0], r), np.int64)
    for s in range(args.warmup):
        flush.zero_()
        _, i = sharded_search(eng, comm, qh[s * Bq:(s + 1) * Bq], r, r2)
        ids_all[s * Bq:(s + 1) * Bq] = i
    c0 = eng.handle.counters()
    step_ms, wall = [], []
    with ClockSampler(local) as clk:
        for s in range(args.warmup, args.warmup + args.steps):
            flush.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(stream)
            _, i = sharded_search(eng, comm, qh[s * Bq:(s + 1) * Bq], r, r2)
            e1.record(stream)
            torch.cuda.synchronize()
            wall.append(time.perf_counter() - t0)
            step_ms.append(e0.elapsed_time(e1))
            ids_all[s * Bq:(s + 1) * Bq] = i
    c1 = eng.handle.counters()
    tot = torch.tensor([sum(step_ms), sum(wall), c1["launches"] - c0["launches"]], dtype=torch.float64,
                       device=device)
    mx = tot.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = tot.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    if rank == 0:
        total_ms = float(mx[0])
        timed = slice(args.warmup * Bq, (args.warmup + args.steps) * Bq)
        recall = float((ids_all[timed, :r] == wl["truth"][timed, :1]).any(axis=1).mean())
        result = {
            "metric": "queries/s at Recall@100 (flat derived search, PQ 4x16 + derived 4x8, N=10M, r2=1000, k=100)",
            "value": round(args.steps * Bq / (total_ms / 1e3), 1), "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8/u16 scan, f32 tables, f64 distances",
            "data": "synthetic (seeded SIFT-like stand-in; GPU-trained 4x16/8 codebooks)",
            "config": {"workload": "BASELINE configs[1] database split into contiguous shards, one per GPU",
                       "n": args.n, "batch": Bq, "r": r, "r2": r2, "recall_at_100": round(recall, 4),
                       "l2": "flushed (256 MB write) before each timed step",
                       "parallelism": f"database sharded x{world}, NCCL all-reduce of score histograms + "
                                      "all-gather of per-shard top-r"},
            "recall_at_100": round(recall, 4),
            "e2e": {"value": round(args.steps * Bq / float(mx[1]), 1), "unit": "queries/s",
                    "h2d_bytes_per_step": Bq * D * 4, "d2h_bytes_per_step": Bq * r * 16,
                    "api": "shard.sharded_search (host queries -> dpq_shard_* C ABI -> host results)"},
            "gpu_launches": int(sm[2]), "clocks": clk.summary(), "setup_s": round(wl["setup_s"], 1),
        }
        print(json.dumps(result), flush=True)
    dist.barrier()
    dist.destroy_process_group()


# ------------------------------------------------------------- reference --

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    wl = build_workload(args, torch.device("cuda", local))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    procs = os.cpu_count() or 1
    t1, _ = cpu_oracle_run(wl, args, 1, 1)
    per_step = max(procs, int(max(1.0, 8.0 / max(t1, 1e-3)) // procs) * procs)  # ~8 s CPU per step
    per_step = min(per_step, args.batch)
    for s in range(args.warmup):
        cpu_oracle_run(wl, args, per_step, procs)
    walls = []
    for s in range(args.steps):
        w, _ = cpu_oracle_run(wl, args, per_step, procs)
        walls.append(w)
    value = args.steps * per_step / sum(walls)
    out = {
        "impl": "reference",
        "metric": "queries/s at Recall@100 (flat derived search, PQ 4x16 + derived 4x8, N=10M, r2=1000, k=100)",
        "value": round(value, 3), "unit": "queries/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(walls) / args.steps, 2), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "numpy (u8 scan, f32 tables, f64 distances)", "data": "synthetic",
        "config": {"workload": "BASELINE configs[1]: flat PQ4x16+derived4x8, N=10M, batch 1024, r2=1000, k=100",
                   "n": args.n, "r": args.r, "r2": args.r2},
        "cpu_baseline": {"value": round(value, 3), "unit": "queries/s", "cores": procs, "kind": "port",
                         "sample": f"{per_step} queries per step on {procs} forked processes "
                                   "(oracle/derived_search.py restating derivedpq)"},
        "e2e": {"value": round(value, 3), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
