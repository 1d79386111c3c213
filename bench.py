"""Benchmark: queries/sec at fixed Recall@100 of the derived two-pass PQ search.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 (default): BASELINE.json configs[1], the metric's single-GPU config —
flat PQ 4x16 + derived 4x8 over N = 10M SIFT-like codes (seeded synthetic
stand-in for SIFT, data="synthetic"), 1024-query steps, R (r2) = 1000,
k (r) = 100.  A step = one batch of 1024 queries through the whole derived
path (tables, guard, scan, threshold, refine + top-k).

N > 1 (torchrun, one process per GPU): BASELINE.json configs[2] — OPQ 4x16 +
derived 4x8 over N = 100M codes split into N contiguous shards (strong
scaling of one database).  Each step runs the shard protocol on the device
(SURVEY §8e): per-shard tables and scan, NCCL all-reduces of the score
histograms (b* identical on every GPU), per-shard refine + top-k, NCCL
all-gather and a device (dist, id) merge.  `--mode replicas` instead runs
query-parallel replicas of configs[1] (no exchange).

Prints ONE JSON line on rank 0.  `value` = device-timed queries/s (CUDA
events on the search stream, inputs resident in HBM, L2 flushed before every
timed step, max over ranks); `e2e` = the public API (FlatIndex.search /
ShardedFlatIndex.search) with host numpy queries in and results out.

`--impl reference` times the UNMODIFIED reference (`derivedpq`, installed in
baseline/_ref) through its own public API FlatIndex.search(Y, 100,
mode="derived", r2=R) on the host cores (rank 0 only), with codes injected
as SURVEY §8c describes.  Its workload (codebooks, codes, queries) is built
by a child process that exits before the reference is loaded, so no repo
shared library is ever mapped into the timing process (checked against
/proc/self/maps).  Both arms print the same `config` dict.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
REF_PATH = ROOT / "baseline" / "_ref"

METRIC = "queries/s at Recall@100 (derived two-pass PQ search, k=100)"


def shard_n1_record():
    """The shard workload (configs[2]) measured on ONE B200 with `bench.py --mode shard --gpus 1`, as
    recorded under profiles/: the N = 1 line of a driver scaling run is configs[1] (the metric's
    single-GPU config, 10M rows), so this is the same-workload point N > 1 lines compare with."""
    src = ROOT / "profiles" / "r2_bench_shard_n1_c3_final.json"
    try:
        line = [l for l in src.read_text().splitlines() if l.startswith("{")][-1]
        d = json.loads(line)
        return {"value": d["value"], "unit": d["unit"], "ms_per_step": d["ms_per_step"],
                "e2e": (d.get("e2e") or {}).get("value"), "recorded": str(src.relative_to(ROOT)),
                "note": "recorded run, not measured in this one"}
    except Exception:
        return None


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default=None, choices=["c2", "c3", "c5"],
                   help="workload (default: c2 = configs[1] at N=1; c3 = configs[2] when sharded)")
    p.add_argument("--mode", default=None, choices=["shard", "replicas"],
                   help="N > 1: database sharded over the GPUs (default) or query-parallel replicas of configs[1]")
    p.add_argument("--n", "--rows", dest="n", type=int, default=None)
    p.add_argument("--batch", type=int, default=None)
    p.add_argument("--r", type=int, default=100)
    p.add_argument("--r2", type=int, default=None)
    p.add_argument("--train", type=int, default=100_000)
    p.add_argument("--kmeans-iters", type=int, default=12)
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--cpu-seconds", type=float, default=20.0, help="wall budget of the cpu_baseline leg")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-comparator", action="store_true",
                   help="skip the fixed-recall comparator (conventional mode + r2 grid): ncu launch lists")
    p.add_argument("--emit-workload", default=None, help=argparse.SUPPRESS)  # internal: reference-arm child
    return p.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def resolve(args, world: int):
    """(cfg, mode) of this run; identical in both arms."""
    from paper_1905_06900_b200 import workloads

    mode = args.mode or ("shard" if world > 1 else "single")  # (--mode shard at N = 1: the protocol on one GPU)
    name = args.config or ("c3" if mode == "shard" else "c2")
    cfg = dict(workloads.CONFIGS[name])
    if args.n:
        cfg["n"] = args.n
    if args.r2:
        cfg["r2"] = args.r2
    if args.batch:
        cfg["batch"] = args.batch
    cfg["r"] = args.r
    return cfg, mode


def config_dict(cfg, args, world: int, mode: str) -> dict:
    """The `config` object both arms print (same keys and values)."""
    par = {"single": "single GPU",
           "shard": f"database split into {world} contiguous shards, one per GPU; NCCL all-reduce of the score "
                    "histograms + all-gather of per-shard top-k with a device merge",
           "replicas": f"{world} query-parallel replicas (every GPU holds the index)"}[mode]
    return {"workload": cfg["label"], "baseline_config": cfg["baseline"], "n": cfg["n"], "m": cfg["m"],
            "dsub": cfg["dsub"], "batch": cfg["batch"], "r": cfg["r"], "r2": cfg["r2"],
            "l2": "flushed (256 MB write) before every timed step", "train_vectors": args.train,
            "seed": args.seed, "parallelism": par}


def dtype_str(cfg):
    return "u8 low-byte scan, u16 codes, f32 tables, f64 distances"


DATA = "synthetic (seeded SIFT/GIST-like stand-in, BASELINE generator; GPU-trained codebooks, GPU-encoded codes)"


# ------------------------------------------------------------------ setup --

def build_flat(cfg, args, device, lo: int, hi: int, nq: int, rank: int = 0, world: int = 1, comm_dev=None):
    """Model (trained on rank 0, broadcast), codes of rows [lo, hi), nq
    queries, exact rank-0 ground truth over the WHOLE database (per-shard
    truths merged)."""
    import torch

    from paper_1905_06900_b200 import workloads

    t0 = time.time()
    m, dsub = cfg["m"], cfg["dsub"]
    if rank == 0:
        cb, der, rot = workloads.train_model(cfg, args.seed, device, args.train, args.kmeans_iters)
    if world > 1:
        import torch.distributed as dist

        cd = comm_dev or device
        shp_cb, shp_d = (m, 65536, dsub), (m, 256, dsub)
        cbt = torch.as_tensor(cb, device=cd) if rank == 0 else torch.empty(shp_cb, device=cd)
        dt = torch.as_tensor(der, device=cd) if rank == 0 else torch.empty(shp_d, device=cd)
        dist.broadcast(cbt, 0)
        dist.broadcast(dt, 0)
        cb, der = cbt.cpu().numpy(), dt.cpu().numpy()
        R0 = workloads.data_rotation(cfg, args.seed)
        rot = None if R0 is None else np.ascontiguousarray(R0.T)
    t1 = time.time()
    centres, _ = workloads.centres_of(cfg, args.seed)
    Y = workloads.queries(cfg, args.seed, nq)
    truth = workloads.StreamingTruth(Y, device)
    codes = workloads.encode_rows(cfg, cb, rot, centres, args.seed, lo, hi, device, truth=truth)
    td, ti = truth.result()
    if world > 1:
        import torch.distributed as dist

        cd = comm_dev or device
        parts_d = [torch.empty(nq, dtype=torch.float64, device=cd) for _ in range(world)]
        parts_i = [torch.empty(nq, dtype=torch.int64, device=cd) for _ in range(world)]
        dist.all_gather(parts_d, torch.as_tensor(td, device=cd))
        dist.all_gather(parts_i, torch.as_tensor(ti, device=cd))
        tr = workloads.merge_truth([(a.cpu().numpy(), b.cpu().numpy()) for a, b in zip(parts_d, parts_i)])
    else:
        tr = ti
    del truth
    torch.cuda.empty_cache()
    t2 = time.time()
    log(f"[rank {rank}] setup: train {t1 - t0:.1f}s, data+encode+truth {t2 - t1:.1f}s")
    return {"codebooks": cb, "derived": der, "rotation": rot, "codes": codes, "row_base": lo, "queries": Y,
            "truth": tr, "setup_s": t2 - t0}


def recall_at(ids, truth, r):
    """recall_at_r (evaluation.py:76-92): fraction of queries whose exact
    rank-0 neighbour is among the first r returned ids."""
    return float((ids[:, :r] == np.asarray(truth)[:, None]).any(axis=1).mean())


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


# ------------------------------------------------- the reference (CPU) --

_REF = {}


def import_reference():
    """The unmodified reference package from baseline/_ref (pip-installed
    copy of /root/reference/pkg), or None when it is not installed."""
    if str(REF_PATH) not in sys.path:
        sys.path.insert(0, str(REF_PATH))
    try:
        import derivedpq  # noqa: F401
        from derivedpq import FlatIndex, ProductQuantizer

        return FlatIndex, ProductQuantizer
    except ImportError:
        return None


def reference_index(codebooks, derived, rotation, codes):
    """A fitted derivedpq.FlatIndex over the given model and codes: the
    quantizer's fitted attributes are set directly and the codes injected as
    `codes_` / `n_`, so the reference searches exactly the
    arrays the GPU searches."""
    FlatIndex, ProductQuantizer = import_reference()
    m, k, dsub = codebooks.shape
    kbar = derived.shape[1]
    pq = ProductQuantizer(m=m, b=int(k).bit_length() - 1, bbar=int(kbar).bit_length() - 1, seed=42)
    pq.codebooks_ = np.ascontiguousarray(codebooks, np.float32)
    pq.derived_codebooks_ = np.ascontiguousarray(derived, np.float32)
    pq.derived_assignments_ = np.tile((np.arange(k) & (kbar - 1)).astype(np.int32), (m, 1))
    pq.distortions_ = np.zeros(m)
    pq.rotation_ = None if rotation is None else np.ascontiguousarray(rotation, np.float32)
    pq.d_, pq.dsub_, pq.k_, pq.kbar_, pq.bbar_ = m * dsub, dsub, k, kbar, int(kbar).bit_length() - 1
    pq.code_dtype_ = np.uint16
    pq.validate()
    idx = FlatIndex(pq)
    idx.codes_ = np.ascontiguousarray(codes)
    idx.n_ = idx.codes_.shape[0]
    return idx


def _ref_worker(span):
    lo, hi = span
    w = _REF
    if w["kind"] == "reference":
        d, i = w["index"].search(w["queries"][lo:hi], w["r"], mode="derived", r2=w["r2"])
    else:  # labelled fallback: the oracle port (oracle/derived_search.py)
        from oracle import derived_search as O

        d, i = O.flat_search(w["codebooks"], w["derived"], w["codes"], w["queries"][lo:hi], w["r"], "derived",
                             w["r2"], rotation=w["rotation"])
    return lo, d, i


class CpuReference:
    """The reference's CPU search path on this host: `procs` forked worker
    processes (index arrays shared copy-on-write, BLAS single-threaded),
    each searching a contiguous slice of the queries through the reference's
    public API; procs = 1 runs in-process (the reference's own model)."""

    def __init__(self, wl, r, r2, procs):
        import multiprocessing as mp

        from threadpoolctl import threadpool_limits

        self._limits = threadpool_limits(1)
        kind = "reference" if import_reference() is not None else "port"
        _REF.clear()
        _REF.update(kind=kind, queries=wl["queries"], r=r, r2=r2, codebooks=wl["codebooks"],
                    derived=wl["derived"], codes=wl["codes"], rotation=wl["rotation"])
        if kind == "reference":
            _REF["index"] = reference_index(wl["codebooks"], wl["derived"], wl["rotation"], wl["codes"])
        self.kind = kind
        self.procs = procs
        self.pool = mp.get_context("fork").Pool(procs) if procs > 1 else None

    def run(self, q0: int, nq: int):
        """Search queries [q0, q0 + nq); returns (wall s, dists, ids)."""
        per = (nq + self.procs - 1) // self.procs
        spans = [(s, min(q0 + nq, s + per)) for s in range(q0, q0 + nq, per)]
        t0 = time.perf_counter()
        res = self.pool.map(_ref_worker, spans) if self.pool else [_ref_worker(sp) for sp in spans]
        wall = time.perf_counter() - t0
        res.sort(key=lambda t: t[0])
        return wall, np.concatenate([d for _, d, _ in res]), np.concatenate([i for _, _, i in res])

    def close(self):
        if self.pool:
            self.pool.close()
            self.pool.join()


def mapped_repo_libs():
    """Shared objects of this repository mapped into the calling process."""
    try:
        maps = Path("/proc/self/maps").read_text()
    except OSError:
        return []
    return sorted({ln.split()[-1] for ln in maps.splitlines()
                   if ln.split()[-1].endswith(".so") and str(ROOT) in ln.split()[-1]
                   and "baseline/_ref" not in ln})


def cpu_baseline(wl, cfg, args, gpu_ids):
    """Bounded sample of the workload through the reference's CPU path on
    all host cores (plus a one-process figure); parity of the GPU ids
    against it on the same queries."""
    procs = os.cpu_count() or 1
    one = CpuReference(wl, cfg["r"], cfg["r2"], 1)
    t1, _, _ = one.run(0, 1)
    n1 = int(max(1, min(16, 5.0 / max(t1, 1e-3))))
    w1, d1, i1 = one.run(0, n1)
    one.close()
    ref = CpuReference(wl, cfg["r"], cfg["r2"], procs)
    nq = int(max(procs, min(len(wl["queries"]), args.cpu_seconds * procs / max(t1, 1e-3))))
    nq = max(procs, (nq // procs) * procs)
    wall, d, i = ref.run(0, nq)
    ref.close()
    same = int(sum(np.array_equal(i[q], gpu_ids[q]) for q in range(nq)))
    return ({"value": nq / wall, "unit": "queries/s", "cores": procs, "kind": ref.kind,
             "sample": f"queries [0, {nq}) of this run's workload through "
                       f"{'derivedpq.FlatIndex.search (baseline/_ref, unmodified)' if ref.kind == 'reference' else 'the oracle port'}"
                       f" on {procs} forked processes, {wall:.1f} s wall",
             "single_process": {"value": n1 / w1, "queries": n1, "wall_s": round(w1, 2)}},
            {"queries_checked": nq, "ids_identical": same, "against": ref.kind})


# ----------------------------------------------------------------- ours --

def roofline(cfg, nb, ms_scan, dc, peak, ms_refine=None):
    """The first-pass scan against HBM, from counters read in this run: plane
    rows the scan read (MPAD B each: the rows of the (g0, g1) runs a query can
    hit for k_scan_direct, the listed chunks per query tile for k_scan_emit),
    LUT tiles bulk-copied into shared memory (k_scan_emit, 128 KB each) and
    the emitted (row, score) records written, per launch, over the CUDA-event
    time of the scan launches."""
    mpad = 4 if cfg["m"] <= 4 else 8
    rec = 4 if (cfg["n"] < (1 << 24) and cfg["m"] == 4) else 8  # emit record width (dpq_flat_create)
    steps = max(1, dc["launch_batches"])
    plane_b = dc["plane_rows"] * mpad / steps
    lut_b = dc["lut_loads"] * 128 * 1024 / steps
    emit_b = dc["emitted"] * rec / steps
    moved = plane_b + lut_b + emit_b
    achieved = moved / (ms_scan * 1e-3) / 1e9
    alg = float(cfg["n"]) * cfg["m"] * 2 * nb  # N * m * 2 B of codes per query
    traffic = None
    try:  # ncu --set full capture of this command (profiles/), DRAM read + write per launch
        prof = json.loads((ROOT / "profiles" / "ncu_scan_traffic.json").read_text())
        if prof.get("config") == cfg["name"]:
            traffic = int(prof["traffic_bytes"])
    except (OSError, ValueError, KeyError):
        pass
    out = {"bound": "hbm", "kernel": "first-pass scan, K2 (k_scan_direct per query over its (g0, g1) runs; "
                                     "k_scan_emit for query tiles left to it)",
           "achieved": round(achieved, 1),
           "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
           "bytes_per_launch": {"plane": int(plane_b), "lut": int(lut_b), "emit": int(emit_b)},
           "per_launch_ms": round(ms_scan, 4),
           "counters": "dpq_counters_ex: plane rows read, LUT tile loads, emitted records",
           "traffic_source": "profiles/ncu_scan_traffic.json (ncu --set full of this config), else null",
           "algorithmic": {"bytes_per_launch": alg, "gbs": round(alg / (ms_scan * 1e-3) / 1e9, 1),
                           "frac": round(alg / (ms_scan * 1e-3) / 1e9 / peak, 3),
                           "note": "SURVEY 8d: N*m*2 B of codes per query x the batch; far above 1 because the "
                                   "rows are sorted by (g0, g1) and a query only reads the runs whose two "
                                   "entries fit under its guard (0.3% of the rows on this data)"},
           "limiter": "instruction issue and load/atomic latency of the per-query compaction (plane rows are "
                      "re-read from L2 by the queries that share a run), not DRAM"}
    if ms_refine:
        # second pass (K5 + K6, the largest share of the step): per candidate a code row (m x code bytes),
        # its emit record and m exact table entries (4 B each) gathered, over the refine phase time
        cand = dc["refined"] / steps
        rb = cand * (cfg["m"] * 2 + rec + cfg["m"] * 4)
        out["second_pass"] = {"kernel": "k_group_tables_reg + k_refine_topk (K5 + K6)",
                              "bytes_per_launch": int(rb), "per_launch_ms": round(ms_refine, 4),
                              "achieved": round(rb / (ms_refine * 1e-3) / 1e9, 1), "unit": "GB/s",
                              "frac": round(rb / (ms_refine * 1e-3) / 1e9 / peak, 4),
                              "limiter": "gather latency, exact (dist, id) selection barriers (issue ~59%)"}
    return out


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6546.2)), "MEASURED_PEAKS.json hbm_gbs"
    return 7700.0, "B200_PROFILING.md fallback"


def run_single(args, cfg):
    import torch

    from paper_1905_06900_b200 import _lib
    from paper_1905_06900_b200.flat import FlatIndex

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    Bq, r, r2 = cfg["batch"], cfg["r"], cfg["r2"]
    nsteps = args.warmup + args.steps
    wl = build_flat(cfg, args, device, 0, cfg["n"], nsteps * Bq)
    idx = FlatIndex.from_arrays(wl["codebooks"], wl["derived"], wl["codes"], rotation=wl["rotation"],
                                device=local)
    h = idx._handle()
    stream = torch.cuda.Stream(device=device)
    h.set_stream(stream.cuda_stream)
    h.set_batch(Bq)
    from paper_1905_06900_b200.flat import rotated_queries

    yr_all = rotated_queries(idx.quantizer, wl["queries"])  # reference call shape (1, d) per query
    qdev = torch.as_tensor(yr_all, device=device)
    out_d = torch.empty((Bq, r), dtype=torch.float64, device=device)
    out_i = torch.empty((Bq, r), dtype=torch.int64, device=device)
    all_ids = np.empty((qdev.shape[0], r), np.int64)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)  # > 126 MB L2
    L = _lib.lib()

    def step(s):
        q = qdev[s * Bq:(s + 1) * Bq]
        _lib.check(L.dpq_flat_search_derived_dev(h.raw, _lib.ptr(q), Bq, r, r2, _lib.ptr(out_d), _lib.ptr(out_i)),
                   "search")

    # timed steps run as a caller's would: no phase events, so batches replay
    # as a CUDA graph (the first warm-up call sizes buffers, the second captures)
    h.set_timing(False)
    for s in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        step(s)
        all_ids[s * Bq:(s + 1) * Bq] = out_i.cpu().numpy()
    torch.cuda.synchronize()
    c0 = h.counters_ex()
    evs = []
    with ClockSampler(local) as clk:
        for s in range(args.warmup, nsteps):
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
    c1 = h.counters_ex()
    # per-phase CUDA-event times (incl. the scan launch) from an instrumented
    # pass over the first timed batches, with its own counter deltas
    phase = []
    h.set_timing(True)
    p0 = h.counters_ex()
    nph = min(args.steps, 3)
    for s in range(args.warmup, args.warmup + nph):
        with torch.cuda.stream(stream):
            flush.zero_()
        step(s)
        phase.append(h.phase_ms().copy())
    h.set_timing(False)
    torch.cuda.synchronize()
    p1 = h.counters_ex()
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    phase = np.array(phase)
    value = args.steps * Bq / (total_ms / 1e3)
    timed = slice(args.warmup * Bq, nsteps * Bq)
    recall = recall_at(all_ids[timed], wl["truth"][timed], r)
    dc = {k: p1[k] - p0[k] for k in p1}
    dc["launch_batches"] = nph
    peak, peak_src = peaks()
    phases = {k: round(float(np.mean(phase[:, i])), 4) for i, k in
              enumerate(["tables", "guard", "scan", "threshold", "refine", "fallback", "batch"])}
    rl = roofline(cfg, Bq, float(np.mean(phase[:, 2])), dc, peak, float(np.mean(phase[:, 4])))
    rl["peak_source"] = peak_src
    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        qh = wl["queries"]
        times = []
        for s in range(args.warmup):  # untimed e2e warm-up (first-call imports, pinned staging, graph)
            idx.search(qh[s * Bq:(s + 1) * Bq], r, mode="derived", r2=r2)
        for s in range(args.warmup, nsteps):
            with torch.cuda.stream(stream):
                flush.zero_()
            stream.synchronize()
            t0 = time.perf_counter()
            d, i = idx.search(qh[s * Bq:(s + 1) * Bq], r, mode="derived", r2=r2)
            times.append(time.perf_counter() - t0)
            assert np.array_equal(i, all_ids[s * Bq:(s + 1) * Bq]), "e2e results differ from device run"
        e2e = {"value": round(args.steps * Bq / sum(times), 1), "unit": "queries/s",
               "h2d_bytes_per_step": Bq * qh.shape[1] * 4, "d2h_bytes_per_step": Bq * r * 16,
               "step_ms": [round(1e3 * t, 3) for t in times],
               "api": f"FlatIndex.search(Y_host, {r}, mode='derived', r2={r2}) -> libdpq C ABI"}
    extra = {} if args.no_comparator else comparator(idx, wl, cfg, args, all_ids, stream, flush)
    cpu = parity = None
    if not args.no_cpu_baseline:
        cpu, parity = cpu_baseline(wl, cfg, args, all_ids)
    result = {
        "metric": METRIC, "value": round(value, 1), "unit": "queries/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": dtype_str(cfg), "data": DATA,
        "config": config_dict(cfg, args, 1, "single"),
        "recall_at_100": round(recall, 4),
        "phase_ms": phases, "roofline": rl, "cpu_baseline": cpu, "parity_sample": parity, "e2e": e2e,
        "gpu_launches": int(c1["launches"] - c0["launches"]),
        "candidates_per_query": round((c1["refined"] - c0["refined"]) / max(1, args.steps * Bq), 1),
        "emitted_per_query": round((c1["emitted"] - c0["emitted"]) / max(1, args.steps * Bq), 1),
        "table_entries_per_query": round((c1["table_entries"] - c0["table_entries"]) / max(1, args.steps * Bq), 1),
        "clocks": clk.summary(), "setup_s": round(wl["setup_s"], 1),
    }
    result.update(extra)
    print(json.dumps(result), flush=True)


R2_GRID = (1000, 2000, 5000, 10_000, 20_000, 50_000, 100_000, 200_000)


def comparator(idx, wl, cfg, args, der_ids, stream, flush):
    """The paper's operating point on the same queries: the conventional
    16-bit search (flat.py:82-93) as the recall reference, the smallest r2 of
    a grid whose derived Recall@100 reaches 99% of it (calibrate_r2,
    evaluation.py:95-128, restated), and queries/s of both through the public
    API (host buffers) at that fixed recall."""
    import torch

    Bq, r = cfg["batch"], cfg["r"]
    cal = slice(args.warmup * Bq, args.warmup * Bq + Bq)  # calibration batch
    Y, truth = wl["queries"][cal], wl["truth"][cal]

    def timed(fn, reps=3):
        best = []
        for _ in range(reps):
            with torch.cuda.stream(stream):
                flush.zero_()
            stream.synchronize()
            t0 = time.perf_counter()
            out = fn()
            best.append(time.perf_counter() - t0)
        return out, statistics.median(best)

    idx.search(Y[:8], r)  # warm-up (sizes the full-table buffers)
    (_, ic), t_conv = timed(lambda: idx.search(Y, r), reps=1)
    full = recall_at(ic, truth, r)
    r2_fix, rec_fix = R2_GRID[-1], None
    for r2 in R2_GRID:
        if r2 > cfg["n"]:
            break
        _, i = idx.search(Y, r, mode="derived", r2=r2)
        rec = recall_at(i, truth, r)
        if rec >= 0.99 * full:
            r2_fix, rec_fix = r2, rec
            break
    if rec_fix is None:
        _, i = idx.search(Y, r, mode="derived", r2=r2_fix)
        rec_fix = recall_at(i, truth, r)
    idx.search(Y, r, mode="derived", r2=r2_fix)  # warm-up (graph of this configuration)
    _, t_der = timed(lambda: idx.search(Y, r, mode="derived", r2=r2_fix))
    return {"fixed_recall": {
        "queries": Bq, "rule": "smallest grid r2 with derived Recall@100 >= 0.99 x conventional (calibrate_r2)",
        "r2_grid": list(R2_GRID), "conventional_16bit": {"recall_at_100": round(full, 4),
                                                         "qps_e2e": round(Bq / t_conv, 1)},
        "derived": {"r2": r2_fix, "recall_at_100": round(rec_fix, 4), "qps_e2e": round(Bq / t_der, 1)},
        "derived_at_bench_r2": {"r2": cfg["r2"],
                                "recall_at_100": round(recall_at(der_ids[cal], truth, r), 4)}}}


# ------------------------------------------------------------ multi-GPU --

def init_dist(local):
    import torch
    import torch.distributed as dist

    ngpu = max(1, torch.cuda.device_count())
    local = local % ngpu  # (functional runs with more ranks than GPUs use gloo)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if "RANK" not in os.environ:  # a single process without torchrun (--mode shard at N = 1)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.update(RANK="0", LOCAL_RANK=str(local), WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(port))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    nccl = world <= ngpu
    if nccl:
        dist.init_process_group("nccl", device_id=device)
    else:
        dist.init_process_group("gloo")
    log(f"[rank {dist.get_rank()}] communicator: backend={dist.get_backend()} nranks={dist.get_world_size()} "
        f"device={device} nccl={torch.cuda.nccl.version() if nccl else None}")
    return device, local, nccl


def run_replicas(args, cfg, rank, world, local):
    """Query-parallel replicas of configs[1]: every rank holds the whole
    index and searches its own batches; step time = max over ranks, value =
    all ranks' queries / that time (weak scaling, no data-path collective)."""
    import torch
    import torch.distributed as dist

    from paper_1905_06900_b200 import _lib
    from paper_1905_06900_b200.flat import FlatIndex

    device, local, nccl = init_dist(local)
    cdev = device if nccl else torch.device("cpu")
    Bq, r, r2 = cfg["batch"], cfg["r"], cfg["r2"]
    nsteps = args.warmup + args.steps
    wl = build_flat(cfg, args, device, 0, cfg["n"], nsteps * Bq * world, rank, 1, cdev)
    idx = FlatIndex.from_arrays(wl["codebooks"], wl["derived"], wl["codes"], rotation=wl["rotation"], device=local)
    h = idx._handle()
    stream = torch.cuda.Stream(device=device)
    h.set_stream(stream.cuda_stream)
    h.set_batch(Bq)
    qdev = torch.as_tensor(wl["queries"], device=device)
    out_d = torch.empty((Bq, r), dtype=torch.float64, device=device)
    out_i = torch.empty((Bq, r), dtype=torch.int64, device=device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    L = _lib.lib()
    mine = lambda s: slice((s * world + rank) * Bq, (s * world + rank + 1) * Bq)  # noqa: E731
    hits = 0

    def step(s):
        _lib.check(L.dpq_flat_search_derived_dev(h.raw, _lib.ptr(qdev[mine(s)]), Bq, r, r2, _lib.ptr(out_d),
                                                 _lib.ptr(out_i)), "search")

    for s in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        step(s)
    torch.cuda.synchronize()
    c0 = h.counters()
    evs = []
    with ClockSampler(local) as clk:
        for s in range(args.warmup, nsteps):
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
            hits += int((out_i.cpu().numpy() == wl["truth"][mine(s)][:, None]).any(axis=1).sum())
    c1 = h.counters()
    dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    wall = 0.0
    if not args.no_e2e:
        for s in range(args.warmup):
            idx.search(wl["queries"][mine(s)], r, mode="derived", r2=r2)
        for s in range(args.warmup, nsteps):
            with torch.cuda.stream(stream):
                flush.zero_()
            stream.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            idx.search(wl["queries"][mine(s)], r, mode="derived", r2=r2)
            wall += time.perf_counter() - t0
    tot = torch.tensor([dev_ms, wall, c1["launches"] - c0["launches"], hits], dtype=torch.float64, device=cdev)
    mx, sm = tot.clone(), tot.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    if rank == 0:
        nq = world * args.steps * Bq
        print(json.dumps({
            "metric": METRIC, "value": round(nq / (float(mx[0]) / 1e3), 1), "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(float(mx[0]) / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_str(cfg), "data": DATA,
            "config": config_dict(cfg, args, world, "replicas"), "recall_at_100": round(float(sm[3]) / nq, 4),
            "e2e": None if args.no_e2e else {
                "value": round(nq / float(mx[1]), 1), "unit": "queries/s",
                "h2d_bytes_per_step": world * Bq * wl["queries"].shape[1] * 4,
                "d2h_bytes_per_step": world * Bq * r * 16,
                "api": "FlatIndex.search(Y_host, ...) per rank, max wall over ranks"},
            "gpu_launches": int(sm[2]), "clocks": clk.summary(), "setup_s": round(wl["setup_s"], 1),
            "n1_same_workload": shard_n1_record()}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def run_sharded(args, cfg, rank, world, local):
    """configs[2]: the database split into `world` contiguous shards; every
    step runs the device-resident shard protocol (shard.DeviceShardSearch:
    C-ABI phases on device buffers, NCCL all-reduces of the histograms,
    all-gather + device merge of the per-shard top-k)."""
    import torch
    import torch.distributed as dist

    from paper_1905_06900_b200.flat import ArrayQuantizer, rotated_queries
    from paper_1905_06900_b200.shard import ShardedFlatIndex

    device, local, nccl = init_dist(local)
    cdev = device if nccl else torch.device("cpu")
    Bq, r, r2 = cfg["batch"], cfg["r"], cfg["r2"]
    n = cfg["n"]
    lo, hi = rank * n // world, (rank + 1) * n // world
    nsteps = args.warmup + args.steps
    wl = build_flat(cfg, args, device, lo, hi, nsteps * Bq, rank, world, cdev)
    npre = min(n, r2)
    pt = (torch.as_tensor(wl["codes"][:npre].astype(np.int32), device=cdev) if rank == 0
          else torch.empty((npre, cfg["m"]), dtype=torch.int32, device=cdev))
    dist.broadcast(pt, 0)  # the replicated global prefix (qmax rows, twopass.py:83-84)
    prefix = pt.cpu().numpy().astype(np.uint16)
    quant = ArrayQuantizer(wl["codebooks"], wl["derived"], wl["rotation"])
    sidx = ShardedFlatIndex(quant, wl["codes"], lo, n, prefix, device=local, batch=Bq)
    eng = sidx.engine
    stream = eng.stream
    qh = wl["queries"]
    ydev = torch.as_tensor(rotated_queries(quant, qh), device=device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    ids_all = np.empty((qh.shape[0], r), np.int64)
    for s in range(args.warmup):
        _, i = eng.search_dev(ydev[s * Bq:(s + 1) * Bq], r, r2)
        ids_all[s * Bq:(s + 1) * Bq] = i.cpu().numpy()
    c0 = eng.handle.counters()
    step_ms = []
    with ClockSampler(local) as clk:
        for s in range(args.warmup, nsteps):
            with torch.cuda.stream(stream):
                flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            with torch.cuda.stream(stream):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            _, i = eng.search_dev(ydev[s * Bq:(s + 1) * Bq], r, r2)
            with torch.cuda.stream(stream):
                e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            ids_all[s * Bq:(s + 1) * Bq] = i.cpu().numpy()
    c1 = eng.handle.counters()
    wall = 0.0
    if not args.no_e2e:
        for s in range(args.warmup):
            sidx.search(qh[s * Bq:(s + 1) * Bq], r, mode="derived", r2=r2)
        for s in range(args.warmup, nsteps):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            _, i = sidx.search(qh[s * Bq:(s + 1) * Bq], r, mode="derived", r2=r2)
            wall += time.perf_counter() - t0
            assert np.array_equal(i, ids_all[s * Bq:(s + 1) * Bq]), "e2e results differ from device run"
    tot = torch.tensor([sum(step_ms), wall, c1["launches"] - c0["launches"]], dtype=torch.float64, device=cdev)
    mx, sm = tot.clone(), tot.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    if rank == 0:
        timed = slice(args.warmup * Bq, nsteps * Bq)
        print(json.dumps({
            "metric": METRIC, "value": round(args.steps * Bq / (float(mx[0]) / 1e3), 1), "unit": "queries/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(float(mx[0]) / args.steps, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": dtype_str(cfg), "data": DATA,
            "config": config_dict(cfg, args, world, "shard"),
            "recall_at_100": round(recall_at(ids_all[timed], wl["truth"][timed], r), 4),
            "e2e": None if args.no_e2e else {
                "value": round(args.steps * Bq / float(mx[1]), 1), "unit": "queries/s",
                "h2d_bytes_per_step": Bq * qh.shape[1] * 4, "d2h_bytes_per_step": Bq * r * 16,
                "api": "ShardedFlatIndex.search(Y_host, ...) on every rank (max wall over ranks)"},
            "gpu_launches": int(sm[2]), "clocks": clk.summary(), "setup_s": round(wl["setup_s"], 1),
            "n1_same_workload": shard_n1_record()}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def run_ours(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg, mode = resolve(args, world)
    if mode == "single":
        return run_single(args, cfg)
    if mode == "replicas":
        return run_replicas(args, cfg, rank, world, local)
    return run_sharded(args, cfg, rank, world, local)


# ------------------------------------------------------------- reference --

def emit_workload(args):
    """Reference-arm child: build the workload on the GPU (this process maps
    libdpq.so for the encoder and exits), run OUR search on the reference's
    query sample for the parity check, save everything the reference needs."""
    import torch

    from paper_1905_06900_b200.flat import FlatIndex

    world = int(os.environ.get("DPQ_BENCH_WORLD", "1"))
    cfg, mode = resolve(args, world)
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    nq = int(os.environ.get("DPQ_BENCH_NQ", "2048"))
    wl = build_flat(cfg, args, device, 0, cfg["n"], nq)
    idx = FlatIndex.from_arrays(wl["codebooks"], wl["derived"], wl["codes"], rotation=wl["rotation"], device=local)
    d, i = idx.search(wl["queries"], cfg["r"], mode="derived", r2=cfg["r2"])
    np.savez(args.emit_workload, codebooks=wl["codebooks"], derived=wl["derived"], codes=wl["codes"],
             queries=wl["queries"], truth=wl["truth"], gpu_d=d, gpu_i=i,
             rotation=wl["rotation"] if wl["rotation"] is not None else np.zeros(0, np.float32))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    cfg, mode = resolve(args, world)
    procs = os.cpu_count() or 1
    nq_pool = 4096
    with tempfile.TemporaryDirectory(prefix="dpq_ref_") as tmp:
        path = os.path.join(tmp, "workload.npz")
        env = dict(os.environ, DPQ_BENCH_WORLD=str(world), DPQ_BENCH_NQ=str(nq_pool))
        for k in ("RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "GROUP_RANK", "ROLE_RANK", "TORCHELASTIC_RUN_ID"):
            env.pop(k, None)
        cmd = [sys.executable, str(Path(__file__).resolve()), "--emit-workload", path] + \
            [a for a in sys.argv[1:] if a not in ("--impl", "reference")]
        t0 = time.time()
        subprocess.run(cmd, check=True, env=env, stdout=sys.stderr)
        z = np.load(path)
        wl = {k: z[k] for k in z.files}
    setup_s = time.time() - t0
    if wl["rotation"].size == 0:
        wl["rotation"] = None
    r, r2 = cfg["r"], cfg["r2"]
    # calibration and the one-process figure (the reference's own model)
    one = CpuReference(wl, r, r2, 1)
    t1, _, _ = one.run(0, 1)
    n1 = int(max(1, min(8, 4.0 / max(t1, 1e-3))))
    w1, _, _ = one.run(1, n1)
    one.close()
    ref = CpuReference(wl, r, r2, procs)
    per_step = procs * int(max(1, min(8, 2.0 / max(t1, 1e-3))))  # ~2 s of work per process per step
    per_step = min(per_step, nq_pool // max(1, args.warmup + args.steps)) or procs
    walls, got_i = [], {}
    q = 0
    for s in range(args.warmup + args.steps):
        w, _, i = ref.run(q, per_step)
        if s >= args.warmup:
            walls.append(w)
        for k in range(per_step):
            got_i[q + k] = i[k]
        q += per_step
    ref.close()
    value = args.steps * per_step / sum(walls)
    qs = sorted(got_i)
    same = int(sum(np.array_equal(got_i[k], wl["gpu_i"][k]) for k in qs))
    ids = np.stack([got_i[k] for k in qs])
    libs = mapped_repo_libs()
    assert not libs, f"repo shared objects mapped into the reference process: {libs}"
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sum(walls) / args.steps, 2),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "numpy (u8 scan, f32 tables, f64 distances)", "data": DATA,
        "config": config_dict(cfg, args, world, mode),
        "cpu_baseline": {"value": round(value, 3), "unit": "queries/s", "cores": procs, "kind": ref.kind,
                         "sample": f"{per_step} queries per step through derivedpq.FlatIndex.search(Y, {r}, "
                                   f"mode='derived', r2={r2}) (baseline/_ref, unmodified) on {procs} forked "
                                   "processes, codes injected (SURVEY 8c)"},
        "single_process": {"value": round(n1 / w1, 3), "queries": n1, "cores": 1},
        "e2e": {"value": round(value, 3), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "recall_at_100_sample": round(recall_at(ids, wl["truth"][qs], r), 4),
        "parity_vs_ours": {"queries": len(qs), "ids_identical": same},
        "native_so_loaded": libs, "setup_s": round(setup_s, 1),
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.emit_workload:
        emit_workload(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
