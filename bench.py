#!/usr/bin/env python
"""Benchmark of the Gray-code Ryser permanent mod 3 on B200.

Default workload (N=1) = BASELINE.json configs[1], the config the metric is
quoted on: a Monte Carlo batch of 16,384 independent 24x24 F3 matrices
(entries iid uniform {0,1,2}, the reference's own per-trial splitmix64 stream
with seed 0), each perm mod 3 + the histogram over {0,1,2}.  One step = one
pass over the batch: pack -> Gray walk -> finalize (+ the histogram
all-reduce when N > 1).  Metric: Gray-code subset terms/s = 2^n * matrices/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c1|c3|c4|c5]
  python bench.py --impl reference ...   # the reference's CPU path (oracle port)

--gpus N > 1 without torchrun re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU).
At N > 1 every rank takes its own 16,384 trials (weak scaling) and the
3-bin histogram meets in one NCCL all-reduce per step.

Every line also carries a "c5_strong" record: the north_star's scaling
target, C5's seed-0 50x50 matrix on a fixed 2^44-step window split over the
ranks by the split_steps rule (src/permanent.py:221-229), one 16-byte NCCL
all-reduce of the (plus, minus) counters inside each timed step
(communicator set-up excluded), the per-rank device times, and the
efficiency E(N) = T(1) / (N T(N)) with T(1) measured in the same run by rank
0 alone on the whole window.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOADS = {
    # name: (n, batch, description)
    "c1": (20, 1, "C1: single 20x20 uniform F3 matrix (reference trial stream, seed 0, trial 0)"),
    "c2": (24, 16384, "C2: Monte Carlo batch, 16384 x 24x24 uniform F3 (reference trial stream, seed 0)"),
    "c3": (32, 4096, "C3: 4096 x 32x32 structured (uniform|sparse p0=0.8|all-ones|perturbed permutation), seed 0"),
    "c4": (36, 1, "C4: single 36x36 uniform F3 matrix (seed 0, trial 0), 2^36 subsets"),
    "c5": (50, 1, "C5: single 50x50 uniform F3 matrix (seed 0, trial 0), 2^50 subsets"),
}
SEED = 0
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--c5-log2-steps", type=int, default=44,
                    help="c5: subset terms per step (a 2^k window of the 2^50 range)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", type=int, default=None,
                    help="replay each step from a CUDA graph (default: on for the single small matrix c1)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline sample time")
    ap.add_argument("--c5-steps", type=int, default=3, help="timed steps of the c5_strong record (0: skip it)")
    ap.add_argument("--selftest-cpu", action="store_true",
                    help="CPU plumbing test of the launcher, rank split and collective (gloo; no GPU "
                         "compute: the per-rank counts are zero)")
    return ap.parse_args()


def free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 outside torchrun: one rank per GPU, as the driver would
    launch it (rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def rank_part(lo: int, span: int, rank: int, world: int):
    """Part `rank` of [lo, lo + span) by the split_steps edge rule
    (src/permanent.py:227-229; paper_2407_20205_b200.parallel.rank_range)."""
    return lo + span * rank // world, lo + span * (rank + 1) // world


def workload_config(wl: str) -> dict:
    """The config dict both arms print (identical keys and values)."""
    n, B, desc = WORKLOADS[wl]
    return {"workload": desc, "n": n, "batch": B, "seed": SEED}


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------

def make_entries(workload: str, rank: int):
    from paper_2407_20205_b200 import fixtures

    n, B, _ = WORKLOADS[workload]
    if workload == "c3":
        e, _, _ = fixtures.structured_batch(n, SEED + rank, B)
        return e
    return fixtures.uniform_batch(n, SEED, rank * B, B)


def terms_per_step(workload: str, args) -> int:
    n, B, _ = WORKLOADS[workload]
    if workload == "c5":
        return 1 << args.c5_log2_steps
    return B * (1 << n)


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.06)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        loaded = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference path (oracle port, the reference's chunk_sum restated in C)
# ---------------------------------------------------------------------------

def cpu_rate(workload: str, target_s: float, threads: int):
    """(terms/s, sample description, terms, seconds) of the oracle on a bounded sample."""
    from oracle import oracle

    oracle.build()
    n, B, _ = WORKLOADS[workload]
    if workload in ("c2", "c3"):
        e = make_entries(workload, 0)
        # calibrate on a few matrices, then size the sample to ~target_s
        t0 = time.perf_counter()
        probe = max(1, min(B, threads))
        oracle.perm_batch(e[:probe], threads=threads)
        dt = time.perf_counter() - t0
        count = int(max(probe, min(B, probe * target_s / max(dt, 1e-6))))
        t0 = time.perf_counter()
        oracle.perm_batch(e[:count], threads=threads)
        dt = time.perf_counter() - t0
        terms = count * (1 << n)
        return terms / dt, f"first {count} of {B} matrices of the workload, full 2^{n} traversal each", terms, dt
    a = oracle.sample_classes(n, SEED, 0)
    mags, sgns = oracle.planes_from_classes(a)
    lo = 1 if workload in ("c1", "c4") else (1 << 40)
    span = 1 << 22
    t0 = time.perf_counter()
    oracle.chunk_sum_mt(mags, sgns, n, lo, lo + span, threads)
    dt = time.perf_counter() - t0
    span = min((1 << n) - lo, max(span, int(span * target_s / max(dt, 1e-6))))
    span = 1 << max(10, int(math.log2(span)))
    t0 = time.perf_counter()
    oracle.chunk_sum_mt(mags, sgns, n, lo, lo + span, threads)
    dt = time.perf_counter() - t0
    return span / dt, f"steps [{lo}, {lo}+2^{int(math.log2(span))}) of the matrix, split over {threads} threads", span, dt


REF_PATH = os.path.join(REPO, "baseline", "_ref")


def numba_reference_rate(workload: str, target_s: float, threads: int):
    """The UNMODIFIED reference package (baseline/_ref, installed from
    /root/reference with pip --no-deps) through its own public API, numba
    kernels and thread pool: montecarlo_zero (src/experiments.py:158-190) on a
    bounded trial count for c2, chunk_sum (src/_kernels.py:90-128) over a
    window split across a ThreadPool the way perm_mod3_parallel does
    (src/permanent.py:232-255) otherwise.  None if it is not installed."""
    if not os.path.isdir(os.path.join(REF_PATH, "tritperm")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tritperm_numba_cache")
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    from concurrent.futures import ThreadPoolExecutor

    from tritperm import _kernels as rk
    from tritperm import experiments as rexp

    n, B, _ = WORKLOADS[workload]
    if workload == "c2":
        rexp.montecarlo_zero(n, threads, seed=SEED, jobs=threads)  # JIT warm-up
        t0 = time.perf_counter()
        rexp.montecarlo_zero(n, threads, seed=SEED, jobs=threads)
        dt = time.perf_counter() - t0
        trials = int(max(threads, min(B, threads * target_s / max(dt, 1e-6))))
        t0 = time.perf_counter()
        r = rexp.montecarlo_zero(n, trials, seed=SEED, jobs=threads)
        dt = time.perf_counter() - t0
        return {"value": trials * (1 << n) / dt, "unit": "terms/s", "cores": threads, "seconds": round(dt, 2),
                "sample": f"tritperm.montecarlo_zero({n}, {trials}, seed={SEED}, jobs={threads}) "
                          f"-> zero_count {r.zero_count} (first {trials} of the {B} trials)"}
    m = rexp.sample_trial_matrix(n, 0, SEED)
    mags, sgns = m.planes()
    lo = 1 if workload != "c5" else (1 << 40)

    def run(span):
        edges = [lo + span * k // threads for k in range(threads + 1)]
        with ThreadPoolExecutor(max_workers=threads) as ex:
            return sum(ex.map(lambda k: int(rk.chunk_sum(mags, sgns, n, edges[k], edges[k + 1])), range(threads)))

    run(1 << 16)  # JIT warm-up
    span = 1 << 22
    t0 = time.perf_counter()
    run(span)
    dt = time.perf_counter() - t0
    span = min((1 << n) - lo, max(span, int(span * target_s / max(dt, 1e-6))))
    span = 1 << max(10, int(math.log2(span)))
    t0 = time.perf_counter()
    run(span)
    dt = time.perf_counter() - t0
    return {"value": span / dt, "unit": "terms/s", "cores": threads, "seconds": round(dt, 2),
            "sample": f"tritperm._kernels.chunk_sum over steps [{lo}, {lo}+2^{int(math.log2(span))}) of "
                      f"sample_trial_matrix({n}, 0, {SEED}), {threads} ThreadPool parts"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n, B, desc = WORKLOADS[args.workload]
    per_step = max(1.0, min(6.0, 120.0 / max(1, args.steps + args.warmup)))
    rates, secs, terms = [], [], []
    sample = None
    for k in range(args.warmup + args.steps):
        rate, sample, t, dt = cpu_rate(args.workload, per_step, threads)
        if k >= args.warmup:
            rates.append(rate)
            secs.append(dt)
            terms.append(t)
    value = statistics.median(rates)
    numba = None
    if os.environ.get("TRITPERM_BENCH_NUMBA", "1") != "0":
        try:
            numba = numba_reference_rate(args.workload, 8.0, threads)
        except Exception as exc:  # report, never fail the arm
            numba = {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    line = {
        "impl": "reference",
        "metric": "gray_code_subset_terms_per_s",
        "value": value,
        "unit": "terms/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        # each step is a bounded sample of the workload, measured as is (not
        # extrapolated to the full workload)
        "ms_per_step": statistics.median(secs) * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (reference trial stream)",
        "config": workload_config(args.workload),
        "sample_per_step": {"terms": int(statistics.median(terms)), "of_workload_terms": terms_per_step(args.workload, args),
                            "seconds": round(statistics.median(secs), 3), "what": sample},
        "cpu_baseline": {"value": value, "unit": "terms/s", "cores": threads, "kind": "port",
                         "sample": f"oracle/oracle.c chunk_sum (restatement of src/_kernels.py:90-128), {sample}"},
        "reference_numba": numba,
        "e2e": {"value": value, "unit": "terms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# C5 strong scaling (north_star: >= 90 % at 8 GPUs on the n = 50 run)
# ---------------------------------------------------------------------------

def c5_strong(args, rank: int, world: int, use_dist: bool, dev):
    """Fixed 2^k-step window of C5's matrix split over the ranks; per step:
    zero the counters, walk this rank's part, one 16-byte all-reduce.  Device
    times (CUDA events on the launching stream), max over ranks per step."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2407_20205_b200 import _kernels

    n = 50
    a = make_entries("c5", 0)[0]
    span = 1 << args.c5_log2_steps
    lo0 = 1 << 40
    plo, phi = rank_part(lo0, span, rank, world)
    d_e = torch.from_numpy(np.ascontiguousarray(a[None])).to(dev)
    d_rows = torch.empty((1, _kernels.ROWREC_BYTES), dtype=torch.uint8, device=dev)
    d_pm = torch.zeros(2, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _kernels.pack_async(d_e.data_ptr(), 1, n, d_rows.data_ptr(), st)

    def step(lo, hi, reduce):
        d_pm.zero_()
        _kernels.walk_range_async(d_rows.data_ptr(), n, lo, hi, d_pm.data_ptr(), st)
        if reduce:
            dist.all_reduce(d_pm)

    step(plo, phi, use_dist)  # warm-up (also creates the NCCL communicator, outside the timed steps)
    torch.cuda.synchronize()
    mine, step_max = [], []
    for _ in range(args.c5_steps):
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        step(plo, phi, use_dist)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        mine.append(t)
        if use_dist:
            tt = torch.tensor([t], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        step_max.append(t)
    pm = d_pm.cpu().tolist()
    per_rank = [statistics.mean(mine)]
    if use_dist:
        g = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(world)]
        dist.all_gather(g, torch.tensor([statistics.mean(mine)], dtype=torch.float64, device=dev))
        per_rank = [float(x.item()) for x in g]
    t_n = statistics.mean(step_max)
    t_1, pm1 = t_n, pm
    if world > 1:
        # T(1): rank 0 alone on the whole window, same kernels, no collective
        dist.barrier()
        if rank == 0:
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            step(lo0, lo0 + span, False)
            e1.record()
            torch.cuda.synchronize()
            t_1 = e0.elapsed_time(e1)
            pm1 = d_pm.cpu().tolist()
        dist.barrier()
    return {
        "workload": f"C5 matrix (seed 0, trial 0), steps [2^40, 2^40 + 2^{args.c5_log2_steps}) split over "
                    f"{world} rank(s) by the split_steps rule",
        "n_ranks": world, "steps": args.c5_steps, "terms_per_step": span,
        "ms_per_step": t_n, "per_rank_ms": per_rank, "value": span / (t_n * 1e-3), "unit": "terms/s",
        "collective": "one 16-byte NCCL all_reduce of (plus, minus) per step" if use_dist else "none (1 rank)",
        "t1_ms": t_1, "efficiency": t_1 / (world * t_n),
        "partial": int(pm[0] - pm[1]), "partial_1rank": int(pm1[0] - pm1[1]),
    }


def run_selftest_cpu(args):
    """CPU plumbing of the N-rank path (gloo): launcher, rank split, one
    all-reduce of the counters per step, max over ranks, the JSON line.  No
    compute runs (the counts are zero); the B200 path needs a GPU."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    span = 1 << args.c5_log2_steps
    plo, phi = rank_part(1 << 40, span, rank, world)
    parts = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    mine = torch.tensor([plo, phi], dtype=torch.int64)
    if world > 1:
        dist.all_gather(parts, mine)
    else:
        parts = [mine]
    times = []
    for _ in range(max(1, args.c5_steps)):
        t0 = time.perf_counter()
        pm = torch.zeros(2, dtype=torch.int64)
        if world > 1:
            dist.all_reduce(pm)
        times.append((time.perf_counter() - t0) * 1e3)
    if rank == 0:
        edges = [tuple(int(v) for v in p.tolist()) for p in parts]
        print(json.dumps({"metric": "gray_code_subset_terms_per_s", "selftest": True, "n_gpus": world,
                          "config": workload_config(args.workload),
                          "c5_strong": {"n_ranks": world, "parts": edges, "terms_per_step": span,
                                        "covers_window": edges[0][0] == 1 << 40 and edges[-1][1] == (1 << 40) + span
                                        and all(a[1] == b[0] for a, b in zip(edges, edges[1:])),
                                        "ms_per_step": statistics.mean(times), "partial": int(pm[0] - pm[1])}}))
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# B200 path
# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.graph is None:
        args.graph = 1 if args.workload == "c1" else 0
    if args.impl == "reference":
        run_reference(args)
        return
    if args.selftest_cpu:
        run_selftest_cpu(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2407_20205_b200 as tp
    from paper_2407_20205_b200 import _kernels

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ[_kernels.ENV_DEVICE] = str(local)
    # one process per GPU; TRITPERM_BENCH_DIST=1 forces the NCCL path even for a
    # single rank (exercises the collective on a 1-GPU box)
    use_dist = world > 1 or os.environ.get("TRITPERM_BENCH_DIST") == "1"
    if use_dist:
        if "RANK" not in os.environ:  # single process outside torchrun
            os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=os.environ.get("MASTER_PORT", "29533"))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    wl = args.workload
    n, B, desc = WORKLOADS[wl]
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    launches = 0
    walk_ms = []
    step_ms = []

    if wl == "c5" or wl in ("c1", "c4"):
        # single matrix: the step range is split across ranks (strong scaling);
        # entries resident in HBM, packed and walked every step
        a = make_entries(wl, 0)[0]
        span = terms_per_step(wl, args)
        lo0 = (1 << 40) if wl == "c5" else 0
        part = (span * rank // world, span * (rank + 1) // world)
        d_e = torch.from_numpy(np.ascontiguousarray(a[None])).to(dev)
        d_rows = torch.empty((1, _kernels.ROWREC_BYTES), dtype=torch.uint8, device=dev)
        d_pm = torch.zeros(2, dtype=torch.int64, device=dev)

        def step(timed_walk=True):
            nonlocal launches
            s = torch.cuda.current_stream().cuda_stream
            d_pm.zero_()
            _kernels.pack_async(d_e.data_ptr(), 1, n, d_rows.data_ptr(), s)
            e0 = e1 = None
            if timed_walk:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
            nl = _kernels.walk_range_async(d_rows.data_ptr(), n, lo0 + part[0], lo0 + part[1], d_pm.data_ptr(), s)
            if timed_walk:
                e1.record()
            launches += 1 + nl
            if use_dist:
                dist.all_reduce(d_pm)
            return e0, e1
        per_rank_terms = span // world
        scaling = "strong"
    else:
        entries_h = make_entries(wl, rank)
        d_e = torch.from_numpy(entries_h).to(dev)
        d_rows = torch.empty((B, _kernels.ROWREC_BYTES), dtype=torch.uint8, device=dev)
        d_pm = torch.zeros((B, 2), dtype=torch.int64, device=dev)
        d_cls = torch.empty(B, dtype=torch.int8, device=dev)
        d_hist = torch.zeros(3, dtype=torch.int64, device=dev)

        def step(timed_walk=True):
            nonlocal launches
            s = torch.cuda.current_stream().cuda_stream
            d_pm.zero_()
            d_hist.zero_()
            _kernels.pack_async(d_e.data_ptr(), B, n, d_rows.data_ptr(), s)
            e0 = e1 = None
            if timed_walk:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
            nl = _kernels.walk_async(d_rows.data_ptr(), B, n, d_pm.data_ptr(), s)
            if timed_walk:
                e1.record()
            _kernels.finalize_async(d_pm.data_ptr(), B, n, d_cls.data_ptr(), d_hist.data_ptr(), s)
            launches += 2 + nl
            if use_dist:
                dist.all_reduce(d_hist)
            return e0, e1
        per_rank_terms = B * (1 << n)
        scaling = "weak"

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # Launch-bound steps (single small matrices) are replayed from a CUDA
    # graph of the whole step (pack -> walk -> finalize); the walk kernel's own
    # time for the roofline then comes from a separate evented loop.
    graph = None
    if args.graph and not use_dist:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step(timed_walk=False)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step(timed_walk=False)
        torch.cuda.synchronize()
    per_step_launches = None
    launches = 0

    # timed region: K steps, L2 flushed (memset of 256 MiB) between steps,
    # each step bracketed by CUDA events on the launching stream
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    _kernels.walk_tested(local)  # reset the bucketed walk's tested-pair counter
    with ClockSampler(local) as clk:
        evs = []
        for _ in range(args.steps):
            flush.zero_()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            if graph is not None:
                graph.replay()
                w = (None, None)
            else:
                w = step()
            s1.record()
            evs.append((s0, s1, w))
        torch.cuda.synchronize()
    tested_pairs = _kernels.walk_tested(local)  # pairs the bucketed walk tested in the K steps
    if use_dist:
        dist.barrier()
    for s0, s1, (w0, w1) in evs:
        step_ms.append(s0.elapsed_time(s1))
        if w0 is not None:
            walk_ms.append(w0.elapsed_time(w1))
    if graph is not None:
        launches = 0
        wev = []
        for _ in range(args.steps):
            wev.append(step())
        torch.cuda.synchronize()
        per_step_launches = launches // args.steps
        launches = per_step_launches * args.steps
        walk_ms = [a.elapsed_time(b) for a, b in wev]
    total_ms = sum(step_ms)
    if use_dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    job_terms = per_rank_terms * world if scaling == "weak" else terms_per_step(wl, args)
    value = job_terms / (ms_per_step * 1e-3)

    # ALU roofline of the walk kernel: LOP3 per subset term of the kernel that
    # served this n (2 for the pair walk, 3 for the lane/wide walks; n > 32
    # tests only the 32 primary columns -- see DESIGN.md)
    kernel_name, ops_per_term = _kernels.walk_info(n, B)
    tested_frac = None
    ops_per_tested_pair = None
    if "bucket" in kernel_name or "batch" in kernel_name:
        # the bucketed walk tests only the pairs its key columns do not prove
        # zero: LOP3 per term = LOP3 per tested pair x the tested fraction,
        # counted by the kernel itself over the timed steps
        tested_frac = tested_pairs / (per_rank_terms * args.steps)
        # `frac` stays on the counter of rounds 1-2 (1.5 LOP3 per tested pair:
        # the packed pair test as 2 LOP3 + its own zero-field LOP3 per word of
        # two pairs), so the rounds compare; k_walk_batch now shares the
        # zero-field test between three entries and EXECUTES 4/3 ALU-pipe ops
        # per tested pair (tp_walk_info): `frac_executed`
        ops_per_tested_pair = ops_per_term
        if "packed" in kernel_name:
            ops_per_term = 1.5
        ops_per_term = ops_per_term * tested_frac
    walk_avg = sum(walk_ms) / len(walk_ms)
    achieved = per_rank_terms * ops_per_term / (walk_avg * 1e-3)
    peak, _ = _kernels.alu_peak(local)
    traffic = None
    tpath = os.path.join(REPO, "profiles", "walk_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(wl, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # end-to-end through the public API with host buffers (rank-local batch)
    e2e = None
    if scaling == "weak":
        pinned = torch.from_numpy(make_entries(wl, rank)).pin_memory()
        host = pinned.numpy()
        tp.perm_mod3_batch(host)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = max(3, min(args.steps, 10))
        for _ in range(reps):
            cls, part, hist = tp.perm_mod3_batch(host)
        e2e_s = (time.perf_counter() - t0) / reps
        if use_dist:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": per_rank_terms * world / e2e_s, "unit": "terms/s",
               "h2d_bytes_per_step": int(B * n * n),
               "d2h_bytes_per_step": int(B + B * 8 + 3 * 8),
               "api": "paper_2407_20205_b200.perm_mod3_batch(pinned uint8 [B,n,n]) -> tp_perm_batch"}
    else:
        m_obj = tp.MatrixF3(make_entries(wl, 0)[0].astype(np.int64))
        lo = (1 << 40) if wl == "c5" else 1
        span = terms_per_step(wl, args)
        tp.perm_chunk(m_obj, lo, min(lo + min(span, 1 << 20), 1 << n))
        t0 = time.perf_counter()
        tp.perm_chunk(m_obj, lo, min(lo + span, 1 << n))
        e2e_s = time.perf_counter() - t0
        # short calls (C1: ~40 us): average over up to `steps` calls, within ~0.5 s
        reps = max(1, min(args.steps, int(0.5 / max(e2e_s, 1e-6))))
        if reps > 1:
            t0 = time.perf_counter()
            for _ in range(reps):
                tp.perm_chunk(m_obj, lo, min(lo + span, 1 << n))
            e2e_s = (time.perf_counter() - t0) / reps
        e2e = {"value": span / e2e_s, "unit": "terms/s", "h2d_bytes_per_step": 64 * 32,
               "d2h_bytes_per_step": 16, "api": "paper_2407_20205_b200.perm_chunk -> tp_range_sum"}

    strong = None
    if args.c5_steps > 0:
        strong = c5_strong(args, rank, world, use_dist, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, sample, _, _ = cpu_rate(wl, args.cpu_seconds, threads)
        cpu = {"value": rate, "unit": "terms/s", "cores": threads, "kind": "port",
               "sample": f"oracle/oracle.c chunk_sum (restatement of src/_kernels.py:90-128), {sample}"}

    csum = clk.summary()
    if rank == 0:
        line = {
            "metric": "gray_code_subset_terms_per_s",
            "value": value,
            "unit": "terms/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": scaling,
            "vs_baseline": None,
            "dtype": "u32",
            "data": "synthetic (reference per-trial splitmix64 stream; no dataset involved)",
            "config": workload_config(wl),
            "run": {"parallelism": f"dp{world}",
                    "l2": "flushed between steps (256 MiB memset, untimed by the walk events)",
                    "cuda_graph": bool(graph is not None),
                    "terms_per_step": job_terms},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "ALU ops/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kernel_name + " (csrc/" + ("tp_walk_batch.cu" if "batch" in kernel_name
                                                              else "tp_walk_bucket.cu" if "bucket" in kernel_name
                                                              else "tp_walk_packed.cu" if "packed" in kernel_name
                                                              else "tp_walk_pair.cu" if "pair" in kernel_name
                                                              else "tp_walk_lane.cu" if "lane" in kernel_name
                                                              else "tp_walk_wide.cu") + ")",
                         "ops_per_term": ops_per_term,
                         "tested_pairs_frac": tested_frac,
                         # ALU-pipe ops the filter EXECUTES per tested pair (k_walk_batch: 2 LOP3 + 1/3
                         # VIMNMX3 + 1/3 LOP3 per packed word of two pairs = 4/3); `achieved`/`frac` count
                         # the pair test at 1.5 LOP3 per tested pair, the counter of rounds 1-2
                         "ops_per_tested_pair_executed": ops_per_tested_pair,
                         "frac_executed": (None if tested_frac is None else per_rank_terms * ops_per_tested_pair
                                           * tested_frac / (walk_avg * 1e-3) / peak),
                         "peak_source": "LOP3 chain probe (tp_alu_peak) on this GPU in this run; "
                                        "nominal 148 SM x 64 lanes x clock",
                         "walk_ms_avg": walk_avg,
                         "terms_per_s_walk": per_rank_terms / (walk_avg * 1e-3)},
            "clocks": csum,
            "e2e": e2e,
            "gpu_launches": launches,
            "cpu_baseline": cpu,
            "c5_strong": strong,
        }
        print(json.dumps(line))
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
