#!/usr/bin/env python
"""Benchmark of the TPA-SCD hot path (Parnell et al., arXiv 1702.07005) on B200.

Headline workload (BASELINE.json configs[2], the webspam-shaped config the metric's target is quoted
on): C3 = 350,000 x 16,609,143 CSR, ~3,728 nnz/row (1.306e9 nnz, fp32 values + int32 indices =
10.4 GB, larger than the 126 MB L2), dual TPA-SCD by example, λ = 1e-3.  Generated on the device by
the seeded generator (synth/); nothing is read from disk.

A step = one local TPA-SCD epoch (scd_epoch: permutation inline, gather-dot, closed-form delta,
atomic scatter; §8(a) rows a1-a6) and, when N > 1, one optimal-gamma aggregation round over NCCL
(a8).  With N GPUs each rank holds its own 350,000-row block of a 350,000·N-row matrix (weak
scaling, global N in λN).  The gap evaluation (a7) is off the clock, as in the paper's plots.

Sub-records on the same JSON line:
  N = 1: "c2" (configs[1], dual and primal), "c4_primal" (configs[3] at K = 1: C3's matrix by feature) and "c5_shard" (one GPU's
         25 M-row shard of configs[4], implicit values), each with its epoch time, nnz/s and the
         roofline of its dominant kernel; "c3_load" (the data layer at full scale: C3 with scattered
         feature ids renumbered by frequency on the device by scd_renumber, then epochs on the result).
  N > 1: "north_star" — configs[4] criteo-shaped, weak-scaled at 25 M rows per rank (the full
         200 M x 75 M at N = 8), dual by example, time and rounds to gap 1e-4 with optimal γ and with
         the add / average baselines; and configs[3] C4 primal by feature at K = N.

`python bench.py --gpus N` with N > 1 relaunches itself under torch.distributed.run (one process per
GPU); under a launcher WORLD_SIZE must equal N.  Prints ONE JSON line (rank 0).  `--impl reference`
times the fp64 oracle (the only "reference" this paper has: it ships no code) on bounded samples of
the same workload on the host cores.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_NNZ = 16   # idx 4 + val 4 + shared-vector gather 4 + atomic 4
BYTES_PER_NNZ_IMPLICIT = 12  # val = NULL (NEXT-1): no value stream
BYTES_PER_COORD = 32  # ptr pair 16 + norm 4 + model RMW 8 + label 4
METRIC = "nnz/s per epoch"
METRIC_FULL = "time-to-duality-gap 1e-4 (s); nnz/s per epoch; HBM GB/s vs B200 peak"
C5_ROWS_PER_GPU = 25_000_000


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML in a background
    thread every 10 ms (a sample on entry and one on exit, so even a 150 ms region has ~15); falls back to
    `nvidia-smi -lms` when NVML is unavailable."""

    _REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.sm, self.mx, self.reasons = [], 0.0, set()
        self.stop = None
        self.th = None
        self.nv = None
        self.f = None
        self.p = None

    def _sample(self):
        nv, h = self.nv, self.h
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
        self.mx = max(self.mx, float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        for n, bit in self._REASONS.items():
            if r & bit:
                self.reasons.add(n)

    def __enter__(self):
        import threading

        try:
            import pynvml as nv

            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[self.gpu].isdigit() else self.gpu
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(idx)
            self._sample()
            self.stop = threading.Event()

            def loop():
                while not self.stop.wait(0.01):
                    try:
                        self._sample()
                    except Exception:
                        return

            self.th = threading.Thread(target=loop, daemon=True)
            self.th.start()
        except Exception:
            self.nv = None
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            try:
                self.p = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                     "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                     "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
            except Exception:
                self.p = None
        return self

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop.set()
            self.th.join(timeout=2)
            try:
                self._sample()
            except Exception:
                pass
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        if self.nv is None and self.f is not None:
            self.f.flush()
            self.f.seek(0)
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for line in self.f.read().splitlines():
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    self.sm.append(float(parts[0]))
                    self.mx = max(self.mx, float(parts[1]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[3:7]):
                    if v.lower() == "active":
                        self.reasons.add(n)
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml" if self.nv is not None else "nvidia-smi"}


def c3_cfg(world: int):
    import synth

    base = synth.CONFIGS["C3"]
    return base.with_rows(base.n_rows * world, name=f"C3x{world}" if world > 1 else "C3")


def host_info() -> dict:
    """The box's host (SURVEY §8(d) oracle timing protocol: nproc, CPU model, RAM)."""
    info = {"nproc": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                info["ram_gb"] = round(int(line.split()[1]) / 1e6, 1)
                break
    except OSError:
        pass
    return info


# ------------------------------------------------------------------------------------------------
# oracle (host) baselines: the only places bench.py executes oracle/
def cpu_baseline(seconds: float = 15.0, rows: int = 20_000):
    """The fp64 oracle's dual epoch (Alg. 1 / Eq. 4, sequential, 1 core) on the first ``rows`` rows
    of C3; returns nnz/s over whole epochs within ~``seconds``."""
    import oracle
    import synth
    from oracle import solver

    cfg = c3_cfg(1).with_rows(rows)
    d = synth.gen_host(cfg)
    pr = solver.Problem.from_csr(d, csc=False)
    nrm = pr.row_norms()
    alpha, wbar = np.zeros(pr.N), np.zeros(pr.M)
    done, t0, ep = 0, time.perf_counter(), 0
    while True:
        ep += 1
        solver.dual_epoch(pr, alpha, wbar, oracle.permutation(3, ep, pr.N), nrm)
        done += pr.nnz
        if time.perf_counter() - t0 >= seconds:
            break
    el = time.perf_counter() - t0
    return {"value": done / el, "unit": "nnz/s", "cores": 1, "kind": "oracle", "host": host_info(),
            "sample": f"C3 rows [0,{rows}) ({pr.nnz:.3g} nnz), {ep} sequential fp64 dual epochs (oracle.c, 1 thread)"}


def oracle_time_to_gap(d_dev, max_epochs: int = 3, target: float = 1e-4):
    """The sequential fp64 oracle on the FULL C3 (the same matrix, host copy): epoch time to gap 1e-4
    (epochs on the clock, the from-scratch gap off it; SURVEY §8(d) oracle timing protocol)."""
    import oracle
    from oracle import ridge, solver

    host = dict(ptr=d_dev["ptr"].cpu().numpy(), idx=d_dev["idx"].cpu().numpy(), val=d_dev["val"].cpu().numpy(),
                y=d_dev["y"].cpu().numpy(), n_rows=d_dev["n_rows"], n_cols=d_dev["n_cols"], lam=d_dev["lam"])
    pr = solver.Problem.from_csr(host, csc=False)
    A = pr.A()
    nrm = pr.row_norms()
    alpha, wbar = np.zeros(pr.N), np.zeros(pr.M)
    acc, gaps = 0.0, []
    for t in range(1, max_epochs + 1):
        t0 = time.perf_counter()
        solver.dual_epoch(pr, alpha, wbar, oracle.permutation(3, t, pr.N), nrm)
        acc += time.perf_counter() - t0
        gaps.append(ridge.dual_report(A, pr.y, pr.lam, alpha)[2])
        if gaps[-1] <= target:
            break
    return {"seconds": acc if gaps[-1] <= target else None, "epochs": len(gaps), "seconds_per_epoch": acc / len(gaps),
            "gap_trace": [float("%.3e" % g) for g in gaps], "cores": 1,
            "what": "full C3 (1.306e9 nnz), sequential fp64 SDCA (oracle.c), epochs to gap 1e-4"}


def cpu_baseline_dist(K: int, rows: int = 400_000, rounds: int = 8):
    """The oracle's Alg. 4 (optimal γ, dual by example) with K worker threads (SURVEY §8(d) oracle
    timing protocol for K > 1): a bounded criteo-shaped sample (`rows` rows, field cardinalities
    scaled by 1/100 so that each worker's copy of w̄ stays small), λN = 2e5 as in the C5 shards."""
    import synth
    from oracle import solver

    cfg = synth.c5_scaled(rows, 1e-2)
    d = synth.gen_host(cfg)
    pr = solver.Problem.from_csr(d, lam=2e5 / rows, csc=False)
    t0 = time.perf_counter()
    solver.run_distributed(pr, "dual", K, "optimal", rounds, seed=5, seed_part=5, record=False, threads=K)
    el = time.perf_counter() - t0
    return {"value": pr.nnz * rounds / el, "unit": "nnz/s", "cores": K, "kind": "oracle",
            "seconds_per_round": el / rounds, "host": host_info(),
            "sample": f"Alg. 4 (optimal gamma) with {K} worker threads, {rounds} rounds, criteo-shaped rows [0,{rows}) "
                      f"(fields scaled 1/100, {pr.nnz} nnz), lambda N = 2e5"}


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return 0
    # each step: one oracle dual epoch on a bounded 6000-row sample of C3 (~2.2e7 nnz)
    import oracle
    import synth
    from oracle import solver

    rows = 6000
    d = synth.gen_host(c3_cfg(1).with_rows(rows))
    pr = solver.Problem.from_csr(d, csc=False)
    nrm = pr.row_norms()
    alpha, wbar = np.zeros(pr.N), np.zeros(pr.M)
    for t in range(args.warmup):
        solver.dual_epoch(pr, alpha, wbar, oracle.permutation(3, t + 1, pr.N), nrm)
    t0 = time.perf_counter()
    for t in range(args.steps):
        solver.dual_epoch(pr, alpha, wbar, oracle.permutation(3, args.warmup + t + 1, pr.N), nrm)
    el = time.perf_counter() - t0
    v = pr.nnz * args.steps / el
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "nnz/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"C3 webspam-shaped dual TPA-SCD; reference arm = fp64 sequential oracle on a "
                                  f"bounded sample (rows [0,{rows}), {pr.nnz} nnz)", "form": "dual", "lambda": 1e-3},
           "cpu_baseline": {"value": v, "unit": "nnz/s", "cores": 1, "kind": "oracle", "host": host_info(),
                            "sample": f"C3 rows [0,{rows}) per step"},
           "e2e": {"value": v, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "note": "the paper ships no code; the reference arm is the sequential fp64 oracle (Alg. 1) on host cores"}
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------
class Ctx:
    """Per-process state shared by the legs.  BENCH_TRANSPORT=hooks (test mode only): the N ranks share
    GPU 0 and the library's collectives go through the scd_collectives host hooks over gloo
    (tests/hostcoll.py) — it exercises the N > 1 legs on a one-GPU box; its times are not results."""

    def __init__(self, rank, world, local):
        import torch

        self.torch = torch
        self.rank, self.world, self.local = rank, world, local
        self.hooks = world > 1 and os.environ.get("BENCH_TRANSPORT") == "hooks"
        self.dist = None
        self.hc = None
        if world > 1:
            import torch.distributed as dist

            if self.hooks:
                dist.init_process_group("gloo")
                sys.path.insert(0, os.path.join(ROOT, "tests"))
                from hostcoll import HostCollectives

                self.hc = HostCollectives()
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            self.dist = dist
        self.comm = None
        self.launches = 0

    def comm_kw(self):
        """The library's transport: an NCCL communicator, or (test mode) the host hooks."""
        if self.hooks:
            return dict(collectives=self.hc.struct)
        return dict(nccl_comm=self.nccl())

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        if self.dist is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cpu" if self.hooks else "cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def nccl(self):
        """The library's NCCL communicator (the library calls NCCL itself; torch only broadcasts the id)."""
        if self.world == 1:
            return None
        if self.comm is None:
            import paper_1702_07005_b200 as scd

            uid = scd.nccl_unique_id() if self.rank == 0 else bytes(128)
            t = self.torch.tensor(list(uid), dtype=self.torch.uint8, device="cuda")
            self.dist.broadcast(t, 0)
            self.comm = scd.nccl_comm_init(bytes(t.cpu().tolist()), self.world, self.rank)
        return self.comm


def kernel_roofline(s, info, kprof, bytes_per_nnz: int, el_ms: float, world: int = 1):
    """Roofline of the dominant kernel (the bin with the most device time, CUDA events on the library
    stream): ALGORITHMIC bytes per launch (16 B/nnz, 12 B/nnz with implicit values,
    + 32 B/coordinate) / average launch duration vs the measured HBM copy peak."""
    peak, peak_src = _peaks()
    bins = info["bins"]
    if not kprof:
        return None
    b_i = max(range(len(kprof)), key=lambda i: kprof[i][0])
    ms_b, cnt_b = kprof[b_i]
    bb = bins[b_i]
    # one launch processes one of the n_slices slices of the bin
    bytes_launch = (bytes_per_nnz * bb["nnz"] + BYTES_PER_COORD * bb["count"]) / info["n_slices"]
    achieved = bytes_launch / (ms_b / cnt_b / 1e3) / 1e9 if cnt_b else None
    if bb["lanes"] >= 4096:
        kname = "k_epoch_cluster_tma" if os.environ.get("SCD_CLUSTER_TMA") == "1" else "k_epoch_cluster"
    elif bb["lanes"] >= 64:
        kname = ("k_epoch_sm_tma" if info.get("sm_head") else "k_epoch_cta_head") if bb.get("head") else "k_epoch_cta"
    else:
        kname = "k_epoch_group_hot" if bb.get("hot") else ("k_epoch_group_comb" if bb["lanes"] == 8 else "k_epoch_group")
    traffic, dram_bytes, l2pct = None, None, None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            rec = tj.get(kname) if isinstance(tj.get(kname), dict) else (tj if (kname + "<") in tj.get("kernel", "") else None)
            if rec:
                traffic = rec.get("dram_bytes_per_launch")
                l2pct = rec.get("l2_tag_requests_pct")
        except Exception:
            traffic = None
    out = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
           "frac": (achieved / peak) if achieved else None, "traffic": traffic,
           "achieved_is": f"algorithmic bytes ({bytes_per_nnz} B/nnz + 32 B/coordinate, SURVEY §8(d)) per launch / "
                          "CUDA-event launch time",
           "kernel": kname, "bin": b_i, "lanes": bb["lanes"], "kernel_ms_avg": ms_b / cnt_b if cnt_b else None,
           "launches_timed": cnt_b, "kernel_share_of_step": ms_b / el_ms if el_ms else None,
           "bytes_per_launch": bytes_launch, "peak_source": peak_src}
    if l2pct is not None:
        # the resource that binds the epoch kernels: L2 tag-request throughput of the same
        # kernel in its ncu --set full capture (profiles/ncu_traffic.json)
        out["l2_tag_requests_pct_of_peak"] = l2pct
    if traffic and cnt_b:
        # measured DRAM bytes of the same kernel (ncu, per launch) over the same launch time: the shared
        # vector's gathers and REDs mostly hit L2, so this is below the algorithmic rate
        out["dram_achieved"] = traffic / (ms_b / cnt_b / 1e3) / 1e9
        out["dram_frac"] = out["dram_achieved"] / peak
    return out


def timed_epochs(ctx, s, stream, first_epoch: int, steps: int, step_fn):
    torch = ctx.torch
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    for t in range(first_epoch, first_epoch + steps):
        step_fn(t)
    ev1.record(stream)
    torch.cuda.synchronize()
    ctx.barrier()
    return ctx.max_over_ranks(ev0.elapsed_time(ev1))


def time_to_gap(ctx, s, stream, step_fn, target=1e-4, max_rounds=60, first=1000):
    """Fresh model; epoch (+ aggregation) device time accumulated until the from-scratch fp64 gap <=
    target (reading c23: the gap is evaluated off the clock after every round)."""
    torch = ctx.torch
    acc, hist, g = 0.0, [], None
    for t in range(1, max_rounds + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.barrier()
        e0.record(stream)
        step_fn(first + t)
        e1.record(stream)
        torch.cuda.synchronize()
        acc += ctx.max_over_ranks(e0.elapsed_time(e1))
        g = s.duality_gap()
        hist.append(g)
        if g <= target or not np.isfinite(g) or g > 1e6:
            break
    return {"seconds": acc / 1e3 if g is not None and g <= target else None, "rounds": len(hist),
            "gap_trace": [float("%.3e" % x) for x in hist[:40]], "target": target}


# ------------------------------------------------------------------------------------------------
def leg_c3(args, ctx):
    """The headline: C3 (webspam-shaped) dual; weak-scaled C3 x N with optimal γ per epoch at N > 1."""
    torch = ctx.torch
    import synth
    import paper_1702_07005_b200 as scd

    rank, world = ctx.rank, ctx.world
    cfg = c3_cfg(world)
    rows = args.rows or synth.CONFIGS["C3"].n_rows
    row0 = rank * rows
    t_gen = time.perf_counter()
    d = synth.gen_device(cfg, row0, rows)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    nnz = int(d["ptr"][-1].item())
    kw = dict(seed=3 + rank, n_global=rows * world, rank=rank, world=world, max_inflight=args.max_inflight,
              **ctx.comm_kw())
    t_create = time.perf_counter()
    s = scd.Solver(d["ptr"], d["idx"], d["val"], rows, cfg.n_cols, d["y"], cfg.lam, "dual", profile=True, **kw)
    t_create = time.perf_counter() - t_create
    stream = torch.cuda.ExternalStream(s.stream_handle)
    info = s.info()

    def step(t):
        s.epoch(t)
        if world > 1:
            s.aggregate("optimal")

    for t in range(1, args.warmup + 1):
        step(t)
    torch.cuda.synchronize()
    s.profile_read()  # drop warm-up kernel timings
    launches0 = s.info()["launches"]
    with ClockSampler(ctx.local) as clk:
        el_ms = timed_epochs(ctx, s, stream, args.warmup + 1, args.steps, step)
    launches = s.info()["launches"] - launches0
    kprof = s.profile_read()
    total_nnz = nnz * world
    value = total_nnz * args.steps / (el_ms / 1e3)
    ms_step = el_ms / args.steps
    roof = kernel_roofline(s, info, kprof, BYTES_PER_NNZ, el_ms, world)
    if roof and roof["kernel"] == "k_epoch_cta_head" and info.get("tail_roll"):
        roof["kernel"] += (f" (head {info['bins'][roof['bin']]['head']} floats combined, flush every "
                           f"{info['bins'][roof['bin']]['flush']}, head/tail gathers from the rolling read copies)")
    if roof and roof["kernel"] == "k_epoch_sm_tma":
        roof["kernel"] += (f" ({info['sm_head']} row groups per SM sharing the head snapshot and pending updates of "
                           f"w̄[0, {info['bins'][roof['bin']]['head']}), rows bulk-copied to shared memory in "
                           f"{info['sm_chunk']}-entry chunks, tail gathers from the rolling read copy)")

    # access-pattern ceiling on this box: the same gathers + REDs over the same matrix with no
    # algorithmic dependency (tools/pattern_bench.cu), against a scratch vector
    pattern = None
    pso = os.path.join(ROOT, "tools", "libpattern.so")
    if os.path.exists(pso) and not args.quick:
        import ctypes as C

        pl = C.CDLL(pso)
        pl.pattern_run.restype = C.c_float
        pl.pattern_run.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        scratch = torch.zeros(cfg.n_cols + 1024, device="cuda")
        sink = torch.zeros(1, device="cuda")
        pms = min(pl.pattern_run(3, d["idx"].data_ptr(), d["val"].data_ptr(), nnz, scratch.data_ptr(),
                                 sink.data_ptr()) for _ in range(2))
        pattern = {"ms": pms, "entries_per_s": nnz / (pms / 1e3), "epoch_over_pattern": ms_step / pms,
                   "what": "gather + red.add of sv[idx] for every stored entry, storage order, no dependencies"}
        if hasattr(pl, "pattern_run2"):
            pl.pattern_run2.restype = C.c_float
            pl.pattern_run2.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_void_p]
            scratch2 = torch.zeros(cfg.n_cols + 1024, device="cuda")
            pms2 = min(pl.pattern_run2(7, d["idx"].data_ptr(), d["val"].data_ptr(), nnz, scratch.data_ptr(),
                                       scratch2.data_ptr(), sink.data_ptr()) for _ in range(2))
            pattern["read_copy"] = {"ms": pms2, "entries_per_s": nnz / (pms2 / 1e3), "epoch_over_pattern": ms_step / pms2,
                                    "what": "gather of a second vector + red.add of sv[idx] for every stored entry"}
            del scratch2
        del scratch

    ttg = None
    if not args.no_ttg:
        s.set_model(np.zeros(rows, np.float32))
        ttg = time_to_gap(ctx, s, stream, step)
        ttg["epochs"] = ttg["rounds"]
    s.profile_read()

    # end to end through the public API with host buffers (pinned): upload + epochs (+ aggregation
    # over NCCL when N > 1) + model read; wall clock per rank between barriers, max over ranks
    e2e = None
    if not args.no_e2e:
        try:
            hp = torch.empty(rows + 1, dtype=torch.int64, pin_memory=True)
            hi = torch.empty(nnz, dtype=torch.int32, pin_memory=True)
            hv = torch.empty(nnz, dtype=torch.float32, pin_memory=True)
            hy = torch.empty(rows, dtype=torch.float32, pin_memory=True)
            hp.copy_(d["ptr"])
            hi.copy_(d["idx"])
            hv.copy_(d["val"])
            hy.copy_(d["y"])
            n_ep = (ttg or {}).get("rounds") or 5
            times = []
            for rep in range(5):
                torch.cuda.synchronize()
                ctx.barrier()
                t0 = time.perf_counter()
                # the public API's defaults, matrix validation included
                s2 = scd.Solver(hp, hi, hv, rows, cfg.n_cols, hy, cfg.lam, "dual", **kw)
                for t in range(1, n_ep + 1):
                    s2.epoch(t)
                    if world > 1:
                        s2.aggregate("optimal")
                s2.get_model()
                el = time.perf_counter() - t0
                s2.close()
                el = ctx.max_over_ranks(el)
                if rep > 0:
                    times.append(el)
            e_s = statistics.median(times)
            e2e = {"value": total_nnz * n_ep / e_s, "unit": "nnz/s",
                   "h2d_bytes_per_step": int(8 * (rows + 1) + 8 * nnz + 4 * rows),
                   "d2h_bytes_per_step": int(4 * rows), "epochs_per_step": n_ep, "seconds_per_step": e_s,
                   "seconds_min": min(times), "seconds_median": e_s, "value_at_min": total_nnz * n_ep / min(times),
                   "seconds_per_rep": [round(x, 4) for x in times],
                   "step": "scd_create from pinned host CSR (H2D, matrix validated) + epochs-to-gap-1e-4"
                           + (" with optimal-gamma aggregation" if world > 1 else "") + " + scd_get_model (D2H)"
                           + ("; bytes per rank" if world > 1 else "")}
            del hp, hi, hv, hy
        except Exception as ex:  # never lose the device-timed line to the e2e leg
            e2e = {"value": None, "error": f"{type(ex).__name__}: {ex}"[:300]}
    s.close()
    ctx.launches += launches
    rec = {"value": value, "ms_per_step": ms_step, "nnz": nnz, "rows": rows, "cfg": cfg, "info": info, "roofline": roof,
           "pattern": pattern, "ttg": ttg, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
           "setup_s": {"generate": t_gen, "create": t_create}}
    return rec, d


def leg_load(args, ctx, d):
    """The data layer at full scale ("ids scattered over 16.6 M and renumbered at load"):
    C3's feature ids are scattered by a random bijection of [0, M) (rows no longer sorted, no frequency
    order), scd_renumber restores a frequency ranking on the device, and the epoch runs on the result.
    Checks: the renumbered per-feature counts are non-increasing, equal to the generator's as a multiset,
    every row strictly increasing; epoch time on the renumbered matrix vs the headline's."""
    torch = ctx.torch
    import synth
    import paper_1702_07005_b200 as scd

    cfg = synth.CONFIGS["C3"]
    N, M = cfg.n_rows, cfg.n_cols
    g = torch.Generator(device="cuda")
    g.manual_seed(1234)
    perm = torch.randperm(M, generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
    idx_s = perm.index_select(0, d["idx"]).contiguous()
    del perm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rp, ri, rv, new_of_old = scd.renumber(d["ptr"], idx_s, d["val"], N, M, "csr")
    e1.record()
    torch.cuda.synchronize()
    ren_ms = e0.elapsed_time(e1)
    del idx_s
    cnt_r = torch.bincount(ri.long(), minlength=M)
    cnt_o = torch.bincount(d["idx"].long(), minlength=M)
    monotone = bool((cnt_r[1:] <= cnt_r[:-1]).all().item())
    same_counts = bool(torch.equal(torch.sort(cnt_r, descending=True).values, torch.sort(cnt_o, descending=True).values))
    rows_sorted = True
    nnz = int(rp[-1].item())
    diff = ri[1:].long() - ri[:-1].long()
    starts = torch.zeros(nnz, dtype=torch.bool, device="cuda")
    starts[rp[1:-1]] = True  # positions that begin a row
    rows_sorted = bool(((diff > 0) | starts[1:]).all().item())
    del cnt_r, cnt_o, diff, starts
    s = scd.Solver(rp, ri, rv, N, M, d["y"], cfg.lam, "dual", seed=3, profile=True)
    stream = torch.cuda.ExternalStream(s.stream_handle)
    info = s.info()
    for t in range(1, 4):
        s.epoch(t)
    torch.cuda.synchronize()
    el = timed_epochs(ctx, s, stream, 4, 5, lambda t: s.epoch(t))
    gap = s.duality_gap()
    s.close()
    del rp, ri, rv, new_of_old
    torch.cuda.empty_cache()
    return {"workload": "C3 with feature ids scattered by a random bijection, renumbered by frequency on the device "
                        "(scd_renumber), then the dual epochs on the renumbered matrix",
            "renumber_ms": ren_ms, "nnz": nnz,
            "checks": {"counts_non_increasing": monotone, "counts_equal_generator_multiset": same_counts,
                       "rows_strictly_increasing": rows_sorted},
            "epoch_ms": el / 5, "gap_after_8_epochs": gap, "sm_head": info.get("sm_head"),
            "head": info["bins"][0].get("head") if info["bins"] else None}


def leg_c4(args, ctx, d):
    """configs[3]: C3's matrix by feature.  N = 1: K = 1 epochs (roofline of the dominant bin, time to
    1e-4).  N > 1: columns partitioned across the ranks (balanced partition, c29), optimal γ rounds."""
    torch = ctx.torch
    import synth
    import paper_1702_07005_b200 as scd

    cfg = synth.CONFIGS["C3"]
    N, M = cfg.n_rows, cfg.n_cols
    if d is None or ctx.world > 1:  # N > 1: every rank needs the whole C3 (it owns columns, not rows)
        d = synth.gen_device(cfg)
    cp, ci, cv = scd.transpose(d["ptr"], d["idx"], d["val"], N, M, "csr")
    y = d["y"]
    world, rank = ctx.world, ctx.rank
    if world > 1:
        # the library's structure-aware partition (stored-entry balanced, reading c29)
        owner = torch.from_numpy(scd.partition_balanced(cp, 4, world).astype(np.int64)).cuda()
        cols = torch.nonzero(owner == rank).flatten()
        lens = (cp[1:] - cp[:-1])[cols]
        sp = torch.zeros(len(cols) + 1, dtype=torch.int64, device="cuda")
        torch.cumsum(lens, 0, out=sp[1:])
        tot = int(sp[-1].item())
        pos = torch.repeat_interleave(cp[cols], lens, output_size=tot) + \
            (torch.arange(tot, device="cuda") - torch.repeat_interleave(sp[:-1], lens, output_size=tot))
        cp, ci, cv = sp, ci[pos].contiguous(), cv[pos].contiguous()
        del pos, owner
        torch.cuda.empty_cache()
    ncols = cp.numel() - 1
    nnz = int(cp[-1].item())
    s = scd.Solver(cp, ci, cv, N, ncols, y, cfg.lam, "primal", seed=4 + 10 * rank, profile=True, rank=rank,
                   world=world, **ctx.comm_kw())
    stream = torch.cuda.ExternalStream(s.stream_handle)
    info = s.info()

    def step(t):
        s.epoch(t)
        if world > 1:
            s.aggregate("optimal")

    for t in range(1, 4):
        step(t)
    torch.cuda.synchronize()
    s.profile_read()
    steps = 10
    l0 = s.info()["launches"]
    el_ms = timed_epochs(ctx, s, stream, 4, steps, step)
    ctx.launches += s.info()["launches"] - l0
    kprof = s.profile_read()
    roof = kernel_roofline(s, info, kprof, BYTES_PER_NNZ, el_ms, world)
    s.set_model(np.zeros(ncols, np.float32))
    ttg = time_to_gap(ctx, s, stream, step, max_rounds=40 if world > 1 else 10)
    s.close()
    del cp, ci, cv
    torch.cuda.empty_cache()
    return {"workload": "C4 (BASELINE configs[3]): C3's matrix by feature, primal TPA-SCD (CSC)"
                        + (f", columns partitioned across {world} GPUs (stored-entry balanced), optimal-gamma "
                           "aggregation each round"
                           if world > 1 else ", K = 1"),
            "nnz_per_gpu": nnz, "columns_per_gpu": ncols, "ms_per_step": el_ms / steps,
            "nnz_per_s": nnz * world * steps / (el_ms / 1e3), "steps": steps, "roofline": roof,
            "time_to_gap": ttg, "schedule": [{k: b[k] for k in ("lanes", "count", "nnz", "grid", "cap", "snap")}
                                             for b in info["bins"]]}


def leg_c2(args, ctx):
    """configs[1]: synthetic sparse 100 k x 50 k with power-law lengths (~1% density), dual by example and
    primal by feature on one GPU: epoch time, nnz/s and time to gap 1e-4 for each form."""
    torch = ctx.torch
    import synth
    import paper_1702_07005_b200 as scd

    cfg = synth.CONFIGS["C2"]
    d = synth.gen_device(cfg)
    N, M = d["n_rows"], d["n_cols"]
    out = {"workload": "C2 (BASELINE configs[1]): 100000 x 50000 power-law rows, ~1% density, 1 GPU"}
    for form in ("dual", "primal"):
        if form == "dual":
            p, i, v = d["ptr"], d["idx"], d["val"]
        else:
            p, i, v = scd.transpose(d["ptr"], d["idx"], d["val"], N, M, "csr")
        s = scd.Solver(p, i, v, N, M, d["y"], cfg.lam, form, seed=2, profile=True)
        stream = torch.cuda.ExternalStream(s.stream_handle)
        info = s.info()
        nnz = s.nnz
        for t in range(1, 4):
            s.epoch(t)
        torch.cuda.synchronize()
        s.profile_read()
        steps = 20
        l0 = s.info()["launches"]
        el_ms = timed_epochs(ctx, s, stream, 4, steps, lambda t: s.epoch(t))
        ctx.launches += s.info()["launches"] - l0
        kprof = s.profile_read()
        roof = kernel_roofline(s, info, kprof, BYTES_PER_NNZ, el_ms)
        s.set_model(np.zeros(N if form == "dual" else M, np.float32))
        ttg = time_to_gap(ctx, s, stream, lambda t: s.epoch(t), max_rounds=20)
        s.close()
        out[form] = {"nnz": nnz, "ms_per_step": el_ms / steps, "nnz_per_s": nnz * steps / (el_ms / 1e3),
                     "roofline": roof, "time_to_gap": ttg,
                     "schedule": [{k: b[k] for k in ("lanes", "count", "nnz", "grid", "head")} for b in info["bins"]]}
    del d
    torch.cuda.empty_cache()
    return out


def leg_c5(args, ctx):
    """configs[4]: criteo-shaped 200 M x 75 M one-hot, values implicit (val = NULL, NEXT-1), dual by
    example, 25 M rows per GPU (global N = 25 M x N: 200 M at N = 8).  N = 1: one shard's epoch (the
    per-GPU compute of the 8-GPU run, λN of the 8-GPU run).  N > 1: rounds of epoch + aggregation to
    gap 1e-4 with optimal γ, and the add / average baselines."""
    torch = ctx.torch
    import synth
    import paper_1702_07005_b200 as scd

    world, rank = ctx.world, ctx.rank
    rows = C5_ROWS_PER_GPU
    cfg = synth.CONFIGS["C5"].with_rows(rows * max(world, 8 if world == 1 else world))
    n_global = rows * 8 if world == 1 else rows * world
    d = synth.gen_device(cfg, rank * rows, rows)
    assert bool((d["val"] == 1.0).all())
    d["val"] = None
    torch.cuda.empty_cache()
    nnz = int(d["ptr"][-1].item())
    out = {"workload": f"C5 criteo-shaped (BASELINE configs[4]): {rows} rows x {cfg.n_cols} features per GPU, "
                       f"39 one-hot fields, implicit values (val = NULL), dual by example, global N = {n_global}",
           "nnz_per_gpu": nnz, "rows_per_gpu": rows, "n_global": n_global}
    if world == 1:
        s = scd.Solver(d["ptr"], d["idx"], None, rows, cfg.n_cols, d["y"], cfg.lam, "dual", seed=5, n_global=n_global,
                       profile=True)
        stream = torch.cuda.ExternalStream(s.stream_handle)
        info = s.info()
        for t in range(1, 4):
            s.epoch(t)
        torch.cuda.synchronize()
        s.profile_read()
        steps = 10
        l0 = s.info()["launches"]
        el_ms = timed_epochs(ctx, s, stream, 4, steps, s.epoch)
        ctx.launches += s.info()["launches"] - l0
        kprof = s.profile_read()
        out.update({"ms_per_step": el_ms / steps, "nnz_per_s": nnz * steps / (el_ms / 1e3), "steps": steps,
                    "roofline": kernel_roofline(s, info, kprof, BYTES_PER_NNZ_IMPLICIT, el_ms),
                    "schedule": [{k: b[k] for k in ("lanes", "count", "nnz", "grid", "block", "flush", "hot", "tau")}
                                 for b in info["bins"]],
                    "note": "one GPU's shard of the 8-GPU run (epoch only; the round adds the 300 MB all-reduce)"})
        s.close()
        return out
    s = scd.Solver(d["ptr"], d["idx"], None, rows, cfg.n_cols, d["y"], cfg.lam, "dual", seed=5 + rank,
                   n_global=n_global, rank=rank, world=world, **ctx.comm_kw())
    stream = torch.cuda.ExternalStream(s.stream_handle)
    modes = {}
    for mode, max_rounds in (("optimal", 30), ("average", 15), ("add", 4)):
        s.set_model(np.zeros(rows, np.float32))
        ttg = time_to_gap(ctx, s, stream, lambda t: (s.epoch(t), s.aggregate(mode)), max_rounds=max_rounds,
                          first=2000 * (1 + len(modes)))
        modes[mode] = ttg
    s.close()
    out["modes"] = modes
    out["time_to_gap_1e-4_s"] = modes["optimal"]["seconds"]
    out["rounds_to_gap_1e-4"] = modes["optimal"]["rounds"] if modes["optimal"]["seconds"] else None
    return out


# ------------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ttg", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the C4 / C5 sub-records")
    ap.add_argument("--quick", action="store_true", help="skip the access-pattern ceiling and the oracle time-to-gap")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--rows", type=int, default=0, help="override rows per rank (debug only)")
    ap.add_argument("--max-inflight", type=int, default=0)
    args = ap.parse_args()
    rank, world, local = _env_rank()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: relaunch under torch.distributed.run (the driver's own launch sets WORLD_SIZE)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={29400 + os.getpid() % 500}", os.path.abspath(__file__),
               *sys.argv[1:]]
        return subprocess.call(cmd)
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: one process per GPU is required"}),
              flush=True)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    assert args.warmup >= 3 or os.environ.get("BENCH_ALLOW_FEW_WARMUP"), "timing rules: warmup >= 3"
    import torch

    hooks = world > 1 and os.environ.get("BENCH_TRANSPORT") == "hooks"
    torch.cuda.set_device(0 if hooks else local)
    if world > 1 and not hooks:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the driver can check the rank count / transport in the log
    ctx = Ctx(rank, world, local)
    rec, d = leg_c3(args, ctx)
    subs = {}
    if not args.no_sub:
        # sub-records / north-star legs; a failing leg never loses the headline line
        if world == 1:
            try:
                subs["c4_primal"] = leg_c4(args, ctx, d)
            except Exception as ex:
                subs["c4_primal"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
            torch.cuda.empty_cache()
            try:
                subs["c2"] = leg_c2(args, ctx)
            except Exception as ex:
                subs["c2"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
            torch.cuda.empty_cache()
            try:
                subs["c3_load"] = leg_load(args, ctx, d)
            except Exception as ex:
                subs["c3_load"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
            torch.cuda.empty_cache()
            oracle_ttg = None
            if rank == 0 and not args.quick and not args.no_cpu_baseline:
                try:
                    oracle_ttg = oracle_time_to_gap(d)
                except Exception as ex:
                    oracle_ttg = {"error": f"{type(ex).__name__}: {ex}"[:300]}
            del d
            torch.cuda.empty_cache()
            try:
                subs["c5_shard"] = leg_c5(args, ctx)
            except Exception as ex:
                subs["c5_shard"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
        else:
            oracle_ttg = None
            del d
            torch.cuda.empty_cache()
            ns = {}
            for name, fn in (("c5_criteo", lambda: leg_c5(args, ctx)), ("c4_by_feature", lambda: leg_c4(args, ctx, None))):
                try:
                    ns[name] = fn()
                except Exception as ex:
                    ns[name] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
                torch.cuda.empty_cache()
            subs["north_star"] = ns
    else:
        oracle_ttg = None
        del d

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_seconds)
        if oracle_ttg:
            cpu["time_to_gap_1e-4"] = oracle_ttg
        if world > 1:
            try:
                cpu["distributed"] = cpu_baseline_dist(world)
            except Exception as ex:
                cpu["distributed"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}

    if rank == 0:
        cfg, info, rows, nnz, ttg = rec["cfg"], rec["info"], rec["rows"], rec["nnz"], rec["ttg"]
        out = {
            "metric": METRIC, "metric_full": METRIC_FULL, "value": rec["value"], "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C3 webspam-shaped (BASELINE configs[2]): dual TPA-SCD by example, "
                                   f"{rows}x{cfg.n_cols} per GPU, {nnz} nnz/GPU, lambda=1e-3"
                                   + (f", optimal-gamma aggregation over NCCL, global N={rows * world}" if world > 1 else ""),
                       "form": "dual", "rows_per_gpu": rows, "n_cols": cfg.n_cols, "nnz_per_gpu": nnz,
                       "lambda": cfg.lam, "l2": "inputs larger than L2 (10.4 GB CSR per GPU, 126 MB L2)",
                       "parallelism": f"dp{world}" if world > 1 else "single GPU",
                       "schedule": info["bins"], "inflight_cap": info["inflight_cap"], "tau_star": info["tau_star"],
                       "tail_read_copy": bool(info.get("tail_snap")), "tail_tau": info.get("tail_tau"),
                       "tail_roll": info.get("tail_roll"), "head_copy": info.get("head_copy"),
                       "n_slices": info.get("n_slices")},
            "time_to_gap_1e-4_s": (ttg or {}).get("seconds"), "time_to_gap": ttg,
            "hbm_gbs": (BYTES_PER_NNZ * nnz * world + BYTES_PER_COORD * rows * world) / (rec["ms_per_step"] / 1e3) / 1e9,
            "roofline": rec["roofline"],
            "access_pattern_ceiling": rec["pattern"],
            "cpu_baseline": cpu, "e2e": rec["e2e"], "gpu_launches": rec["gpu_launches"],
            "gpu_launches_all_legs": ctx.launches,
            "clocks": rec["clocks"], "setup_s": rec["setup_s"],
            **subs,
        }
        if hooks:
            out["transport"] = "hooks (test mode: all ranks on GPU 0, collectives through host gloo; not a result)"
        print(json.dumps(out, default=float), flush=True)
    if ctx.comm:
        import paper_1702_07005_b200 as scd

        scd.nccl_comm_destroy(ctx.comm)
    if ctx.dist is not None:
        ctx.dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
