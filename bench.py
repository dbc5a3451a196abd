#!/usr/bin/env python
"""Benchmark of the TPA-SCD hot path (Parnell et al., arXiv 1702.07005) on B200.

Workload (BASELINE.json configs[2], the webspam-shaped config the metric's target is quoted on):
C3 = 350,000 x 16,609,143 CSR, ~3,728 nnz/row (1.305e9 nnz, fp32 values + int32 indices =
10.4 GB, larger than the 126 MB L2), dual TPA-SCD by example, λ = 1e-3.  Generated on the device
by the seeded generator (synth/); nothing is read from disk.

A step = one local TPA-SCD epoch (scd_epoch: permutation inline, gather-dot, closed-form delta,
atomic scatter; §8(a) rows a1-a6) and, when N > 1, one optimal-gamma aggregation round over NCCL
(a8).  With N GPUs each rank holds its own 350,000-row block of a 350,000·N-row matrix (weak
scaling, global N in λN).  The gap evaluation (a7) is off the clock, as in the paper's plots.

Prints ONE JSON line (rank 0).  `--impl reference` times the fp64 oracle (the only "reference"
this paper has: it ships no code) on bounded samples of the same workload on the host cores.
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
BYTES_PER_COORD = 32  # ptr pair 16 + norm 4 + model RMW 8 + label 4
METRIC = "nnz/s per epoch"
METRIC_FULL = "time-to-duality-gap 1e-4 (s); nnz/s per epoch; HBM GB/s vs B200 peak"


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
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


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


def cpu_baseline(seconds: float = 15.0, rows: int = 20_000):
    """The fp64 oracle's dual epoch (Alg. 1 / Eq. 4, sequential, 1 core) on the first ``rows`` rows
    of C3; returns nnz/s over whole epochs within ~``seconds``."""
    import oracle
    import synth
    from oracle import solver

    cfg = c3_cfg(1).with_rows(rows)
    d = synth.gen_host(cfg)
    pr = solver.Problem.from_csr(d)
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
    pr = solver.Problem.from_csr(d)
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ttg", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--rows", type=int, default=0, help="override rows per rank (debug only)")
    ap.add_argument("--max-inflight", type=int, default=0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    assert args.warmup >= 3 or os.environ.get("BENCH_ALLOW_FEW_WARMUP"), "timing rules: warmup >= 3"

    import torch

    import synth
    import paper_1702_07005_b200 as scd

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = c3_cfg(world)
    rows = args.rows or synth.CONFIGS["C3"].n_rows
    row0 = rank * rows
    t_gen = time.perf_counter()
    d = synth.gen_device(cfg, row0, rows)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    nnz = int(d["ptr"][-1].item())
    comm = None
    if world > 1:
        uid = scd.nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
        dist.broadcast(t, 0)
        comm = scd.nccl_comm_init(bytes(t.cpu().tolist()), world, rank)
    # The library creates its own stream; torch only wraps it to record the timing events.
    kw = dict(seed=3 + rank, n_global=rows * world, rank=rank, world=world, nccl_comm=comm, max_inflight=args.max_inflight)
    t_create = time.perf_counter()
    s = scd.Solver(d["ptr"], d["idx"], d["val"], rows, cfg.n_cols, d["y"], cfg.lam, "dual", profile=True, **kw)
    t_create = time.perf_counter() - t_create
    stream = torch.cuda.ExternalStream(s.stream_handle)
    info = s.info()

    def step(t):
        s.epoch(t)
        if world > 1:
            s.aggregate("optimal")

    def barrier():
        if dist is not None:
            dist.barrier()

    for t in range(1, args.warmup + 1):
        step(t)
    torch.cuda.synchronize()
    s.profile_read()  # drop warm-up kernel timings
    launches0 = s.info()["launches"]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for t in range(args.warmup + 1, args.warmup + args.steps + 1):
            step(t)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    el_ms = ev0.elapsed_time(ev1)
    launches = s.info()["launches"] - launches0
    kprof = s.profile_read()
    if dist is not None:
        tt = torch.tensor([el_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el_ms = float(tt.item())
    total_nnz = nnz * world
    value = total_nnz * args.steps / (el_ms / 1e3)
    ms_step = el_ms / args.steps

    # roofline of the dominant kernel (the bin with the most device time)
    peak, peak_src = _peaks()
    bins = info["bins"]
    b_i = max(range(len(kprof)), key=lambda i: kprof[i][0]) if kprof else 0
    ms_b, cnt_b = kprof[b_i] if kprof else (float("nan"), 0)
    # one launch processes one of the n_slices slices of the bin
    bytes_launch = (BYTES_PER_NNZ * bins[b_i]["nnz"] + BYTES_PER_COORD * bins[b_i]["count"]) / info["n_slices"]
    achieved = bytes_launch / (ms_b / cnt_b / 1e3) / 1e9 if cnt_b else None
    bb = bins[b_i]
    kname = ("k_epoch_split" if bb.get("split") else "k_epoch_cta_head" if bb.get("head") else "k_epoch_cta") \
        if bb["lanes"] >= 64 else "k_epoch_group"
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            # only a capture of the same kernel counts (names: "...k_epoch_cta_head<1, 256, 16>...")
            if (kname + "<") in tj.get("kernel", ""):
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    kernel_share = (ms_b / (el_ms if world == 1 else el_ms)) if cnt_b else None

    # access-pattern ceiling on this box: the same gathers + REDs over the same matrix with no
    # algorithmic dependency (tools/pattern_bench.cu), against a scratch vector
    pattern = None
    pso = os.path.join(ROOT, "tools", "libpattern.so")
    if os.path.exists(pso):
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
            # the same with the gathers served from a second vector (the head kernel's tail read copy)
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

    # time to duality gap 1e-4 from a fresh start (epoch + aggregation time only, gap off the clock)
    ttg = None
    if not args.no_ttg:
        s.set_model(np.zeros(rows, np.float32))
        acc, hist, g = 0.0, [], None
        for t in range(1, 61):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record(stream)
            step(1000 + t)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if dist is not None:
                tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                ms = float(tt.item())
            acc += ms
            g = s.duality_gap()
            hist.append(g)
            if g <= 1e-4:
                break
        ttg = {"seconds": acc / 1e3 if g is not None and g <= 1e-4 else None, "epochs": len(hist),
               "gap_trace": [float("%.3e" % x) for x in hist[:12]], "target": 1e-4}
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
            n_ep = (ttg or {}).get("epochs") or 5
            times = []
            for rep in range(5):
                torch.cuda.synchronize()
                barrier()
                t0 = time.perf_counter()
                s2 = scd.Solver(hp, hi, hv, rows, cfg.n_cols, hy, cfg.lam, "dual", validate=False, **kw)
                for t in range(1, n_ep + 1):
                    s2.epoch(t)
                    if world > 1:
                        s2.aggregate("optimal")
                model = s2.get_model()
                el = time.perf_counter() - t0
                s2.close()
                if dist is not None:
                    tt = torch.tensor([el], dtype=torch.float64, device="cuda")
                    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                    el = float(tt.item())
                if rep > 0:
                    times.append(el)
            e_s = statistics.median(times)
            e2e = {"value": total_nnz * n_ep / e_s, "unit": "nnz/s",
                   "h2d_bytes_per_step": int(8 * (rows + 1) + 8 * nnz + 4 * rows),
                   "d2h_bytes_per_step": int(4 * rows), "epochs_per_step": n_ep, "seconds_per_step": e_s,
                   "seconds_per_rep": [round(x, 4) for x in times],
                   "step": "scd_create from pinned host CSR (H2D) + epochs-to-gap-1e-4"
                           + (" with optimal-gamma aggregation" if world > 1 else "") + " + scd_get_model (D2H)"
                           + ("; bytes per rank" if world > 1 else "")}
            del hp, hi, hv, hy
        except Exception as ex:  # never lose the device-timed line to the e2e leg
            e2e = {"value": None, "error": f"{type(ex).__name__}: {ex}"[:300]}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_seconds)

    if rank == 0:
        out = {
            "metric": METRIC, "metric_full": METRIC_FULL, "value": value, "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C3 webspam-shaped (BASELINE configs[2]): dual TPA-SCD by example, "
                                   f"{rows}x{cfg.n_cols} per GPU, {nnz} nnz/GPU, lambda=1e-3"
                                   + (f", optimal-gamma aggregation over NCCL, global N={rows * world}" if world > 1 else ""),
                       "form": "dual", "rows_per_gpu": rows, "n_cols": cfg.n_cols, "nnz_per_gpu": nnz,
                       "lambda": cfg.lam, "l2": "inputs larger than L2 (10.4 GB CSR per GPU, 126 MB L2)",
                       "parallelism": f"dp{world}" if world > 1 else "single GPU",
                       "schedule": bins, "inflight_cap": info["inflight_cap"], "tau_star": info["tau_star"],
                       "tail_read_copy": bool(info.get("tail_snap")), "tail_tau": info.get("tail_tau"),
                       "tail_roll": info.get("tail_roll"), "n_slices": info.get("n_slices")},
            "time_to_gap_1e-4_s": (ttg or {}).get("seconds"), "time_to_gap": ttg,
            "hbm_gbs": (BYTES_PER_NNZ * total_nnz + BYTES_PER_COORD * rows * world) / (ms_step / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": f"{kname} (bin {b_i}, {bb['lanes']} lanes/coord"
                                   + (f", head {bb['head']} floats combined, flush every {bb['flush']}" if bb.get("head") else "")
                                   + ((", tail gathers from the read copy refreshed in rolling chunks (one launch per epoch)"
                                       if info.get("tail_roll") else ", tail gathers from the per-slice read copy")
                                      if bb.get("head") and info.get("tail_snap") else "")
                                   + ")",
                         "kernel_ms_avg": ms_b / cnt_b if cnt_b else None, "kernel_share_of_step": kernel_share,
                         "bytes_per_launch": bytes_launch, "peak_source": peak_src,
                         "byte_model": "16 B/nnz (idx+val+gather+atomic) + 32 B/coordinate"},
            "access_pattern_ceiling": pattern,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(),
            "setup_s": {"generate": t_gen, "create": t_create},
        }
        print(json.dumps(out), flush=True)
    s.close()
    if comm:
        scd.nccl_comm_destroy(comm)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
