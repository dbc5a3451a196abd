"""Distributed SCD (Alg. 3 / 4) with K logical workers on ONE B200: per-round duality gap, γ and
device time per worker, for the paper's aggregation modes (add / average / optimal).

  python tools/dist_convergence.py C4 8 30      # C3 matrix in CSC, primal by feature, K in {1,2,4,8}
  python tools/dist_convergence.py C5 8 20      # criteo-shaped 200M x 75M, dual by example, K = 8

Every worker is a full scd context on its own shard; a round = one local epoch per worker
(timed with CUDA events on its stream) + scd_aggregate_group; the gap of the global model comes
from scd_evaluate_group.  With K GPUs the per-round time would be max_k(epoch_k) + the NCCL
all-reduce of the shared-vector delta; the table reports the mean worker epoch (the per-GPU
compute) and the all-reduce estimate from the measured 8-rank bus bandwidth (725 GB/s,
B200_PROFILING.md)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1702_07005_b200 as scd  # noqa: E402

BUSBW = 725e9


def col_shards(p, i, v, owner, K):
    """CSC column shards of (p, i, v) for owner[c] in [0, K) (device tensors)."""
    lens = p[1:] - p[:-1]
    out = []
    for k in range(K):
        cols = torch.nonzero(owner == k).flatten()
        ln = lens[cols]
        np_ = torch.zeros(len(cols) + 1, dtype=torch.int64, device=p.device)
        torch.cumsum(ln, 0, out=np_[1:])
        tot = int(np_[-1].item())
        starts = torch.repeat_interleave(p[cols], ln, output_size=tot)
        offs = torch.arange(tot, device=p.device) - torch.repeat_interleave(np_[:-1], ln, output_size=tot)
        pos = starts + offs
        out.append((np_, i[pos].contiguous(), v[pos].contiguous() if v is not None else None, len(cols)))
        del starts, offs, pos
    return out


PARTS = int(os.environ.get("DIST_PARTS", "1"))  # > 1: sub-epoch rounds (scd_epoch_part)


def run(solvers, mode, rounds, n_shared, stop=float(os.environ.get("DIST_STOP", "1e-6"))):
    recs = []
    for r in range(1, rounds * PARTS + 1):
        ms = []
        for s in solvers:
            st = torch.cuda.ExternalStream(s.stream_handle)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            if PARTS > 1:
                s.epoch_part((r - 1) // PARTS + 1, (r - 1) % PARTS, PARTS)
            else:
                s.epoch(r)
            e1.record(st)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t0 = time.perf_counter()
        g = scd.aggregate_group(solvers, mode)
        agg_ms = 1e3 * (time.perf_counter() - t0)
        P, D, gap = scd.evaluate_group(solvers)
        recs.append(dict(round=r, gamma=g, gap=gap, P=P, worker_ms_mean=float(np.mean(ms)),
                         worker_ms_max=float(np.max(ms)), agg_ms_single_gpu=agg_ms))
        if not np.isfinite(gap) or gap > 1e6 or gap <= stop:
            break
    return recs


def main():
    which, kmax, rounds = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    results = {}
    if which == "C4":
        cfg = synth.CONFIGS["C3"]
        d = synth.gen_device(cfg)
        p, i, v = scd.transpose(d["ptr"], d["idx"], d["val"], d["n_rows"], d["n_cols"], "csr")
        y = d["y"]
        del d
        torch.cuda.empty_cache()
        for K in [k for k in (1, 2, 4, 8) if k <= kmax]:
            # DIST_PART=balanced: stored-entry balanced partition (reading c29, NEXT-3); default: random (c15)
            if os.environ.get("DIST_PART") == "balanced":
                owner = torch.from_numpy(scd.partition_balanced(p, 4, K).astype(np.int64)).cuda()
            else:
                owner = torch.from_numpy(scd.partition(4, cfg.n_cols, K).astype(np.int64)).cuda()
            shards = col_shards(p, i, v, owner, K)
            nnz_k = [int(sp[-1].item()) for sp, _, _, _ in shards]
            print(f"K={K} partition {os.environ.get('DIST_PART', 'random')}: nnz per worker max/mean "
                  f"{max(nnz_k) / (sum(nnz_k) / K):.4f}", flush=True)
            for mode in [m for m in (("add", "average", "optimal") if K > 1 else ("average",))
                         if K == 1 or m in os.environ.get("DIST_MODES", "optimal,average,add")]:
                solvers = [scd.Solver(sp, si, sv_, cfg.n_rows, nc, y, cfg.lam, "primal", seed=10 + k)
                           for k, (sp, si, sv_, nc) in enumerate(shards)]
                recs = run(solvers, mode, rounds, cfg.n_rows)
                results[f"K={K} {mode}"] = recs
                print(f"K={K} {mode:8s} gaps {' '.join('%.1e' % x['gap'] for x in recs)}", flush=True)
                print(f"          gamma {' '.join('%.3f' % x['gamma'] for x in recs)}  "
                      f"worker epoch mean {np.mean([x['worker_ms_mean'] for x in recs]):.2f} ms, "
                      f"max {np.mean([x['worker_ms_max'] for x in recs]):.2f} ms", flush=True)
                for s in solvers:
                    s.close()
            del shards
            torch.cuda.empty_cache()
    else:  # C5: dual by example, K contiguous row blocks of the 200M-row matrix (iid rows)
        cfg = synth.CONFIGS["C5"]
        K = kmax
        rows = cfg.n_rows // K
        shards = []
        for k in range(K):
            d = synth.gen_device(cfg, k * rows, rows)
            assert bool((d["val"] == 1).all())
            shards.append((d["ptr"], d["idx"], d["y"]))
            del d
        for mode in [m for m in ("optimal", "average", "add") if m in os.environ.get("DIST_MODES", "optimal,average,add")]:
            solvers = [scd.Solver(sp, si, None, rows, cfg.n_cols, sy, cfg.lam, "dual", seed=10 + k,
                                  n_global=cfg.n_rows) for k, (sp, si, sy) in enumerate(shards)]
            recs = run(solvers, mode, rounds if mode != "add" else 4, cfg.n_cols, stop=1e-6)
            results[f"K={K} {mode}"] = recs
            print(f"K={K} {mode:8s} gaps {' '.join('%.1e' % x['gap'] for x in recs)}", flush=True)
            print(f"          gamma {' '.join('%.3f' % x['gamma'] for x in recs[:12])}  "
                  f"worker epoch {np.mean([x['worker_ms_mean'] for x in recs]):.2f} ms  "
                  f"allreduce est {2 * (K - 1) / K * 4 * cfg.n_cols / BUSBW * 1e3:.2f} ms", flush=True)
            for s in solvers:
                s.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    sfx = f"_parts{PARTS}" if PARTS > 1 else ""
    json.dump(results, open(os.path.join(ROOT, "gpurun_out", f"dist_{which}{sfx}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
