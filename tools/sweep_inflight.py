"""Convergence-vs-concurrency sweep (GPU): gap per epoch and epoch time for several caps on the
number of coordinates in flight.  Usage: python tools/sweep_inflight.py C2 dual 0,64,256,1024"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1702_07005_b200 as scd  # noqa: E402


def main():
    cfgname, form = sys.argv[1], sys.argv[2]
    caps = [int(x) for x in sys.argv[3].split(",")]
    epochs = int(sys.argv[4]) if len(sys.argv) > 4 else 12
    cfg = synth.CONFIGS[cfgname] if cfgname in synth.CONFIGS else None
    if cfgname.startswith("C5s"):
        cfg = synth.c5_scaled(int(2e6), 1e-1)
    d = synth.gen_device(cfg)
    n_rows, n_cols = d["n_rows"], d["n_cols"]
    if form == "primal":
        p, i, v = scd.transpose(d["ptr"], d["idx"], d["val"], n_rows, n_cols, "csr")
    else:
        p, i, v = d["ptr"], d["idx"], d["val"]
    rec = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    for cap in caps:
        st = torch.cuda.Stream() if os.environ.get("SWEEP_TORCH_STREAM") else None
        s = scd.Solver(p, i, v, n_rows, n_cols, d["y"], cfg.lam, form, seed=int(os.environ.get("SWEEP_SEED", 4)),
                       max_inflight=max(cap, 0), profile=True, deterministic=cap < 0, recompute_every=rec, stream=st)
        info = s.info()
        gaps, ms = [], []
        for t in range(1, epochs + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s.epoch(t)
            torch.cuda.synchronize()
            ms.append(1e3 * (time.perf_counter() - t0))
            gaps.append(s.duality_gap())
        prof = s.profile_read()
        print(f"{cfgname} {form} cap={cap} bins={[(b['lanes'], b['count'], b['grid'], b['block'], b['cap'], round(b['tau'])) for b in info['bins']]}")
        print(f"   ms/epoch median {np.median(ms):.3f}  kernels {[(round(a / max(c, 1), 3), c) for a, c in prof]}")
        print("   gaps " + " ".join("%.2e" % g for g in gaps), flush=True)
        s.close()


if __name__ == "__main__":
    main()
