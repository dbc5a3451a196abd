"""Atomic TPA-SCD vs the "wild" (non-atomic scatter, PASSCoDe-Wild) variant on one config:
epoch time, fp64 gap per epoch, and the shared-vector inconsistency ||w̄ - Aᵀα||∞/||Aᵀα||∞ at the end
(SURVEY NEXT-4).  Usage: python tools/wild_compare.py C3 dual 8"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1702_07005_b200 as scd  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
form = sys.argv[2] if len(sys.argv) > 2 else "dual"
E = int(sys.argv[3]) if len(sys.argv) > 3 else 8
d = synth.gen_device(cfg)
mat = (d["ptr"], d["idx"], d["val"])
if form == "primal":
    mat = scd.transpose(*mat, d["n_rows"], d["n_cols"], "csr")
for wild in (False, True):
    s = scd.Solver(*mat, d["n_rows"], d["n_cols"], d["y"], cfg.lam, form, seed=4, wild=wild)
    es = torch.cuda.ExternalStream(s.stream_handle)
    ms, gaps = [], []
    for t in range(1, E + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(es)
        s.epoch(t)
        e1.record(es)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        gaps.append(s.duality_gap())
    # consistency of the maintained shared vector with the model (recomputed in fp64 by the library)
    sh = torch.from_numpy(s.get_shared()).double()
    s.recompute_shared()
    ref = torch.from_numpy(s.get_shared()).double()
    drift = float((sh - ref).abs().max() / ref.abs().max())
    print(f"{'wild  ' if wild else 'atomic'} {cfg.name} {form}: epoch ms median {np.median(ms[1:]):.2f}  "
          f"drift {drift:.2e}  gaps " + " ".join(f"{g:.2e}" for g in gaps), flush=True)
    s.close()
