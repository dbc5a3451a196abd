"""Head-combining kernel sweep: epoch time and convergence per (SCD_HEAD, SCD_HEAD_FLUSH) setting.

usage: python tools/head_sweep.py C3 dual "0:0 12288:0 12288:4 16384:3 ..."   (H:flush, flush 0 = auto)
Every setting creates a fresh context (the knobs are read at create), times 6 epochs after one
warm-up epoch on the library stream, then restarts from zero and records the fp64 gap after
epochs 1..4 (convergence must not degrade).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1702_07005_b200 as scd  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
form = sys.argv[2] if len(sys.argv) > 2 else "dual"
settings = (sys.argv[3] if len(sys.argv) > 3 else "0:0 12288:0").split()
d = synth.gen_device(cfg)
if form == "primal":
    cp, ci, cv = scd.transpose(d["ptr"], d["idx"], d["val"], d["n_rows"], d["n_cols"], "csr")
    mat = (cp, ci, cv)
else:
    mat = (d["ptr"], d["idx"], d["val"])
for st in settings:
    h, f = st.split(":")
    os.environ["SCD_HEAD"] = h
    if f != "0":
        os.environ["SCD_HEAD_FLUSH"] = f
    else:
        os.environ.pop("SCD_HEAD_FLUSH", None)
    s = scd.Solver(*mat, d["n_rows"], d["n_cols"], d["y"], cfg.lam, form, seed=4)
    inf = s.info()
    es = torch.cuda.ExternalStream(s.stream_handle)
    s.epoch(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(es)
    for t in range(2, 8):
        s.epoch(t)
    e1.record(es)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 6
    s.set_model(torch.zeros(inf["n_coord"]).numpy())
    gaps = []
    for t in range(1, 5):
        s.epoch(100 + t)
        gaps.append(s.duality_gap())
    b0 = inf["bins"][0]
    print(f"H={h:>6} flush={f:>2} -> head={b0['head']} flush={b0['flush']} split={b0['split']} "
          f"dies={inf['n_die_sm']} lat={inf['die_lat']} nnz0={inf['split_nnz0'] / max(inf['nnz'], 1):.3f} grid={b0['grid']} cap={b0['cap']}: "
          f"epoch {ms:.2f} ms  gaps " + " ".join(f"{g:.2e}" for g in gaps), flush=True)
    s.close()
