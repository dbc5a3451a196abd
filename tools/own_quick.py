import os, sys, time
sys.path.insert(0, "/root/repo")
import torch, synth
import paper_1702_07005_b200 as scd
cfg = synth.CONFIGS["C3"]
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
d = synth.gen_device(cfg.with_rows(rows))
lam = 1e-3 * 350_000 / rows
s = scd.Solver(d["ptr"], d["idx"], d["val"], rows, cfg.n_cols, d["y"], lam, "dual", seed=4)
inf = s.info(); print({k: inf[k] for k in ("own", "own_warps", "own_err", "sm_head", "n_slices")}, inf["bins"], flush=True)
st = torch.cuda.ExternalStream(s.stream_handle)
for t in range(1, 7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); s.epoch(t); e1.record(st); torch.cuda.synchronize()
    print(t, "%.3f ms" % e0.elapsed_time(e1), "gap %.3e" % s.duality_gap(), "err", s.info()["own_err"], flush=True)
x = s.get_model().astype("float64"); w = s.get_shared().astype("float64")
import numpy as np
from oracle import ridge
A = ridge.as_matrix(d["ptr"].cpu().numpy(), d["idx"].cpu().numpy(), d["val"].cpu().numpy(), rows, cfg.n_cols)
v = A.T @ x
print("drift", np.abs(w - v).max() / np.abs(v).max())
