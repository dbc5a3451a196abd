"""Run a few epochs of one config/form for profiling (ncu -k regex:k_epoch -s <skip> -c <n>).
Usage: python tools/prof_epoch.py C3 dual 4"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1702_07005_b200 as scd  # noqa: E402

cfgname, form, epochs = sys.argv[1], sys.argv[2], int(sys.argv[3])
cfg = synth.CONFIGS[cfgname]
d = synth.gen_device(cfg)
p, i, v = d["ptr"], d["idx"], d["val"]
if form == "primal":
    p, i, v = scd.transpose(p, i, v, d["n_rows"], d["n_cols"], "csr")
s = scd.Solver(p, i, v, d["n_rows"], d["n_cols"], d["y"], cfg.lam, form, seed=4)
print(s.info(), flush=True)
for t in range(1, epochs + 1):
    s.epoch(t)
torch.cuda.synchronize()
print("gap", s.duality_gap())
