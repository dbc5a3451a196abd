"""Run a few epochs of one config/form for profiling (ncu -k regex:k_epoch -s <skip> -c <n>), or
time them (--time).  Config names: C2, C3, or C5:<rows> (criteo-shaped, first <rows> rows).
Usage: python tools/prof_epoch.py C3 dual 4 [--time]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1702_07005_b200 as scd  # noqa: E402

cfgname, form, epochs = sys.argv[1], sys.argv[2], int(sys.argv[3])
if cfgname.startswith("C5:"):
    cfg = synth.CONFIGS["C5"].with_rows(int(cfgname[3:]))
else:
    cfg = synth.CONFIGS[cfgname]
t0 = time.perf_counter()
d = synth.gen_device(cfg)
p, i, v = d["ptr"], d["idx"], d["val"]
if os.environ.get("PROF_IMPLICIT"):  # one-hot data: drop the all-ones value array (NEXT-1)
    assert bool((v == 1).all())
    v = None
    del d["val"]
if form == "primal":
    p, i, v = scd.transpose(p, i, v, d["n_rows"], d["n_cols"], "csr")
torch.cuda.synchronize()
t1 = time.perf_counter()
s = scd.Solver(p, i, v, d["n_rows"], d["n_cols"], d["y"], cfg.lam, form, seed=4, profile="--time" in sys.argv,
               n_global=int(os.environ.get("PROF_NGLOBAL", 0)), max_inflight=int(os.environ.get("PROF_CAP", 0)))
torch.cuda.synchronize()
t2 = time.perf_counter()
print(cfg.name, form, "nnz", s.nnz, "setup %.2fs create %.2fs" % (t1 - t0, t2 - t1), s.info(), flush=True)
es = torch.cuda.ExternalStream(s.stream_handle)
gaps, ms = [], []
for t in range(1, epochs + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(es)
    s.epoch(t)
    e1.record(es)
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
    if "--time" in sys.argv:
        gaps.append(s.duality_gap())
print("epoch ms", " ".join("%.2f" % m for m in ms))
if gaps:
    print("gaps", " ".join("%.2e" % g for g in gaps))
    print("kernels", s.profile_read())
    print("nnz/s (median epoch) %.3e" % (s.nnz / (sorted(ms)[len(ms) // 2] / 1e3)))
