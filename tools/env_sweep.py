"""Epoch time + convergence for a list of library environment settings (each creates a fresh context).
usage: python tools/env_sweep.py C5:25000000 dual "SCD_HOT=0;SCD_HOT=4096,SCD_HOT_F=3" [n_global]
Each setting: 1 warm-up epoch, 4 timed epochs (library stream), then a fresh start and the fp64
gap after epochs 1..4."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1702_07005_b200 as scd  # noqa: E402

name, form, settings = sys.argv[1], sys.argv[2], sys.argv[3].split(";")
n_global = int(sys.argv[4]) if len(sys.argv) > 4 else 0
cfg = synth.CONFIGS["C5"].with_rows(int(name[3:])) if name.startswith("C5:") else synth.CONFIGS[name]
d = synth.gen_device(cfg)
mat = (d["ptr"], d["idx"], d["val"])
if form == "primal":
    mat = scd.transpose(*mat, d["n_rows"], d["n_cols"], "csr")
keys = set()
for st in settings:
    for kv in filter(None, st.split(",")):
        keys.add(kv.split("=")[0])
for st in settings:
    for k in keys:
        os.environ.pop(k, None)
    for kv in filter(None, st.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    s = scd.Solver(*mat, d["n_rows"], d["n_cols"], d["y"], cfg.lam, form, seed=4, n_global=n_global)
    inf = s.info()
    es = torch.cuda.ExternalStream(s.stream_handle)
    s.epoch(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(es)
    for t in range(2, 6):
        s.epoch(t)
    e1.record(es)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 4
    s.set_model(torch.zeros(inf["n_coord"]).numpy())
    gaps = []
    for t in range(1, 5):
        s.epoch(100 + t)
        gaps.append(s.duality_gap())
    b0 = max(inf["bins"], key=lambda b: b["nnz"])
    print(f"[{st or 'default'}] bin lanes={b0['lanes']} grid={b0['grid']} cap={b0['cap']} hot={b0.get('hot', 0)} "
          f"flush={b0['flush']} tail_snap={inf.get('tail_snap')} tail_tau={inf.get('tail_tau', 0):.0f} slices={inf['n_slices']} roll={inf.get('tail_roll', 0)} hcopy={inf.get('head_copy', 0)} hotcopy={inf.get('hot_copy', 0)} tp={inf.get('hot_tp', 0)} hp={inf.get('hot_hp', 0)} httau={inf.get('hot_tail_tau', 0):.3g}: epoch {ms:.2f} ms  gaps " + " ".join(f"{g:.2e}" for g in gaps)
          + "  snap " + ",".join(f"{b['lanes']}:{b.get('snap', 0)}" for b in inf["bins"]), flush=True)
    s.close()
