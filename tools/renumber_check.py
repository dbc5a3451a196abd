"""Epoch time and convergence of a criteo-shaped shard before / after the device frequency
renumbering of the feature space (scd_renumber), to see whether a globally frequency-ranked
shared vector (hot tail entries packed into fewer lines) helps the L2 hit rate of the tail.
usage: python tools/renumber_check.py [rows=25000000] [n_global=200000000]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1702_07005_b200 as scd  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 25_000_000
n_global = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000_000
cfg = synth.CONFIGS["C5"].with_rows(rows)
d = synth.gen_device(cfg)


def run(tag, p, i, v):
    s = scd.Solver(p, i, v, d["n_rows"], d["n_cols"], d["y"], cfg.lam, "dual", seed=4, n_global=n_global)
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
    s.set_model(torch.zeros(d["n_rows"]).numpy())
    gaps = []
    for t in range(1, 5):
        s.epoch(100 + t)
        gaps.append(s.duality_gap())
    b = s.info()["bins"][0]
    print(f"[{tag}] hot={b['hot']} flush={b['flush']} cover={s.info()['hot_cover']:.3f}: epoch {ms:.2f} ms  gaps "
          + " ".join(f"{g:.2e}" for g in gaps), flush=True)
    s.close()


run("generator ids", d["ptr"], d["idx"], d["val"])
p2, i2, v2, _ = scd.renumber(d["ptr"], d["idx"], d["val"], d["n_rows"], d["n_cols"], "csr")
torch.cuda.synchronize()
del d["idx"], d["val"]
run("frequency-renumbered", p2, i2, v2)
