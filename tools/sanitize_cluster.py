"""compute-sanitizer driver for the heavy-coordinate cluster kernels (C2 primal: 27 dense columns of
100 000 entries -> the 8-CTA cluster bin, TMA-staged slices) and the dual / implicit-value variants.
  compute-sanitizer --tool memcheck python tools/sanitize_cluster.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1702_07005_b200 as scd  # noqa: E402

d = synth.gen_host(synth.CONFIGS["C2"])
cp, ci, cv = scd.transpose(d["ptr"], d["idx"], d["val"], d["n_rows"], d["n_cols"], "csr")
for val in (cv, None):
    s = scd.Solver(cp, ci, val, d["n_rows"], d["n_cols"], d["y"], 1e-3, "primal", seed=3)
    kinds = [b["lanes"] for b in s.info()["bins"]]
    assert 4096 in kinds, kinds
    for t in (1, 2):
        s.epoch(t)
    print("primal", "implicit" if val is None else "explicit", kinds, "gap %.3e" % s.duality_gap(), flush=True)
    s.close()
print("sanitize_cluster done")
