"""Small end-to-end exercise of every kernel family for compute-sanitizer (memcheck / racecheck):
deterministic and asynchronous epochs (CTA, sub-warp, combining, cluster bins), the head-combining
CTA kernel (plain, with the shared-memory view, with the tail read copy and next-coordinate
prefetch), the die-split kernel, the wild scatter, the
hot-set kernel (and its view), the fused peer-memory aggregation, device renumbering, empty
rows/cols, implicit values, gap/objective, aggregation (group and 1-rank NCCL), transpose,
permutation."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1702_07005_b200 as scd  # noqa: E402


def run(d, form, **kw):
    p, i, v = d["ptr"], d["idx"], d["val"]
    if form == "primal":
        p, i, v = scd.transpose(p, i, v, d["n_rows"], d["n_cols"], "csr")
    s = scd.Solver(p, i, v, d["n_rows"], d["n_cols"], d["y"], d["lam"], form, seed=3, **kw)
    for t in (1, 2):
        s.epoch(t)
    s.epoch_part(3, 0, 2)
    s.epoch_part(3, 1, 2)
    g = s.duality_gap()
    P, D = s.objective()
    s.aggregate("optimal")
    s.get_shared()
    s.close()
    return g, P, D


# mixed lengths: short (group/comb), medium (warp), long (CTA) and very long (cluster) coordinates
rng = np.random.default_rng(0)
n_rows, n_cols = 6000, 3000
lens = np.concatenate([rng.integers(1, 60, 2900), rng.integers(100, 900, 80), rng.integers(2000, 5900, 15),
                       np.full(5, 5990)])
rows = []
for c, L in enumerate(lens):
    rows.append(np.sort(rng.choice(n_rows, size=min(L, n_rows), replace=False)))
ptr = np.zeros(n_cols + 1, np.int64)
ptr[1:] = np.cumsum([len(r) for r in rows])
cidx = np.concatenate(rows).astype(np.int32)
cval = rng.random(len(cidx)).astype(np.float32)
# this is CSC (columns); make the CSR view for the dual
rp, ri, rv = scd.transpose(ptr, cidx, cval, n_rows, n_cols, "csc")
d = dict(ptr=rp, idx=ri, val=rv, y=np.sign(rng.standard_normal(n_rows)).astype(np.float32), n_rows=n_rows,
         n_cols=n_cols, lam=1e-2)
for form in ("dual", "primal"):
    for kw in (dict(deterministic=True), dict(), dict(max_inflight=3)):
        print(form, kw, run(d, form, **kw), flush=True)
c5 = synth.gen_host(synth.c5_scaled(4000, 1e-3))
c5["val"] = None
print("implicit", run(c5, "dual"), flush=True)
e = synth.random_sparse(300, 200, 0.05, 3, empty_rows=7, empty_cols=9)
print("empty", run(e, "dual"), run(e, "primal"), flush=True)
uid = scd.nccl_unique_id()
comm = scd.nccl_comm_init(uid, 1, 0)
print("nccl", run(e, "dual", nccl_comm=comm), flush=True)
scd.nccl_comm_destroy(comm)
a = [scd.Solver(e["ptr"], e["idx"], e["val"], 300, 200, e["y"], 0.01, "dual", seed=k) for k in range(2)]
for s in a:
    s.epoch(1)
print("group", scd.aggregate_group(a, "optimal"))
assert np.array_equal(np.sort(scd.permutation(1, 2, 1000)), np.arange(1000))
for form in ("dual", "primal"):
    print("wild", form, run(d, form, wild=True), flush=True)
# webspam-shaped rows (C3 prefix, λN = 350 as in the full C3) put every row in the CTA bin with a grid
# covering every SM: head-combining kernel, with and without the per-slice tail read copy
c3 = synth.gen_host(synth.CONFIGS["C3"].with_rows(1500))
c3["lam"] = 350.0 / 1500
for env in ({}, {"SCD_TAIL_SNAP": "1"}, {"SCD_TAIL_SNAP": "0"}):
    os.environ.update(env)
    s = scd.Solver(c3["ptr"], c3["idx"], c3["val"], 1500, c3["n_cols"], c3["y"], c3["lam"], "dual", seed=3)
    inf = s.info()
    s.close()
    print("c3 prefix", env, inf["bins"][0], "tail_snap", inf["tail_snap"], run(c3, "dual"), flush=True)
    for k in env:
        del os.environ[k]
# rolling refresh of the tail copy (one head-kernel launch per epoch): needs a bin of >= 8 x 657 rows
# (default: the SM-shared head kernel with bulk-copied rows; SCD_SM_HEAD=0: the per-CTA head kernel)
c3r = synth.gen_host(synth.CONFIGS["C3"].with_rows(20_000))
c3r["lam"] = 350.0 / 20_000
for env in ({}, {"SCD_SM_HEAD": "0"}):
    os.environ.update(env)
    s = scd.Solver(c3r["ptr"], c3r["idx"], c3r["val"], 20_000, c3r["n_cols"], c3r["y"], c3r["lam"], "dual", seed=3)
    inf = s.info()
    s.close()
    print("c3 rolling", env, inf["bins"][0], "tail_roll", inf["tail_roll"], "sm_head", inf["sm_head"], inf["sm_ch"],
          inf["sm_rh"], run(c3r, "dual"), flush=True)
    for k in env:
        del os.environ[k]
# criteo-shaped rows with λN = 2e5 (as in the 8-GPU shards): the hot-set kernel, explicit and implicit values
c5h = synth.gen_host(synth.CONFIGS["C5"].with_rows(1_000_000))
c5h["lam"] = 0.2
for env in ({},):
    os.environ.update(env)
    s = scd.Solver(c5h["ptr"], c5h["idx"], c5h["val"], c5h["n_rows"], c5h["n_cols"], c5h["y"], c5h["lam"], "dual",
                   seed=3)
    inf = s.info()
    s.close()
    print("c5 hot", env, inf["bins"][0], run(c5h, "dual"), flush=True)
    for k in env:
        del os.environ[k]
# fused peer-memory aggregation through a 1-rank communicator; device renumbering
os.environ["SCD_P2P_AGG"] = "1"
comm = scd.nccl_comm_init(scd.nccl_unique_id(), 1, 0)
print("p2p", run(e, "dual", nccl_comm=comm), run(e, "primal", nccl_comm=comm), flush=True)
scd.nccl_comm_destroy(comm)
del os.environ["SCD_P2P_AGG"]
r = scd.renumber(e["ptr"], e["idx"], e["val"], 300, 200, "csr")
print("renumber", int(r[3].sum()), flush=True)
print("sanitize_small done")
