"""The sequential fp64 oracle run in the GPU schedule's visiting order (coordinates binned by length,
bins interleaved in S slices, each bin in its own permutation; reading c24), on C4 (primal)
or C3 (dual): separates the effect of the visiting order from that of asynchrony.

  python tools/orc_binned_order.py C4 6 8      # 6 epochs, 8 slices
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def binned_order(lengths, seed, epoch, S, lims=(64, 1024, 16384), order="longest", slices=None):
    """order: 'longest' (launch order of the library: longest bin first in every slice), 'shortest',
    or 'spread' (the heavy bin's slice split into `spread` pieces between the other bins' pieces).
    slices: per-bin slice counts (longest first) overriding S."""
    import oracle

    b = np.searchsorted(np.asarray(lims), lengths, side="left")  # 0: <=64, 1: <=1024, 2: <=16384, 3: more
    b[lengths == 0] = -1
    bins = [np.nonzero(b == k)[0] for k in (3, 2, 1, 0) if np.any(b == k)]  # launch order: longest first
    perms = [bl[oracle.permutation(seed, epoch, len(bl), stream=1 + i)] for i, bl in enumerate(bins)]
    if order == "shortest":
        perms = perms[::-1]
    out = []
    for q in range(S):
        for p in perms:
            n = len(p)
            out.append(p[n * q // S: n * (q + 1) // S])
    return np.concatenate(out)


def main():
    import synth
    from oracle import ridge, solver

    which, E = sys.argv[1], int(sys.argv[2])
    variants = [v.split(":") for v in sys.argv[3:]]  # "S:order"
    cfg = synth.CONFIGS["C3"]
    t0 = time.perf_counter()
    d = synth.gen_host(cfg)
    pr = solver.Problem.from_csr(d)
    A = pr.A()
    print(f"setup {time.perf_counter() - t0:.1f} s", flush=True)
    allres = {}
    for S, order in variants:
        S = int(S)
        res = []
        if which == "C4":
            lens = np.diff(pr.cptr)
            x, sv, nrm = np.zeros(pr.M), np.zeros(pr.N), pr.col_norms()
            for t in range(1, E + 1):
                solver.primal_epoch(pr, x, sv, binned_order(lens, 4, t, S, order=order), nrm)
                res.append(ridge.primal_report(A, pr.y, pr.lam, x)[2])
        else:
            lens = np.diff(pr.rptr)
            x, sv, nrm = np.zeros(pr.N), np.zeros(pr.M), pr.row_norms()
            for t in range(1, E + 1):
                solver.dual_epoch(pr, x, sv, binned_order(lens, 3, t, S, lims=(64, 64, 16384), order=order), nrm)
                res.append(ridge.dual_report(A, pr.y, pr.lam, x)[2])
        print(f"S={S:3d} {order:9s} gaps " + " ".join(f"{g:.3e}" for g in res), flush=True)
        allres[f"{S}:{order}"] = res
    os.makedirs(os.path.join(ROOT, "profiles", "data"), exist_ok=True)
    json.dump(dict(which=which, variants=allres),
              open(os.path.join(ROOT, "profiles", "data", f"orc_binned_{which}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
