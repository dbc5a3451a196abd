"""Per-epoch gaps with and without the block order of the short-coordinate bins (reading c28), against
the sequential envelope (4 oracle seeds), on the GPU tests' criteo-shaped problems.

  python tools/block_order_check.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    import synth
    from envelope import envelope
    from oracle import solver
    import paper_1702_07005_b200 as scd

    cases = [("c5 prefix 2M, lam 0.1", synth.CONFIGS["C5"].with_rows(2_000_000), 0.1, 8),
             ("short rows c5_scaled(200k, 1e-2), lam 1e-3", synth.c5_scaled(200_000, 1e-2), 1e-3, 8),
             ("c5 prefix 2M, lam 1e-3", synth.CONFIGS["C5"].with_rows(2_000_000), 1e-3, 8)]
    for name, cfg, lam, E in cases:
        d = synth.gen_host(cfg)
        pr = solver.Problem.from_csr(d, lam=lam, csc=False)
        hi, lo = envelope(pr, "dual", E)
        print(name, "envelope", " ".join("%.2e" % x for x in hi), flush=True)
        for bo in (0, 1):
            s = scd.Solver(d["ptr"], d["idx"], d["val"], pr.N, pr.M, d["y"], lam, "dual", seed=5, block_order=bo)
            b = s.info()["bins"][0]
            g = []
            for t in range(1, E + 1):
                s.epoch(t)
                g.append(s.duality_gap())
            s.close()
            print(f"  block_order={bo} (lanes {b['lanes']} hot {b['hot']} grid {b['grid']} flush {b['flush']} cap {b['cap']} "
                  f"count {b['count']}): ratio " + " ".join("%.2f" % (x / h) for x, h in zip(g, hi)), flush=True)


if __name__ == "__main__":
    main()
