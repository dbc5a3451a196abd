"""Sequential fp64 oracle trajectories over several epoch-permutation seeds (TEST FIXTURE WRITER).

Any uniformly random visiting order is an equally valid execution of Alg. 1, and the
per-epoch duality gap of the sequential method varies a lot with the order (C4, epoch 3: 6.0e-6 to
4.7e-5 over four seeds).  The per-epoch band of the full-size GPU tests (reading c27) is
therefore taken against this envelope, not against one seed.  Calls only oracle/ (and the shared
input generator synth/); writes tests/golden/seq_envelope_<cfg>.json.

  python tools/seq_envelope.py C3 6 3 4 5 6      # dual, 6 epochs, seeds 3..6
  python tools/seq_envelope.py C4 5 4 5 6 7      # primal (C3's matrix by feature)
  python tools/seq_envelope.py C5s 4 5 6 7 8     # dual, one 25 M-row shard of C5 (standalone, λN = 2e5)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import oracle
    import synth
    from oracle import ridge, solver

    which, E, seeds = sys.argv[1], int(sys.argv[2]), [int(x) for x in sys.argv[3:]]
    t0 = time.perf_counter()
    if which == "C5s":  # one GPU's shard of C5 as a standalone dual problem (25 M rows, values 1), with
        # λ = 8e-3 so that λN = 2e5 as in each shard of the 8-GPU run (global N = 200 M, λ = 1e-3)
        import dataclasses

        d = synth.gen_host(dataclasses.replace(synth.CONFIGS["C5"].with_rows(25_000_000), lam=8e-3))
    else:
        d = synth.gen_host(synth.CONFIGS["C3"])
    pr = solver.Problem.from_csr(d, csc=which == "C4")
    del d
    A = pr.A()
    print(f"setup {time.perf_counter() - t0:.1f} s", flush=True)
    dual = which != "C4"
    out = {"config": which, "epochs": E, "form": "dual" if dual else "primal", "lambda": pr.lam,
           "what": "sequential fp64 oracle (oracle.c Alg. 1) per-epoch duality gap (ridge.*_report, from scratch) "
                   "for several epoch-permutation seeds, full-size BASELINE configs[2]/[3]", "seeds": {}}
    for seed in seeds:
        if dual:
            x, sv, nrm = np.zeros(pr.N), np.zeros(pr.M), pr.row_norms()
        else:
            x, sv, nrm = np.zeros(pr.M), np.zeros(pr.N), pr.col_norms()
        gaps, Ps = [], []
        for t in range(1, E + 1):
            if dual:
                solver.dual_epoch(pr, x, sv, oracle.permutation(seed, t, pr.N), nrm)
                P, D, G = ridge.dual_report(A, pr.y, pr.lam, x)
            else:
                solver.primal_epoch(pr, x, sv, oracle.permutation(seed, t, pr.M), nrm)
                P, D, G = ridge.primal_report(A, pr.y, pr.lam, x)
            gaps.append(G)
            Ps.append(P)
        out["seeds"][str(seed)] = {"gap": gaps, "P": Ps}
        print(f"seed {seed}: " + " ".join(f"{g:.3e}" for g in gaps), flush=True)
    out["envelope_max"] = [max(v["gap"][t] for v in out["seeds"].values()) for t in range(E)]
    out["envelope_min"] = [min(v["gap"][t] for v in out["seeds"].values()) for t in range(E)]
    with open(os.path.join(ROOT, "tests", "golden", f"seq_envelope_{which}.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
