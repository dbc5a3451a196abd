"""Full-size per-epoch comparison of the benchmarked schedule with the sequential fp64 oracle.

  python tools/fullsize_band.py C3 6     # dual, BASELINE configs[2], bench.py's schedule (seed 3)
  python tools/fullsize_band.py C4 6     # primal, C3's matrix by feature (K = 1, seed 4)

The CUDA path runs E epochs of the default schedule (tuned placement, library stream) with the
fp64 from-scratch gap after every epoch (off the clock); the oracle (oracle.c Alg. 1, 1 core, fp64)
runs E sequential epochs on the same matrix (host copy of the synth output; the CSC for the primal
is the oracle's own transpose) and evaluates P, D and the gap from scratch (ridge.*_report).
Prints per-epoch gaps, their ratio, and the objective of each side; writes JSON if asked."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(which: str, epochs: int, oracle_epochs: int | None = None):
    import torch

    import oracle
    import synth
    from oracle import ridge, solver
    import paper_1702_07005_b200 as scd

    oracle_epochs = oracle_epochs or epochs
    cfg = synth.CONFIGS["C3"]
    d = synth.gen_device(cfg)
    N, M = d["n_rows"], d["n_cols"]
    out = {"config": which, "epochs": epochs}
    # ---- CUDA path (the benchmarked schedule)
    t0 = time.perf_counter()
    if which == "C3":
        s = scd.Solver(d["ptr"], d["idx"], d["val"], N, M, d["y"], cfg.lam, "dual", seed=3)
    else:
        cp, ci, cv = scd.transpose(d["ptr"], d["idx"], d["val"], N, M, "csr")
        s = scd.Solver(cp, ci, cv, N, M, d["y"], cfg.lam, "primal", seed=4)
    out["schedule"] = s.info()
    gpu = []
    stream = torch.cuda.ExternalStream(s.stream_handle)
    for t in range(1, epochs + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.epoch(t)
        e1.record(stream)
        torch.cuda.synchronize()
        P, D = s.objective()
        gpu.append(dict(epoch=t, ms=e0.elapsed_time(e1), P=P, D=D, gap=s.duality_gap()))
    x_gpu = s.get_model().astype(np.float64)
    s.close()
    if which != "C3":
        del cp, ci, cv
    out["gpu_s"] = time.perf_counter() - t0
    host = dict(ptr=d["ptr"].cpu().numpy(), idx=d["idx"].cpu().numpy(), val=d["val"].cpu().numpy(),
                y=d["y"].cpu().numpy(), n_rows=N, n_cols=M, lam=cfg.lam)
    del d
    torch.cuda.empty_cache()
    # ---- oracle (sequential fp64, 1 core)
    t0 = time.perf_counter()
    pr = solver.Problem.from_csr(host)
    A = pr.A()
    out["oracle_setup_s"] = time.perf_counter() - t0
    orc = []
    if which == "C3":
        x, sv, nrm = np.zeros(N), np.zeros(M), pr.row_norms()
        Pg, Dg, Gg = ridge.dual_report(A, pr.y, pr.lam, x_gpu)
    else:
        x, sv, nrm = np.zeros(M), np.zeros(N), pr.col_norms()
        Pg, Dg, Gg = ridge.primal_report(A, pr.y, pr.lam, x_gpu)
    out["gpu_model_by_oracle"] = dict(P=Pg, D=Dg, gap=Gg)
    ep_s = []
    for t in range(1, oracle_epochs + 1):
        t1 = time.perf_counter()
        if which == "C3":
            solver.dual_epoch(pr, x, sv, oracle.permutation(3, t, N), nrm)
        else:
            solver.primal_epoch(pr, x, sv, oracle.permutation(4, t, M), nrm)
        ep_s.append(time.perf_counter() - t1)
        P, D, G = (ridge.dual_report if which == "C3" else ridge.primal_report)(A, pr.y, pr.lam, x)
        orc.append(dict(epoch=t, s=ep_s[-1], P=P, D=D, gap=G))
        print(f"oracle epoch {t}: {ep_s[-1]:.2f} s gap {G:.3e} P {P:.12g}", flush=True)
    out["oracle"] = orc
    out["gpu"] = gpu
    out["ratio"] = [g["gap"] / o["gap"] for g, o in zip(gpu, orc)]
    Pstar = orc[-1]["P"]
    out["Pstar"] = Pstar
    out["Pstar_cert"] = orc[-1]["gap"]  # P_orc - P* <= G_orc (weak duality)
    out["gpu_rel_obj"] = abs(Pg - Pstar) / abs(Pstar)
    return out


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "C3"
    E = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    EO = int(sys.argv[3]) if len(sys.argv) > 3 else E
    out = run(which, E, EO)
    for g, o in zip(out["gpu"], out["oracle"]):
        print(f"epoch {g['epoch']}: gpu gap {g['gap']:.3e} ({g['ms']:.2f} ms)  oracle gap {o['gap']:.3e} "
              f"({o['s']:.2f} s)  ratio {g['gap'] / o['gap']:.3f}")
    print(f"P* (oracle, {len(out['oracle'])} epochs) {out['Pstar']:.12g} cert {out['Pstar_cert']:.2e}; gpu model by oracle "
          f"P {out['gpu_model_by_oracle']['P']:.12g} gap {out['gpu_model_by_oracle']['gap']:.3e} rel {out['gpu_rel_obj']:.2e}")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"band_{which}.json"), "w") as f:
        json.dump(out, f, indent=1, default=str)


if __name__ == "__main__":
    main()
