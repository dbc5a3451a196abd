"""Full-size checks (BASELINE.json configs[2] = C3, 350 000 x 16 609 143, 1.306e9 nnz; configs[3] = C4,
the same matrix by feature; one GPU's shard of configs[4]) in the launch configuration bench.py times
(default schedule, tuned placement, library stream).

C3 and C4 run the sequential fp64 oracle (oracle.c Alg. 1, one core, ~3-6 s per epoch) beside the
CUDA path on the same matrix (the host copy of the synth output; the primal's CSC is the oracle's own
transpose) and compare them epoch by epoch: the asynchronous iterates are not unique (reading c19),
so the comparison is on the duality gap per epoch ("near-perfect convergence ... as a function
of epochs", the band recorded as reading c27 in DESIGN.md) and on the optimum (north_star: objective
within 1e-5 relative of the oracle's converged objective, gap <= 1e-5), the GPU's model being
evaluated by the oracle in fp64.  The C5 shard (no full oracle run fits the test budget) is
certified through the oracle's objective and gap on the GPU's model (weak duality)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import ridge, solver

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1702_07005_b200 as scd  # noqa: E402

GPU_EPOCHS = 5
BAND = 1.25         # reading c27: measured 1.06-1.09 x the envelope maximum (C3, C4), 0.3-1.1 elsewhere
ORACLE_EPOCHS = 6   # C3 oracle gap 1.2e-10 after 6 epochs (profiles/data/band_C3.json): P* certified to ~2e-10


def _envelope(name):
    import json
    import os

    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"seq_envelope_{name}.json")) as f:
        return json.load(f)


def _side_by_side(form: str, band: float, envelope: str, cfg=None, seed: int = 3, implicit: bool = False,
                  gpu_epochs: int = GPU_EPOCHS, oracle_epochs: int = ORACLE_EPOCHS, gap_at: int = 3):
    cfg = cfg or synth.CONFIGS["C3"]
    d = synth.gen_device(cfg)
    N, M = d["n_rows"], d["n_cols"]
    if implicit:  # one-hot data with implicit values (NEXT-1, P:460 footnote): the library gets val = NULL
        assert bool((d["val"] == 1.0).all())
        d["val"] = None
    if form == "dual":
        s = scd.Solver(d["ptr"], d["idx"], d["val"], N, M, d["y"], cfg.lam, "dual", seed=seed)
    else:
        cp, ci, cv = scd.transpose(d["ptr"], d["idx"], d["val"], N, M, "csr")
        s = scd.Solver(cp, ci, cv, N, M, d["y"], cfg.lam, "primal", seed=seed)
        kinds = {b["lanes"] for b in s.info()["bins"]}
        assert 4096 in kinds and 256 in kinds, kinds  # cluster and CTA bins both exercised
        del cp, ci, cv
    info = s.info()
    g0 = s.duality_gap()
    gaps, objs = [], []
    for t in range(1, gpu_epochs + 1):
        s.epoch(t)
        gaps.append(s.duality_gap())
        objs.append(s.objective())
    x = s.get_model().astype(np.float64)
    sv = s.get_shared().astype(np.float64)
    s.close()
    host = dict(ptr=d["ptr"].cpu().numpy(), idx=d["idx"].cpu().numpy(),
                val=None if d["val"] is None else d["val"].cpu().numpy(), y=d["y"].cpu().numpy(), n_rows=N, n_cols=M,
                lam=cfg.lam)
    del d
    torch.cuda.empty_cache()
    pr = solver.Problem.from_csr(host, csc=form == "primal")
    A = pr.A()
    report = ridge.dual_report if form == "dual" else ridge.primal_report
    Pg, Dg, Gg = report(A, pr.y, pr.lam, x)  # the GPU's final model, evaluated by the oracle in fp64
    xo, svo = (np.zeros(N), np.zeros(M)) if form == "dual" else (np.zeros(M), np.zeros(N))
    nrm = pr.row_norms() if form == "dual" else pr.col_norms()
    orc = []
    for t in range(1, oracle_epochs + 1):
        if form == "dual":
            solver.dual_epoch(pr, xo, svo, oracle.permutation(seed, t, N), nrm)
        else:
            solver.primal_epoch(pr, xo, svo, oracle.permutation(seed, t, M), nrm)
        orc.append(report(A, pr.y, pr.lam, xo))
    Pstar, Gstar = orc[-1][0], orc[-1][2]
    print("gpu gaps", ["%.3e" % g for g in gaps])
    print("seq gaps", ["%.3e" % o[2] for o in orc])
    print("ratios  ", ["%.3f" % (g / o[2]) for g, o in zip(gaps, orc)])
    print(f"P* {Pstar:.12g} (cert {Gstar:.1e}), GPU model: P {Pg:.12g} gap {Gg:.3e}")
    # the GPU's fp64 evaluation kernels agree with the oracle's on the same model
    assert objs[-1][0] == pytest.approx(Pg, rel=1e-9) and objs[-1][1] == pytest.approx(Dg, rel=1e-9)
    assert gaps[-1] == pytest.approx(Gg, rel=1e-6)
    # the gap at the start is the closed form ||y||²/(2N) (dual G_D(0)) / ||Aᵀy||²/(2λN²) (primal G_P(0))
    g0_ref = 0.5 * float(pr.y @ pr.y) / N if form == "dual" else float(np.sum((A.T @ pr.y) ** 2)) / (2 * pr.lam * N * N)
    assert g0 == pytest.approx(g0_ref, rel=1e-9)
    # per-epoch band against the sequential method (reading c27): any random visiting order is a valid
    # Alg. 1 run, and the sequential gap per epoch varies with the order (tests/golden/seq_envelope_*.json,
    # written by tools/seq_envelope.py from oracle/ only); the GPU must stay within `band` x the largest
    # sequential gap of the recorded seeds, while above the fp32 floor
    env = _envelope(envelope)
    print("envelope", ["%.3e" % e for e in env["envelope_max"]])
    print("ratio to envelope max", ["%.3f" % (g / e) for g, e in zip(gaps, env["envelope_max"])])
    assert env["lambda"] == pytest.approx(cfg.lam) and str(seed) in env["seeds"]
    # the recorded trajectory of this seed is the live oracle run's (same data, same order)
    for o, e in zip(orc, env["seeds"][str(seed)]["gap"]):
        assert o[2] == pytest.approx(e, rel=1e-6)
    for t, g in enumerate(gaps[:len(env["envelope_max"])]):
        if env["envelope_min"][t] > 1e-8 * g0:
            assert g <= band * env["envelope_max"][t], (t + 1, g, env["envelope_max"][t], band)
    # north_star tolerances at full size: gap <= 1e-5 and the objective within 1e-5 of the optimum
    assert gaps[gap_at - 1] <= 1e-5, gaps
    # P* is certified by the oracle's own gap (weak duality: P_orc - P* <= G_orc), 100x inside the tolerance
    assert Gstar <= 1e-7 * abs(Pstar) and abs(Pg - Pstar) <= 1e-5 * abs(Pstar), (Pg, Pstar, Gstar)
    return A, x, sv, info


def test_c3_dual_full_size_against_oracle():
    """Bench schedule on C3 (k_epoch_sm_tma, one launch per epoch): per-epoch gap within 1.25x of the
    sequential fp64 SDCA's envelope over 4 seeds (measured <= 1.07x), optimum to 1e-5."""
    A, alpha, wbar, info = _side_by_side("dual", BAND, "C3")
    b = info["bins"][0]
    assert len(info["bins"]) == 1 and b["head"] > 0 and info["tail_roll"] > 0 and info["sm_head"] > 0, info  # the bench kernel
    # shared-vector consistency on the active features (fp32 accumulation drift)
    v = A.T @ alpha
    act = np.nonzero(v)[0]
    rng = np.random.default_rng(0)
    cols = rng.choice(act, size=min(20000, len(act)), replace=False)
    err = np.abs(wbar[cols] - v[cols]).max() / np.abs(v).max()
    assert err <= 1e-4, err


def test_c4_primal_full_size_against_oracle():
    """BASELINE configs[3] at K = 1: C3's matrix by feature (device stable transpose to CSC, 16.6 M
    columns of which 15.9 M empty, heavy columns on the cluster kernel), per-epoch band against the
    sequential fp64 SCD (reading c27) and the optimum to 1e-5; w = Aβ on sampled rows."""
    A, beta, w, _ = _side_by_side("primal", BAND, "C4", seed=4, gap_at=4)
    u = A @ beta
    rng = np.random.default_rng(1)
    rows = rng.choice(A.shape[0], size=20000, replace=False)
    err = np.abs(w[rows] - u[rows]).max() / np.abs(u).max()
    # fp32 drift of the residual: every r_i takes one RED per stored entry of row i per epoch (~3 700 on
    # average, 16 384 at most), 5 epochs: ~1e5 roundings at ulp(|r_i|) ~ 6e-8 |r_i|; observed 1.0e-4 of
    # max |Aβ| after 5 epochs (8e-5 after 3).  recompute_every / scd_recompute_shared (NEXT-2) reset it.
    assert err <= 5e-4, err


def test_c5_shard_full_size_against_oracle():
    """One GPU's shard of BASELINE configs[4] (criteo-shaped, 25 M rows x 75 M features, 975 M one-hot
    entries with implicit values: val = NULL, NEXT-1) as a standalone dual problem (λN as in the 8-GPU run)
    on the hot-set kernel
    (k_epoch_group_hot), beside the sequential fp64 SDCA on the same rows (values 1.0 stored
    explicitly): per-epoch band (reading c27), gap <= 1e-5 and the optimum to 1e-5."""
    import dataclasses

    # λ = 8e-3: λN = 2e5 as in every shard of the 8-GPU run (N = 200 M, λ = 1e-3), so the staleness bound
    # and the hot-set kernel's launch shape are those of the benchmarked shard (bench.py c5_shard)
    cfg = dataclasses.replace(synth.CONFIGS["C5"].with_rows(25_000_000), lam=8e-3)
    A, alpha, wbar, info = _side_by_side("dual", BAND, "C5s", cfg=cfg, seed=5, implicit=True, gpu_epochs=4,
                                         oracle_epochs=7, gap_at=4)
    b = info["bins"][0]
    assert len(info["bins"]) == 1 and b["lanes"] == 8 and b["hot"] > 0, info
    v = A.T @ alpha
    act = np.nonzero(v)[0]
    rng = np.random.default_rng(2)
    cols = rng.choice(act, size=min(50000, len(act)), replace=False)
    err = np.abs(wbar[cols] - v[cols]).max() / np.abs(v).max()
    assert err <= 1e-4, err
