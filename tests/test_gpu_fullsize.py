"""Full-size checks (BASELINE.json configs[2] = C3, 350 000 x 16 609 143, 1.306e9 nnz) in the
launch configuration bench.py times (default schedule, tuned placement, library stream).

The oracle cannot replay an asynchronous epoch, so at this size the CUDA path is checked through
quantities the oracle computes independently from the GPU's returned model and the generated data:
  * the fp64 objective / gap kernels against scipy (the oracle's ridge.py) on the same model;
  * consistency of the maintained shared vector with Aᵀα on sampled columns (fp32 drift bound);
  * the gap after two epochs (the async epoch must actually descend).
The matrix is generated on the device by synth (bit-exact with the host twin, test_gpu_parity) and
copied to the host for the oracle."""
import numpy as np
import pytest

import synth
from oracle import ridge

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1702_07005_b200 as scd  # noqa: E402


def test_c3_dual_full_size_against_oracle():
    cfg = synth.CONFIGS["C3"]
    d = synth.gen_device(cfg)
    s = scd.Solver(d["ptr"], d["idx"], d["val"], d["n_rows"], d["n_cols"], d["y"], cfg.lam, "dual", seed=3)
    g0 = s.duality_gap()
    for t in (1, 2):
        s.epoch(t)
    P, D = s.objective()
    g = s.duality_gap()
    alpha = s.get_model().astype(np.float64)
    wbar = s.get_shared().astype(np.float64)
    A = ridge.as_matrix(d["ptr"].cpu().numpy(), d["idx"].cpu().numpy(), d["val"].cpu().numpy(), d["n_rows"],
                        d["n_cols"], "csr")
    y = d["y"].cpu().numpy().astype(np.float64)
    s.close()
    del d
    v = A.T @ alpha
    Po = ridge.primal_objective(A, y, cfg.lam, v / cfg.lam)
    Do = ridge.dual_objective(A, y, cfg.lam, alpha)
    go = ridge.gap_dual_gradform(A, y, cfg.lam, alpha)
    assert P == pytest.approx(Po, rel=1e-9)
    assert D == pytest.approx(Do, rel=1e-9)
    assert g == pytest.approx(go, rel=1e-6)
    assert g0 == pytest.approx(0.5 * (y @ y) / len(y), rel=1e-9)  # G_D(0) = ||y||²/(2N)
    assert g < 1e-3 * g0, (g0, g)
    # shared-vector consistency on the active features (fp32 accumulation drift)
    act = np.nonzero(v)[0]
    rng = np.random.default_rng(0)
    cols = rng.choice(act, size=min(20000, len(act)), replace=False)
    err = np.abs(wbar[cols] - v[cols]).max() / np.abs(v).max()
    assert err <= 1e-4, err


def test_c4_primal_full_size_against_oracle():
    """BASELINE configs[3] at K = 1: C3's matrix by feature (device stable transpose to CSC, 16.6 M
    columns of which 15.9 M empty, heavy columns on the cluster kernel), 3 epochs, certified by the
    oracle's fp64 objective and gap on the returned β and by w = Aβ on sampled rows."""
    cfg = synth.CONFIGS["C3"]
    d = synth.gen_device(cfg)
    cp, ci, cv = scd.transpose(d["ptr"], d["idx"], d["val"], d["n_rows"], d["n_cols"], "csr")
    s = scd.Solver(cp, ci, cv, d["n_rows"], d["n_cols"], d["y"], cfg.lam, "primal", seed=4)
    kinds = {b["lanes"] for b in s.info()["bins"]}
    assert 4096 in kinds and 256 in kinds, kinds  # cluster and CTA bins both exercised
    del cp, ci, cv
    g0 = s.duality_gap()
    for t in (1, 2, 3):
        s.epoch(t)
    P, D = s.objective()
    g = s.duality_gap()
    beta = s.get_model().astype(np.float64)
    w = s.get_shared().astype(np.float64)
    s.close()
    A = ridge.as_matrix(d["ptr"].cpu().numpy(), d["idx"].cpu().numpy(), d["val"].cpu().numpy(), d["n_rows"],
                        d["n_cols"], "csr")
    y = d["y"].cpu().numpy().astype(np.float64)
    del d
    Po = ridge.primal_objective(A, y, cfg.lam, beta)
    go = ridge.gap_primal_gradform(A, y, cfg.lam, beta)
    assert P == pytest.approx(Po, rel=1e-9)
    assert g == pytest.approx(go, rel=1e-6)
    assert g < 1e-3 * g0, (g0, g)
    u = A @ beta
    rng = np.random.default_rng(1)
    rows = rng.choice(len(y), size=20000, replace=False)
    err = np.abs(w[rows] - u[rows]).max() / np.abs(u).max()
    assert err <= 1e-4, err


def test_c5_shard_full_size_against_oracle():
    """One GPU's shard of BASELINE configs[4] (criteo-shaped, 25 M rows x 75 M features, 975 M one-hot
    entries, the CTA-combining 8-lane kernel) as a standalone dual problem: 3 epochs, certified by the
    oracle's fp64 objectives and gap on the returned α and by w̄ = Aᵀα on sampled features."""
    cfg = synth.CONFIGS["C5"].with_rows(25_000_000)
    d = synth.gen_device(cfg)
    s = scd.Solver(d["ptr"], d["idx"], d["val"], d["n_rows"], d["n_cols"], d["y"], cfg.lam, "dual", seed=5)
    assert s.info()["bins"][0]["lanes"] == 8
    g0 = s.duality_gap()
    for t in (1, 2, 3):
        s.epoch(t)
    P, D = s.objective()
    g = s.duality_gap()
    alpha = s.get_model().astype(np.float64)
    wbar = s.get_shared().astype(np.float64)
    s.close()
    A = ridge.as_matrix(d["ptr"].cpu().numpy(), d["idx"].cpu().numpy(), d["val"].cpu().numpy(), d["n_rows"],
                        d["n_cols"], "csr")
    y = d["y"].cpu().numpy().astype(np.float64)
    del d
    v = A.T @ alpha
    assert P == pytest.approx(ridge.primal_objective(A, y, cfg.lam, v / cfg.lam), rel=1e-9)
    assert D == pytest.approx(ridge.dual_objective(A, y, cfg.lam, alpha), rel=1e-9)
    assert g == pytest.approx(ridge.gap_dual_gradform(A, y, cfg.lam, alpha), rel=1e-6)
    assert g < 1e-2 * g0, (g0, g)
    act = np.nonzero(v)[0]
    rng = np.random.default_rng(2)
    cols = rng.choice(act, size=min(50000, len(act)), replace=False)
    err = np.abs(wbar[cols] - v[cols]).max() / np.abs(v).max()
    assert err <= 1e-4, err
