"""Pins of the fp64 oracle against what the paper and mathematics fix (not against itself).

P:n = PAPER.md line n; S:n = SPEC.md line n (hand-derived values of the paper's formulas).
Each pin is chosen so that a plausible mistake in the oracle (dropped term, wrong sign or
index, transposed operand) fails it:
  - SPEC hand values of Eq. (1)-(7) on 1-2 dimensional instances (golden fixture)
  - the normal-equation closed form (a library solve of AᵀA + λN I, independent of SCD)
  - per-update stationarity of the exact 1-D minimiser
  - monotone objective under exact coordinate descent
  - strong duality and the Fenchel maps at the closed-form optimum
  - finite-difference gradients (the gap's gradient form uses them)
  - the exact line search: 3-point quadratic fit and golden-section search
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth
from oracle import ridge, solver


def _prob_from_dense(A, y, lam):
    A = np.asarray(A, np.float32)
    S = sp.csr_matrix(A)
    S.sort_indices()
    d = dict(ptr=S.indptr.astype(np.int64), idx=S.indices.astype(np.int32), val=S.data.astype(np.float32),
             y=np.asarray(y, np.float32), n_rows=A.shape[0], n_cols=A.shape[1], lam=lam)
    return solver.Problem.from_csr(d)


def _rand_prob(n, m, density, seed, lam):
    d = synth.random_sparse(n, m, density, seed)
    d["lam"] = lam
    return solver.Problem.from_csr(d)


# ------------------------------------------------------------------ SPEC hand values
def test_hand_objectives(golden):
    for c in golden["primal_objective"]:
        A = np.array(c["A"])
        assert ridge.primal_objective(sp.csr_matrix(A), np.array(c["y"]), c["lam"], np.array(c["beta"])) == \
            pytest.approx(c["expect"], rel=1e-14, abs=1e-15), c["cite"]
    for c in golden["dual_objective"]:
        A = np.array(c["A"])
        assert ridge.dual_objective(sp.csr_matrix(A), np.array(c["y"]), c["lam"], np.array(c["alpha"])) == \
            pytest.approx(c["expect"], rel=1e-14, abs=1e-15), c["cite"]


def test_hand_maps(golden):
    for c in golden["dual_to_primal"]:
        np.testing.assert_allclose(ridge.dual_to_primal(sp.csr_matrix(np.array(c["A"])), c["lam"], np.array(c["alpha"])),
                                   c["expect"], rtol=1e-14, err_msg=c["cite"])
    for c in golden["primal_to_dual"]:
        np.testing.assert_allclose(ridge.primal_to_dual(sp.csr_matrix(np.array(c["A"])), np.array(c["y"]),
                                                        np.array(c["beta"])), c["expect"], rtol=1e-14, err_msg=c["cite"])


def test_hand_closed_form(golden):
    for c in golden["closed_form"]:
        np.testing.assert_allclose(ridge.closed_form(sp.csr_matrix(np.array(c["A"])), np.array(c["y"]), c["lam"]),
                                   c["expect"], rtol=1e-13, atol=1e-15, err_msg=c["cite"])


def test_hand_primal_update(golden):
    for c in golden["primal_update"]:
        pr = _prob_from_dense(c["A"], c["y"], c["lam"])
        beta = np.array(c["beta"], np.float64)
        w = np.array(c["w"], np.float64)
        b0 = beta[c["m"]]
        solver.primal_epoch(pr, beta, w, [c["m"]])
        assert beta[c["m"]] - b0 == pytest.approx(c["expect_delta"], rel=1e-14), c["cite"]
        np.testing.assert_allclose(w, c["expect_w"], rtol=1e-14, atol=1e-15, err_msg=c["cite"])


def test_hand_dual_update(golden):
    for c in golden["dual_update"]:
        pr = _prob_from_dense(c["A"], c["y"], c["lam"])
        alpha = np.array(c["alpha"], np.float64)
        wbar = np.array(c["wbar"], np.float64)
        a0 = alpha[c["n"]]
        solver.dual_epoch(pr, alpha, wbar, [c["n"]])
        assert alpha[c["n"]] - a0 == pytest.approx(c["expect_delta"], rel=1e-14), c["cite"]
        np.testing.assert_allclose(wbar, c["expect_wbar"], rtol=1e-14, atol=1e-15, err_msg=c["cite"])


def test_hand_gamma(golden):
    for c in golden["gamma_primal"]:
        g = ridge.gamma_primal(np.array(c["w"]), np.array(c["y"]), np.array(c["beta"]), np.array(c["dw"]),
                               np.array(c["dbeta"]), c["lam"], c["N"])
        assert g == pytest.approx(c["expect"], rel=1e-14, abs=0), c["cite"]
    for c in golden["gamma_dual"]:
        g = ridge.gamma_dual(np.array(c["alpha"]), np.array(c["wbar"]), np.array(c["y"]), np.array(c["dalpha"]),
                             np.array(c["dwbar"]), c["lam"], c["N"])
        assert g == pytest.approx(c["expect"], rel=1e-14), c["cite"]


# ------------------------------------------------------------------ closed form / convergence
@pytest.mark.parametrize("lam", [1e-3, 0.1, 1.0])
@pytest.mark.parametrize("seed", [11, 12, 13])
def test_sequential_scd_reaches_closed_form(lam, seed):
    """Alg. 1 converges to β* = (AᵀA + λN I)⁻¹Aᵀy; SDCA mapped through Eq. (5) too."""
    pr = _rand_prob(120, 40, 0.3, seed, lam)
    A = pr.A()
    bstar = ridge.closed_form(A, pr.y, lam)
    beta, w, h = solver.solve(pr, "primal", 3000, seed=seed, record=False)
    np.testing.assert_allclose(beta, bstar, atol=1e-9 * max(1, np.abs(bstar).max()))
    alpha, wbar, _ = solver.solve(pr, "dual", 3000, seed=seed, record=False)
    np.testing.assert_allclose(ridge.dual_to_primal(A, lam, alpha), bstar, atol=1e-8 * max(1, np.abs(bstar).max()))
    # the shared vectors stay consistent with the models
    np.testing.assert_allclose(w, A @ beta, atol=1e-10)
    np.testing.assert_allclose(wbar, A.T @ alpha, atol=1e-10)


def test_c1_dense_closed_form():
    """Config C1 (BASELINE.json configs[0]): 1000x100 dense, λ = 1e-3, primal SCD vs normal equations."""
    d = synth.gen_host(synth.CONFIGS["C1"])
    pr = solver.Problem.from_csr(d)
    A = pr.A()
    bstar = ridge.closed_form(A, pr.y, pr.lam)
    beta, w, h = solver.solve(pr, "primal", 60, seed=1)
    assert np.abs(beta - bstar).max() <= 1e-10 * np.abs(bstar).max()
    assert h[-1]["gap"] <= 1e-12
    assert abs(h[-1]["P"] - ridge.primal_objective(A, pr.y, pr.lam, bstar)) <= 1e-12


def test_strong_duality_and_maps():
    """P(β*) = D(α*), β* = Aᵀα*/λ, α* = (y - Aβ*)/N."""
    pr = _rand_prob(60, 25, 0.4, 5, 1e-2)
    A = pr.A()
    bstar = ridge.closed_form(A, pr.y, pr.lam)
    astar = ridge.closed_form_dual(A, pr.y, pr.lam)
    assert ridge.primal_objective(A, pr.y, pr.lam, bstar) == pytest.approx(ridge.dual_objective(A, pr.y, pr.lam, astar),
                                                                          rel=1e-12)
    np.testing.assert_allclose(ridge.dual_to_primal(A, pr.lam, astar), bstar, rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(ridge.primal_to_dual(A, pr.y, bstar), astar, rtol=1e-10, atol=1e-13)
    assert ridge.gap_primal(A, pr.y, pr.lam, bstar) <= 1e-13
    assert ridge.gap_dual(A, pr.y, pr.lam, astar) <= 1e-13


# ------------------------------------------------------------------ per-update properties
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_stationarity_after_every_update(seed):
    """After each exact coordinate step the partial derivative vanishes."""
    pr = _rand_prob(80, 30, 0.3, seed, 0.05)
    beta, w = np.zeros(pr.M), np.zeros(pr.N)
    alpha, wbar = np.zeros(pr.N), np.zeros(pr.M)
    for t in range(1, 4):
        st = solver.primal_epoch(pr, beta, w, oracle.permutation(seed, t, pr.M), stat=True)
        assert np.abs(st).max() <= 1e-12
        st = solver.dual_epoch(pr, alpha, wbar, oracle.permutation(seed, t, pr.N), stat=True)
        assert np.abs(st).max() <= 1e-10


def test_objective_monotone_per_update():
    """Exact coordinate minimisation never increases P (primal) / never decreases D (dual)."""
    pr = _rand_prob(40, 15, 0.4, 9, 0.01)
    A = pr.A()
    beta, w = np.zeros(pr.M), np.zeros(pr.N)
    prev = ridge.primal_objective(A, pr.y, pr.lam, beta)
    for t in range(1, 4):
        for m in oracle.permutation(9, t, pr.M):
            solver.primal_epoch(pr, beta, w, [m])
            cur = ridge.primal_objective(A, pr.y, pr.lam, beta)
            assert cur <= prev + 1e-12 * abs(prev)
            prev = cur
    alpha, wbar = np.zeros(pr.N), np.zeros(pr.M)
    prev = ridge.dual_objective(A, pr.y, pr.lam, alpha)
    for t in range(1, 4):
        for n in oracle.permutation(9, t, pr.N):
            solver.dual_epoch(pr, alpha, wbar, [n])
            cur = ridge.dual_objective(A, pr.y, pr.lam, alpha)
            assert cur >= prev - 1e-12 * abs(prev)
            prev = cur


def test_update_is_exact_line_minimiser():
    """Δ of Eq. (2) equals the argmin of the 1-D quadratic P(β + δ e_m) found numerically."""
    pr = _rand_prob(50, 20, 0.4, 21, 0.03)
    A = pr.A()
    rng = np.random.default_rng(0)
    beta = rng.standard_normal(pr.M)
    for m in range(pr.M):
        b2, w2 = beta.copy(), A @ beta
        solver.primal_epoch(pr, b2, w2, [m])
        q = [ridge.primal_objective(A, pr.y, pr.lam, beta + d * np.eye(pr.M)[m]) for d in (-1.0, 0.0, 1.0)]
        dstar = (q[0] - q[2]) / (2 * (q[0] + q[2] - 2 * q[1]))
        assert b2[m] - beta[m] == pytest.approx(dstar, rel=1e-9, abs=1e-12)


# ------------------------------------------------------------------ gap forms and gradients
def test_gap_forms_agree_and_nonnegative():
    pr = _rand_prob(70, 30, 0.3, 31, 0.02)
    A = pr.A()
    rng = np.random.default_rng(1)
    for _ in range(10):
        beta = rng.standard_normal(pr.M) * 0.3
        alpha = rng.standard_normal(pr.N) * 0.05
        g1, g2 = ridge.gap_primal(A, pr.y, pr.lam, beta), ridge.gap_primal_gradform(A, pr.y, pr.lam, beta)
        assert g1 >= 0 and g2 == pytest.approx(g1, rel=1e-10)
        g1, g2 = ridge.gap_dual(A, pr.y, pr.lam, alpha), ridge.gap_dual_gradform(A, pr.y, pr.lam, alpha)
        assert g1 >= 0 and g2 == pytest.approx(g1, rel=1e-10)
        # weak duality
        assert ridge.primal_objective(A, pr.y, pr.lam, beta) >= ridge.dual_objective(A, pr.y, pr.lam, alpha) - 1e-12


def test_reports_match_definitions():
    """ridge.dual_report / primal_report (shared sparse products, used at full size) equal the
    separate definitions at random points, and at the closed-form optimum P = D and G = 0."""
    pr = _rand_prob(70, 30, 0.3, 32, 0.02)
    A = pr.A()
    rng = np.random.default_rng(3)
    for _ in range(5):
        beta = rng.standard_normal(pr.M) * 0.3
        alpha = rng.standard_normal(pr.N) * 0.05
        P, D, G = ridge.dual_report(A, pr.y, pr.lam, alpha)
        assert P == pytest.approx(ridge.primal_objective(A, pr.y, pr.lam, ridge.dual_to_primal(A, pr.lam, alpha)),
                                  rel=1e-12)
        assert D == pytest.approx(ridge.dual_objective(A, pr.y, pr.lam, alpha), rel=1e-12)
        assert G == pytest.approx(ridge.gap_dual(A, pr.y, pr.lam, alpha), rel=1e-9)
        P, D, G = ridge.primal_report(A, pr.y, pr.lam, beta)
        assert P == pytest.approx(ridge.primal_objective(A, pr.y, pr.lam, beta), rel=1e-12)
        assert D == pytest.approx(ridge.dual_objective(A, pr.y, pr.lam, ridge.primal_to_dual(A, pr.y, beta)),
                                  rel=1e-12)
        assert G == pytest.approx(ridge.gap_primal(A, pr.y, pr.lam, beta), rel=1e-9)
    bstar = ridge.closed_form(A, pr.y, pr.lam)
    astar = ridge.closed_form_dual(A, pr.y, pr.lam)
    for P, D, G in (ridge.primal_report(A, pr.y, pr.lam, bstar), ridge.dual_report(A, pr.y, pr.lam, astar)):
        assert P == pytest.approx(D, rel=1e-12) and G <= 1e-20


def test_gradients_finite_difference():
    """Analytic partials P:83 and P:109 vs central differences."""
    pr = _rand_prob(30, 12, 0.5, 41, 0.1)
    A = pr.A()
    rng = np.random.default_rng(2)
    beta, alpha = rng.standard_normal(pr.M), rng.standard_normal(pr.N) * 0.1
    gp, gd = ridge.primal_grad(A, pr.y, pr.lam, beta), ridge.dual_grad(A, pr.y, pr.lam, alpha)
    h = 1e-5
    for m in range(pr.M):
        e = np.eye(pr.M)[m] * h
        fd = (ridge.primal_objective(A, pr.y, pr.lam, beta + e) - ridge.primal_objective(A, pr.y, pr.lam, beta - e)) / (2 * h)
        assert fd == pytest.approx(gp[m], rel=1e-6, abs=1e-8)
    for n in range(pr.N):
        e = np.eye(pr.N)[n] * h
        fd = (ridge.dual_objective(A, pr.y, pr.lam, alpha + e) - ridge.dual_objective(A, pr.y, pr.lam, alpha - e)) / (2 * h)
        assert fd == pytest.approx(gd[n], rel=1e-6, abs=1e-8)


# ------------------------------------------------------------------ aggregation γ
def _golden_section(f, a, b, tol=1e-10):
    g = (np.sqrt(5) - 1) / 2
    c, d = b - g * (b - a), a + g * (b - a)
    while abs(b - a) > tol:
        if f(c) < f(d):
            b = d
        else:
            a = c
        c, d = b - g * (b - a), a + g * (b - a)
    return 0.5 * (a + b)


def test_gamma_is_exact_line_search():
    """γ* of Eq. (7) (corrected, c3/c5) and γ̄* (corrected, c4) are the exact minimiser of the
    stated line search: checked by a 3-point quadratic fit and golden section
    on the states produced by real distributed rounds and on random states."""
    pr = _rand_prob(100, 40, 0.3, 51, 0.01)
    A = pr.A()
    N = pr.N
    rng = np.random.default_rng(3)
    for trial in range(20):
        beta0 = rng.standard_normal(pr.M) * 0.2
        dbeta = rng.standard_normal(pr.M) * 0.1 * (rng.random(pr.M) < 0.5)
        w0, dw = A @ beta0, A @ dbeta
        g = ridge.gamma_primal(w0, pr.y, beta0, dw, dbeta, pr.lam, N)
        q = lambda t: ridge.primal_objective_at(pr.y, pr.lam, beta0 + t * dbeta, w0 + t * dw)
        g3 = (q(-1.0) - q(1.0)) / (2 * (q(1.0) + q(-1.0) - 2 * q(0.0)))
        assert g == pytest.approx(g3, rel=1e-8, abs=1e-12)
        assert g == pytest.approx(_golden_section(q, -10 * abs(g) - 1, 10 * abs(g) + 1), abs=1e-6)
        assert q(g) <= min(q(0.0), q(0.25)) + 1e-15

        alpha0 = rng.standard_normal(N) * 0.01
        dalpha = rng.standard_normal(N) * 0.01 * (rng.random(N) < 0.5)
        wb0, dwb = A.T @ alpha0, A.T @ dalpha
        gd = ridge.gamma_dual(alpha0, wb0, pr.y, dalpha, dwb, pr.lam, N)
        qd = lambda t: -ridge.dual_objective_at(pr.y, pr.lam, alpha0 + t * dalpha, wb0 + t * dwb)
        g3 = (qd(-1.0) - qd(1.0)) / (2 * (qd(1.0) + qd(-1.0) - 2 * qd(0.0)))
        assert gd == pytest.approx(g3, rel=1e-8, abs=1e-12)
        assert gd == pytest.approx(_golden_section(qd, -10 * abs(gd) - 1, 10 * abs(gd) + 1), abs=1e-6)


def test_printed_eq7_is_not_the_line_search_minimiser():
    """Documents reading c3: the printed numerator <w, Δw> is NOT the minimiser (it would pass
    the 3-point test only by accident); the corrected <w - y, Δw> is."""
    pr = _rand_prob(60, 25, 0.4, 61, 0.01)
    A = pr.A()
    rng = np.random.default_rng(4)
    beta0, dbeta = rng.standard_normal(pr.M) * 0.2, rng.standard_normal(pr.M) * 0.1
    w0, dw = A @ beta0, A @ dbeta
    N, lam = pr.N, pr.lam
    printed = -(w0 @ dw + N * lam * beta0 @ dbeta) / (dw @ dw + N * lam * dbeta @ dbeta)
    q = lambda t: ridge.primal_objective_at(pr.y, lam, beta0 + t * dbeta, w0 + t * dw)
    g3 = (q(-1.0) - q(1.0)) / (2 * (q(1.0) + q(-1.0) - 2 * q(0.0)))
    assert abs(printed - g3) > 1e-3
    assert ridge.gamma_primal(w0, pr.y, beta0, dw, dbeta, lam, N) == pytest.approx(g3, rel=1e-9)


# ------------------------------------------------------------------ distributed simulator
@pytest.mark.parametrize("form", ["primal", "dual"])
@pytest.mark.parametrize("mode", ["add", "average"])
def test_k1_distributed_equals_sequential(form, mode):
    """K = 1 with γ = 1 (= 1/K) reproduces the local solver exactly."""
    pr = _rand_prob(90, 35, 0.3, 71, 0.02)
    x1, s1, h1 = solver.solve(pr, form, 5, seed=7)
    x2, s2, h2 = solver.run_distributed(pr, form, 1, mode, 5, seed=7, seed_part=3)
    # x0 + 1·(x_k - x0) equals x_k up to one rounding per entry
    np.testing.assert_allclose(x2, x1, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(s2, s1, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("form", ["primal", "dual"])
def test_adaptive_never_worse_than_average(form):
    """γ* minimises the round's objective: never worse than γ = 0 or 1/K;
    scalar decomposition over disjoint supports is exercised by the simulator."""
    pr = _rand_prob(200, 80, 0.1, 81, 1e-3)
    A = pr.A()
    K = 4
    owner = oracle.partition(5, pr.M if form == "primal" else pr.N, K)
    x0, s0, _ = solver.run_distributed(pr, form, K, "optimal", 3, seed=1, seed_part=5, record=False)
    # one more round by hand, evaluating the objective at γ = 0, 1/K, γ*
    dx = np.zeros_like(x0)
    ds = np.zeros_like(s0)
    for k in range(K):
        loc = np.nonzero(owner == k)[0]
        xk, sk = x0.copy(), s0.copy()
        order = loc[oracle.permutation(1 + k, 4, len(loc))]
        if form == "primal":
            solver.primal_epoch(pr, xk, sk, order)
        else:
            solver.dual_epoch(pr, xk, sk, order)
        dx += xk - x0
        ds += sk - s0
    if form == "primal":
        f = lambda g: ridge.primal_objective(A, pr.y, pr.lam, x0 + g * dx)
        gs = ridge.gamma_primal(s0, pr.y, x0, ds, dx, pr.lam, pr.N)
        assert f(gs) <= min(f(0.0), f(1.0 / K)) + 1e-14
        # scalar decomposition
        parts = [(x0[owner == k] @ dx[owner == k], dx[owner == k] @ dx[owner == k]) for k in range(K)]
        assert sum(p[0] for p in parts) == pytest.approx(x0 @ dx, rel=1e-12)
        assert sum(p[1] for p in parts) == pytest.approx(dx @ dx, rel=1e-12)
    else:
        f = lambda g: -ridge.dual_objective(A, pr.y, pr.lam, x0 + g * dx)
        gs = ridge.gamma_dual(x0, s0, pr.y, dx, ds, pr.lam, pr.N)
        assert f(gs) <= min(f(0.0), f(1.0 / K)) + 1e-14


@pytest.mark.slow
def test_distributed_threads_do_not_change_the_result():
    pr = _rand_prob(120, 60, 0.2, 77, 0.01)
    for form in ("primal", "dual"):
        a = solver.run_distributed(pr, form, 4, "optimal", 3, seed=1, seed_part=2)
        b = solver.run_distributed(pr, form, 4, "optimal", 3, seed=1, seed_part=2, threads=4)
        assert np.array_equal(a[0], b[0]) and [h["gamma"] for h in a[2]] == [h["gamma"] for h in b[2]]


def test_distributed_slowdown_shape():
    """Fig. 3 shape ("approximately linear slow-down"): with averaging, epochs to a
    fixed gap are nondecreasing in K; adaptive aggregation (Alg. 4) at K = 8 needs fewer epochs
    than averaging.  Desk-scale analogue of SPEC acceptance 7."""
    d = synth.gen_host(synth.ZipfRowsCfg("dist", 4000, 1000, 1000, 1.0, 40.0, 0.5, 4, 200, seed=17))
    pr = solver.Problem.from_csr(d)
    pr.lam = 1e-3
    target = 1e-4 * ridge.primal_objective(pr.A(), pr.y, pr.lam, np.zeros(pr.M))

    def epochs_to(K, mode, rounds=300):
        _, _, h = solver.run_distributed(pr, "primal", K, mode, rounds, seed=3, seed_part=9)
        for i, r in enumerate(h):
            if r["gap"] <= target:
                return i + 1
        return rounds + 1

    e = [epochs_to(K, "average") for K in (1, 2, 4, 8)]
    assert all(e[i] <= e[i + 1] for i in range(3)), e
    assert epochs_to(8, "optimal") < e[3]


# ------------------------------------------------------------------ integer artefacts (invariants)
@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 64, 100, 1023, 1024, 1025, 65537])
def test_permutation_is_bijection(n):
    for t in (0, 1, 7):
        p = oracle.permutation(12345, t, n)
        assert np.array_equal(np.sort(p), np.arange(n))


@pytest.mark.parametrize("n,blk", [(0, 32), (1, 32), (31, 32), (32, 32), (1000, 32), (1003, 8), (5000, 1), (777, 777)])
def test_block_order_is_a_bijection_of_whole_blocks(n, blk):
    """Reading c28: the full blocks of blk consecutive coordinates are visited whole, in the order of
    the permutation over the blocks; the partial block last; blk = 1 is the plain permutation."""
    o = oracle.block_order(5, 3, n, blk, stream=1)
    assert np.array_equal(np.sort(o), np.arange(n))
    nf = n // blk
    if blk == 1:
        assert np.array_equal(o, oracle.permutation(5, 3, n, stream=1))
    for b in range(nf):
        blkv = o[b * blk:(b + 1) * blk]
        assert blkv[0] % blk == 0 and np.array_equal(blkv, blkv[0] + np.arange(blk))
    if nf > 1:
        assert np.array_equal(o[:nf * blk:blk] // blk, oracle.permutation(5, 3, nf, stream=1))
    assert np.array_equal(o[nf * blk:], np.arange(nf * blk, n))


@pytest.mark.parametrize("k", [1, 2, 3, 8])
def test_partition_balanced_invariants(k):
    """Reading c29: every coordinate gets one owner; counts differ by at most one; each worker's stored
    entries are within one longest coordinate of every other's (snake dealing of decreasing lengths)."""
    rng = np.random.default_rng(k)
    lens = np.concatenate([rng.zipf(1.6, 3000).clip(1, 5000), np.zeros(57, np.int64)])
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    own = oracle.partition_balanced(ptr, 11, k)
    assert own.min() >= 0 and own.max() < k
    cnt = np.bincount(own, minlength=k)
    assert cnt.max() - cnt.min() <= 1
    load = np.bincount(own, weights=lens, minlength=k)
    assert load.max() - load.min() <= lens.max()


def test_partition_balanced_hand_example():
    """Lengths 5,1,4,2,3,0 over k = 2: sorted 5,4,3,2,1,0 (coordinates 0,2,4,3,1,5) dealt 0,1,1,0,0,1."""
    ptr = np.concatenate([[0], np.cumsum([5, 1, 4, 2, 3, 0])]).astype(np.int64)
    assert oracle.partition_balanced(ptr, 3, 2).tolist() == [0, 0, 1, 0, 1, 1]


def test_permutation_depends_on_epoch_and_is_mixing():
    n = 4096
    ps = [oracle.permutation(99, t, n) for t in range(1, 41)]
    assert all(not np.array_equal(ps[0], q) for q in ps[1:])
    # position of element 0 roughly uniform; fixed points ~ Poisson(1)
    fixed = np.mean([np.sum(q == np.arange(n)) for q in ps])
    assert 0.2 < fixed < 3.0
    pos = np.array([np.nonzero(q == 0)[0][0] for q in ps])
    assert pos.std() > n / 8


@pytest.mark.parametrize("count,k,sizes", [(5, 2, [3, 2]), (4, 1, [4]), (8, 8, [1] * 8), (0, 3, [0, 0, 0]),
                                           (1000, 7, None)])
def test_partition_invariants(count, k, sizes):
    """Disjoint, complete, sizes differ by at most one."""
    own = oracle.partition(3, count, k)
    cnt = np.bincount(own, minlength=k) if count else np.zeros(k, int)
    assert cnt.sum() == count and cnt.max() - cnt.min() <= 1
    if sizes is not None:
        assert sorted(cnt.tolist(), reverse=True) == sorted(sizes, reverse=True)


def test_transpose_examples_and_involution():
    # CSR [[1,0],[0,2]] -> CSC col0={(0,1)}, col1={(1,2)}
    p, i, v = oracle.transpose([0, 1, 2], [0, 1], [1.0, 2.0], 2)
    assert p.tolist() == [0, 1, 2] and i.tolist() == [0, 1] and v.tolist() == [1.0, 2.0]
    # CSR [[0,3]] -> col0 empty, col1 = {(0,3)}
    p, i, v = oracle.transpose([0, 1], [1], [3.0], 2)
    assert p.tolist() == [0, 0, 1] and i.tolist() == [0] and v.tolist() == [3.0]
    d = synth.random_sparse(37, 23, 0.2, 5, empty_rows=3, empty_cols=2)
    p, i, v = oracle.transpose(d["ptr"], d["idx"], d["val"], 23)
    for c in range(23):
        assert np.all(np.diff(i[p[c]:p[c + 1]]) > 0)
    p2, i2, v2 = oracle.transpose(p, i, v, 37)
    assert np.array_equal(p2, d["ptr"]) and np.array_equal(i2, d["idx"]) and np.array_equal(v2, d["val"])
    # squared norms: cols of CSC == rows of CSR of the transpose
    dense = sp.csr_matrix((d["val"].astype(np.float64), d["idx"], d["ptr"]), shape=(37, 23)).toarray()
    np.testing.assert_allclose(oracle.sq_norms(p, v), (dense ** 2).sum(0), rtol=1e-15)
    np.testing.assert_allclose(oracle.sq_norms(d["ptr"], d["val"]), (dense ** 2).sum(1), rtol=1e-15)
    # [[1,0],[0,2]] cols -> (1, 4); [[1,2],[3,4]] rows -> (5, 25)
    assert oracle.sq_norms([0, 1, 2], [1.0, 2.0]).tolist() == [1.0, 4.0]
    assert oracle.sq_norms([0, 2, 4], [1.0, 2.0, 3.0, 4.0]).tolist() == [5.0, 25.0]


def test_sub_epoch_rounds_cover_each_coordinate_once_and_converge_faster():
    """Sub-epoch aggregation: with K = 1 and γ = 1 the parts of an epoch compose to the
    whole epoch exactly; with K = 8 more frequent rounds need no more epochs than one round per epoch."""
    pr = _rand_prob(300, 120, 0.1, 91, 1e-3)
    x1, s1, _ = solver.run_distributed(pr, "primal", 1, "add", 3, seed=4, seed_part=1)
    x4, s4, _ = solver.run_distributed(pr, "primal", 1, "add", 12, seed=4, seed_part=1, parts=4)
    np.testing.assert_allclose(x4, x1, rtol=1e-12, atol=1e-15)
    _, _, h1 = solver.run_distributed(pr, "primal", 8, "average", 10, seed=4, seed_part=1)
    _, _, h4 = solver.run_distributed(pr, "primal", 8, "average", 40, seed=4, seed_part=1, parts=4)
    assert h4[-1]["gap"] <= h1[-1]["gap"]
