"""Ridge-regression objectives, Fenchel maps, duality gaps, closed form and aggregation γ
(TEST INFRASTRUCTURE ONLY; fp64 numpy/scipy; see oracle/__init__.py).

Citations: P:n = PAPER.md line n.  Each function is the paper's definition written out.
A is a scipy.sparse matrix (N x M) of the fp32 data promoted to fp64.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def as_matrix(ptr, idx, val, n_rows: int, n_cols: int, layout: str = "csr") -> sp.spmatrix:
    """fp64 scipy matrix of the stored fp32 data (layout 'csr': outer = rows, 'csc': outer = cols)."""
    data = np.asarray(val, np.float32).astype(np.float64)
    if layout == "csr":
        return sp.csr_matrix((data, np.asarray(idx), np.asarray(ptr)), shape=(n_rows, n_cols))
    return sp.csc_matrix((data, np.asarray(idx), np.asarray(ptr)), shape=(n_rows, n_cols))


def primal_objective(A, y, lam, beta) -> float:
    """Eq. (1):  P(β) = 1/(2N) ||Aβ - y||² + λ/2 ||β||²."""
    N = A.shape[0]
    r = A @ beta - y
    return float(r @ r / (2.0 * N) + 0.5 * lam * (beta @ beta))


def primal_objective_at(y, lam, beta, w) -> float:
    """Line-search objective of §IV.B: P(β, w) = 1/(2N)||w - y||² + λ/2||β||² with w trusted as Aβ."""
    N = len(y)
    r = w - y
    return float(r @ r / (2.0 * N) + 0.5 * lam * (beta @ beta))


def dual_objective(A, y, lam, alpha) -> float:
    """Eq. (3):  D(α) = -N/2 ||α||² - 1/(2λ) ||Aᵀα||² + αᵀy."""
    N = A.shape[0]
    v = A.T @ alpha
    return float(-0.5 * N * (alpha @ alpha) - (v @ v) / (2.0 * lam) + alpha @ y)


def dual_objective_at(y, lam, alpha, wbar) -> float:
    """D(α) with w̄ trusted as Aᵀα (dual line search)."""
    N = len(y)
    return float(-0.5 * N * (alpha @ alpha) - (wbar @ wbar) / (2.0 * lam) + alpha @ y)


def primal_grad(A, y, lam, beta) -> np.ndarray:
    """∂P/∂β = (1/N) Aᵀ(Aβ - y) + λβ."""
    N = A.shape[0]
    return (A.T @ (A @ beta - y)) / N + lam * beta


def dual_grad(A, y, lam, alpha) -> np.ndarray:
    """∂D/∂α = -Nα - (1/λ) A Aᵀα + y."""
    N = A.shape[0]
    return -N * alpha - (A @ (A.T @ alpha)) / lam + y


def dual_to_primal(A, lam, alpha) -> np.ndarray:
    """Eq. (5):  β = (1/λ) Aᵀα."""
    return (A.T @ alpha) / lam


def primal_to_dual(A, y, beta) -> np.ndarray:
    """Eq. (6):  α = (1/N)(y - Aβ)."""
    return (y - A @ beta) / A.shape[0]


def gap_primal(A, y, lam, beta) -> float:
    """G_P(β) = |P(β) - D((y - Aβ)/N)|   (§II.C)."""
    return abs(primal_objective(A, y, lam, beta) - dual_objective(A, y, lam, primal_to_dual(A, y, beta)))


def gap_dual(A, y, lam, alpha) -> float:
    """G_D(α) = |P(Aᵀα/λ) - D(α)|   (§II.C)."""
    return abs(primal_objective(A, y, lam, dual_to_primal(A, lam, alpha)) - dual_objective(A, y, lam, alpha))


def gap_primal_gradform(A, y, lam, beta) -> float:
    """G_P(β) = ||∇P(β)||² / (2λ) — algebraically identical to gap_primal (DESIGN.md c13);
    no cancellation, so it is the form the GPU evaluates.  Pinned equal to gap_primal."""
    g = primal_grad(A, y, lam, beta)
    return float(g @ g / (2.0 * lam))


def gap_dual_gradform(A, y, lam, alpha) -> float:
    """G_D(α) = ||∇D(α)||² / (2N) — identical to gap_dual (DESIGN.md c13)."""
    g = dual_grad(A, y, lam, alpha)
    return float(g @ g / (2.0 * A.shape[0]))


def dual_report(A, y, lam, alpha) -> tuple[float, float, float]:
    """(P(Aᵀα/λ), D(α), G_D(α)) with the two sparse products shared (large problems):
    v = Aᵀα, q = Av;  P = ||q/λ - y||²/(2N) + ||v||²/(2λ)  (Eq. 1 at β = v/λ, Eq. 5),
    D = -N/2||α||² - ||v||²/(2λ) + αᵀy  (Eq. 3),  G_D = ||y - Nα - q/λ||²/(2N)  (c13).
    Pinned equal to primal_objective / dual_objective / gap_dual_gradform."""
    N = A.shape[0]
    v = A.T @ alpha
    q = A @ v
    vv = float(v @ v)
    r = q / lam - y
    g = y - N * alpha - q / lam
    return (float(r @ r) / (2.0 * N) + vv / (2.0 * lam), float(-0.5 * N * (alpha @ alpha) - vv / (2.0 * lam) + alpha @ y),
            float(g @ g) / (2.0 * N))


def primal_report(A, y, lam, beta) -> tuple[float, float, float]:
    """(P(β), D((y - Aβ)/N), G_P(β)) with the two sparse products shared:
    res = y - Aβ, g = Aᵀres;  P = ||res||²/(2N) + λ/2||β||²  (Eq. 1),
    D(α̂ = res/N) = -||res||²/(2N) - ||g||²/(2λN²) + yᵀres/N  (Eq. 3, Eq. 6),
    G_P = ||λβ - g/N||²/(2λ)  (c13).  Pinned equal to the separate functions."""
    N = A.shape[0]
    res = y - A @ beta
    g = A.T @ res
    rr = float(res @ res)
    gr = lam * beta - g / N
    return (rr / (2.0 * N) + 0.5 * lam * float(beta @ beta),
            -rr / (2.0 * N) - float(g @ g) / (2.0 * lam * N * N) + float(y @ res) / N, float(gr @ gr) / (2.0 * lam))


def closed_form(A, y, lam, cap: int = 4096) -> np.ndarray:
    """β* = argmin P = (AᵀA + λN I)⁻¹ Aᵀy  (zero of the gradient P:83; dense solve, M <= cap)."""
    N, M = A.shape
    if M > cap:
        raise ValueError(f"closed form refused: M={M} > cap={cap}")
    Ad = A.toarray() if sp.issparse(A) else np.asarray(A)
    H = Ad.T @ Ad + lam * N * np.eye(M)
    return np.linalg.solve(H, Ad.T @ y)


def closed_form_dual(A, y, lam, cap: int = 4096) -> np.ndarray:
    """α* = argmax D = λ (λN I + AAᵀ)⁻¹ y  (zero of the dual gradient P:109; N <= cap)."""
    N, M = A.shape
    if N > cap:
        raise ValueError(f"closed form refused: N={N} > cap={cap}")
    Ad = A.toarray() if sp.issparse(A) else np.asarray(A)
    return np.linalg.solve(lam * N * np.eye(N) + Ad @ Ad.T, lam * y)


def gamma_primal(w, y, beta, dw, dbeta, lam, N) -> float:
    """Optimal aggregation γ* = argmin_γ P(β + γΔβ, w + γΔw)  (§IV.B, Eq. 7).

    Eq. (7) is printed with <w, Δw>; the derivative of the stated line search gives
    <w - y, Δw> (DESIGN.md c3), and β is the round's base point (c5):
        γ* = -(<w - y, Δw> + Nλ<β, Δβ>) / (||Δw||² + Nλ||Δβ||²);   zero update -> 0 (c16).
    """
    den = float(dw @ dw + N * lam * (dbeta @ dbeta))
    if den == 0.0:
        return 0.0
    return -float((w - y) @ dw + N * lam * (beta @ dbeta)) / den


def gamma_dual(alpha, wbar, y, dalpha, dwbar, lam, N) -> float:
    """Optimal dual aggregation γ̄* = argmax_γ D(α + γΔα)  (§IV.B).

    The printed denominator has N||α||²; the derivative gives N||Δα||² (DESIGN.md c4):
        γ̄* = (<Δα, y> - N<Δα, α> - (1/λ)<Δw̄, w̄>) / ((1/λ)||Δw̄||² + N||Δα||²).
    """
    den = float(dwbar @ dwbar / lam + N * (dalpha @ dalpha))
    if den == 0.0:
        return 0.0
    return float(dalpha @ y - N * (dalpha @ alpha) - (dwbar @ wbar) / lam) / den
