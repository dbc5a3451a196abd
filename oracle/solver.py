"""Sequential SCD / SDCA (Alg. 1) and the distributed Alg. 3/4 simulator
(TEST INFRASTRUCTURE ONLY; fp64; see oracle/__init__.py).  P:n = PAPER.md line n.

The epochs themselves run in oracle.c (orc_primal_epoch / orc_dual_epoch), written out
from Alg. 1 with the update rules Eq. (2) and Eq. (4).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import ridge
from ._lib import lib, p, permutation, partition, sq_norms, transpose


@dataclass
class Problem:
    """Ridge problem (A, y, λ) of §II.  A held as both CSR and CSC (fp32 values as
    stored; promoted to fp64 in every computation), y promoted to fp64."""
    n_rows: int
    n_cols: int
    rptr: np.ndarray
    ridx: np.ndarray
    rval: np.ndarray
    y: np.ndarray
    lam: float
    cptr: np.ndarray = field(default=None)
    cidx: np.ndarray = field(default=None)
    cval: np.ndarray = field(default=None)

    @staticmethod
    def from_csr(d: dict, lam: float | None = None, csc: bool = True) -> "Problem":
        """d["val"] = None: implicit values (one-hot data, P:460 footnote) stored explicitly as 1.0.
        csc=False skips the CSC copy (dual-only use: row norms and Eq. (4) epochs need only CSR)."""
        val = d["val"] if d["val"] is not None else np.ones(len(d["idx"]), np.float32)
        pr = Problem(int(d["n_rows"]), int(d["n_cols"]), np.ascontiguousarray(d["ptr"], np.int64),
                     np.ascontiguousarray(d["idx"], np.int32), np.ascontiguousarray(val, np.float32),
                     np.asarray(d["y"], np.float32).astype(np.float64), float(d["lam"] if lam is None else lam))
        if csc:
            pr.cptr, pr.cidx, pr.cval = transpose(pr.rptr, pr.ridx, pr.rval, pr.n_cols)
        return pr

    @property
    def N(self) -> int:
        return self.n_rows

    @property
    def M(self) -> int:
        return self.n_cols

    @property
    def nnz(self) -> int:
        return int(self.rptr[-1])

    def A(self):
        return ridge.as_matrix(self.rptr, self.ridx, self.rval, self.n_rows, self.n_cols, "csr")

    def col_norms(self) -> np.ndarray:
        return sq_norms(self.cptr, self.cval)

    def row_norms(self) -> np.ndarray:
        return sq_norms(self.rptr, self.rval)


def primal_epoch(pr: Problem, beta, w, order, col_norms=None, stat: bool = False, lamN: float | None = None):
    """One pass of Alg. 1 (primal) over ``order`` (global column ids), in place.
    Returns the per-update stationarity ∂P/∂β_m if ``stat``."""
    col_norms = pr.col_norms() if col_norms is None else col_norms
    order = np.ascontiguousarray(order, np.int64)
    st = np.empty(max(len(order), 1)) if stat else None
    lamN = pr.lam * pr.N if lamN is None else lamN
    lib().orc_primal_epoch(pr.N, p(pr.cptr), p(pr.cidx), p(pr.cval), p(pr.y), pr.lam, lamN, p(col_norms), p(beta),
                           p(w), p(order), len(order), p(st))
    return st[: len(order)] if stat else None


def dual_epoch(pr: Problem, alpha, wbar, order, row_norms=None, stat: bool = False, n_global: int | None = None):
    """One pass of Alg. 1 with the dual rule Eq. (4) over ``order`` (global row ids), in place.
    ``n_global`` is the N in λN (global N, DESIGN.md c14)."""
    row_norms = pr.row_norms() if row_norms is None else row_norms
    order = np.ascontiguousarray(order, np.int64)
    st = np.empty(max(len(order), 1)) if stat else None
    lib().orc_dual_epoch(p(pr.rptr), p(pr.ridx), p(pr.rval), p(pr.y), pr.lam, pr.N if n_global is None else n_global,
                         p(row_norms), p(alpha), p(wbar), p(order), len(order), p(st))
    return st[: len(order)] if stat else None


def solve(pr: Problem, form: str, epochs: int, seed: int, first_epoch: int = 1, record=True):
    """Sequential SCD (form='primal') or SDCA (form='dual'), Alg. 1: epoch t visits coordinates
    in the order P_t = permutation(seed, t) (DESIGN.md c8).  Returns (model, shared, history)
    where history[i] = dict(epoch, P, D, gap) evaluated from scratch (DESIGN.md c13)."""
    A = pr.A() if record else None
    hist = []
    if form == "primal":
        x = np.zeros(pr.M)
        s = np.zeros(pr.N)
        nrm = pr.col_norms()
        for t in range(first_epoch, first_epoch + epochs):
            primal_epoch(pr, x, s, permutation(seed, t, pr.M), nrm)
            if record:
                P, D, G = ridge.primal_report(A, pr.y, pr.lam, x)
                hist.append(dict(epoch=t, P=P, D=D, gap=G))
    elif form == "dual":
        x = np.zeros(pr.N)
        s = np.zeros(pr.M)
        nrm = pr.row_norms()
        for t in range(first_epoch, first_epoch + epochs):
            dual_epoch(pr, x, s, permutation(seed, t, pr.N), nrm)
            if record:
                P, D, G = ridge.dual_report(A, pr.y, pr.lam, x)
                hist.append(dict(epoch=t, P=P, D=D, gap=G))
    else:
        raise ValueError(form)
    return x, s, hist


def run_distributed(pr: Problem, form: str, K: int, mode: str, rounds: int, seed: int, seed_part: int,
                    first_epoch: int = 1, record: bool = True, parts: int = 1, threads: int = 1):
    """Distributed SCD, Alg. 3 (mode 'average', γ = 1/K) / 'add' (γ = 1) /
    Alg. 4 (mode 'optimal', γ from Eq. 7 corrected), simulated with K logical workers.

    Partition: owner = partition(seed_part, M or N, K) (DESIGN.md c15); worker k's coordinates
    are its owned ids in increasing order, visited each round in the order
    local_ids[permutation(seed + k, t, |local_ids|)].  λN uses the global N (c14).  Every worker
    starts the round from the broadcast shared vector and its base model (c6); the aggregation
    scalars are taken at the base point (c5).
    parts > 1: sub-epoch rounds ("communicate shared vector updates more frequently"):
    round r runs part p = r mod parts of epoch t = first_epoch + r div parts, i.e. the positions
    [len·p/parts, len·(p+1)/parts) of each worker's epoch order, then aggregates.
    threads > 1: the K local epochs of a round run in that many host threads (the epochs are C calls
    that release the GIL; each worker owns its copies, so the result does not depend on it).
    Returns (model, shared, history) with history[i] = dict(epoch, gamma, P, D, gap)."""
    A = pr.A() if record else None
    n_coord = pr.M if form == "primal" else pr.N
    owner = partition(seed_part, n_coord, K)
    local = [np.nonzero(owner == k)[0].astype(np.int64) for k in range(K)]
    N = pr.N
    if form == "primal":
        x0 = np.zeros(pr.M)      # β (global concatenation of the β_k, disjoint supports)
        s0 = np.zeros(pr.N)      # w = Aβ, broadcast each round
        nrm = pr.col_norms()
    else:
        x0 = np.zeros(pr.N)      # α
        s0 = np.zeros(pr.M)      # w̄ = Aᵀα
        nrm = pr.row_norms()
    hist = []
    for r in range(rounds):
        t, p = first_epoch + r // parts, r % parts
        dx = np.zeros_like(x0)
        ds = np.zeros_like(s0)

        def local_epoch(k):
            xk = x0.copy()
            sk = s0.copy()
            nk = len(local[k])
            order = local[k][permutation(seed + k, t, nk)[nk * p // parts: nk * (p + 1) // parts]]
            if form == "primal":
                primal_epoch(pr, xk, sk, order, nrm)
            else:
                dual_epoch(pr, xk, sk, order, nrm, n_global=N)
            return xk, sk

        if threads > 1:
            from concurrent.futures import ThreadPoolExecutor

            with ThreadPoolExecutor(max_workers=threads) as ex:
                results = list(ex.map(local_epoch, range(K)))
        else:
            results = [local_epoch(k) for k in range(K)]
        for xk, sk in results:  # summed in worker order whatever the threads
            dx += xk - x0          # Δβ_k / Δα_k live on disjoint supports
            ds += sk - s0          # Σ_k Δw_k  (Alg. 3/4 "Aggregate updates")
        if mode == "add":
            g = 1.0
        elif mode == "average":
            g = 1.0 / K
        elif mode == "optimal":
            if form == "primal":
                g = ridge.gamma_primal(s0, pr.y, x0, ds, dx, pr.lam, N)
            else:
                g = ridge.gamma_dual(x0, s0, pr.y, dx, ds, pr.lam, N)
        else:
            raise ValueError(mode)
        s0 = s0 + g * ds
        x0 = x0 + g * dx
        if record:
            P, D, gap = (ridge.primal_report if form == "primal" else ridge.dual_report)(A, pr.y, pr.lam, x0)
            hist.append(dict(epoch=t, gamma=g, P=P, D=D, gap=gap))
    return x0, s0, hist
