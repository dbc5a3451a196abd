"""Logical-K workers on one device: the group evaluation (scd_evaluate_group) of the global model
against the oracle (GPU)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import ridge, solver

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1702_07005_b200 as scd  # noqa: E402
from test_gpu_parity import _shards  # noqa: E402


@pytest.mark.parametrize("form", ["primal", "dual"])
def test_evaluate_group_matches_oracle(form):
    d = synth.gen_host(synth.CONFIGS["C2"].with_rows(1500))
    pr = solver.Problem.from_csr(d)
    A = pr.A()
    K, seed, sp_ = 3, 5, 7
    solvers = [scd.Solver(p, i, v, nr, nc, y, pr.lam, form, seed=seed + k, n_global=pr.N)
               for k, (p, i, v, nr, nc, y) in enumerate(_shards(d, pr, form, K, sp_))]
    for t in (1, 2):
        for s in solvers:
            s.epoch(t)
        scd.aggregate_group(solvers, "optimal")
    P, D, g = scd.evaluate_group(solvers)
    owner = oracle.partition(sp_, pr.M if form == "primal" else pr.N, K)
    x = np.zeros(len(owner))
    for k, s in enumerate(solvers):
        x[owner == k] = s.get_model()
    if form == "primal":
        Po, go = ridge.primal_objective(A, pr.y, pr.lam, x), ridge.gap_primal_gradform(A, pr.y, pr.lam, x)
        Do = ridge.dual_objective(A, pr.y, pr.lam, ridge.primal_to_dual(A, pr.y, x))
    else:
        Po = ridge.primal_objective(A, pr.y, pr.lam, ridge.dual_to_primal(A, pr.lam, x))
        Do, go = ridge.dual_objective(A, pr.y, pr.lam, x), ridge.gap_dual_gradform(A, pr.y, pr.lam, x)
    assert P == pytest.approx(Po, rel=1e-9)
    assert D == pytest.approx(Do, rel=1e-9)
    assert g == pytest.approx(go, rel=1e-7)
