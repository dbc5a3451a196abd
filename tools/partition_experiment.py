"""Oracle experiment (reading c29): Alg. 4 (optimal gamma, K = 8) on a criteo-shaped dual problem
(100 000 rows, field cardinalities scaled by 0.002, lambda N = 2e5) with the rows partitioned at random
(reading c15) or grouped by the value of one one-hot field before dealing contiguous blocks.
Runs on the CPU:  python tools/partition_experiment.py"""
import sys, numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import synth, oracle
from oracle import solver, ridge
cfg = synth.c5_scaled(100_000, 0.002)
d = synth.gen_host(cfg)
pr = solver.Problem.from_csr(d, lam=2.0, csc=False)
A = pr.A()
K = 8
N = pr.N
# field-grouped: key = value of the smallest categorical field (card ~10 after scaling?)
off = cfg.offsets; card = np.asarray(cfg.cards)
print("cards", card[:13].tolist()[:3], sorted(card[13:].tolist())[:8])
def run(owner, rounds=20, label=""):
    local = [np.nonzero(owner == k)[0] for k in range(K)]
    x0 = np.zeros(N); s0 = np.zeros(pr.M); nrm = pr.row_norms()
    gaps = []
    for t in range(1, rounds + 1):
        dx = np.zeros(N); ds = np.zeros(pr.M)
        for k in range(K):
            xk, sk = x0.copy(), s0.copy()
            order = local[k][oracle.permutation(10 + k, t, len(local[k]))]
            solver.dual_epoch(pr, xk, sk, order, nrm, n_global=N)
            dx += xk - x0; ds += sk - s0
        g = ridge.gamma_dual(x0, s0, pr.y, dx, ds, pr.lam, N)
        x0 = x0 + g * dx; s0 = s0 + g * ds
        gaps.append(ridge.dual_report(A, pr.y, pr.lam, x0)[2])
    print(label, " ".join("%.1e" % x for x in gaps), flush=True)
rand = oracle.partition(5, N, K)
run(rand, label="random      ")
# group rows by value of field f: sort by key, deal contiguous blocks
rows_field = lambda f: d["idx"].reshape(N, 39)[:, f]
for f in (13 + int(np.argmin(card[13:])), 0):
    key = rows_field(f)
    order = np.lexsort((rand, key))
    owner = np.empty(N, np.int32); owner[order] = (np.arange(N) * K) // N
    run(owner, label=f"field {f:2d} (card {card[f]})")
# two smallest fields combined
fs = 13 + np.argsort(card[13:])[:2]
key = rows_field(fs[0]) * 100000 + rows_field(fs[1])
order = np.lexsort((rand, key)); owner = np.empty(N, np.int32); owner[order] = (np.arange(N) * K) // N
run(owner, label="fields 2 smallest")
