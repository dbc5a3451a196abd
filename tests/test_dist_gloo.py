"""World-size-2 multi-process test (CPU, gloo) of the distributed protocol the library runs over
NCCL in scd_aggregate: each rank runs its local epoch on its shard, then ONE all-reduce of the
shared-vector delta and of the per-worker scalars <x0_k, Δx_k>, ||Δx_k||², <y_k, Δx_k>, while
<sv0, Δ> and ||Δ||² are computed locally on the replicated vectors; every rank derives the same γ
(Alg. 3/4; readings c3-c6).  The two processes must reproduce the in-process Alg. 3/4
simulator of the oracle.  Also checks the NCCL-id bootstrap the bench uses (broadcast of the
128-byte ncclUniqueId through torch.distributed)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, form, mode, out, protocol="allreduce"):
    import torch
    import torch.distributed as dist

    import oracle
    import synth
    from oracle import ridge, solver

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = synth.gen_host(synth.CONFIGS["C2"].with_rows(800))
        pr = solver.Problem.from_csr(d)
        K, seed, seed_part, rounds = world, 10, 3, 4
        n_coord = pr.M if form == "primal" else pr.N
        owner = oracle.partition(seed_part, n_coord, K)
        loc = np.nonzero(owner == rank)[0]
        x0 = np.zeros(n_coord)
        s0 = np.zeros(pr.N if form == "primal" else pr.M)
        nrm = pr.col_norms() if form == "primal" else pr.row_norms()
        gammas = []
        for t in range(1, rounds + 1):
            xk, sk = x0.copy(), s0.copy()
            order = loc[oracle.permutation(seed + rank, t, len(loc))]
            if form == "primal":
                solver.primal_epoch(pr, xk, sk, order, nrm)
            else:
                solver.dual_epoch(pr, xk, sk, order, nrm, n_global=pr.N)
            dx = (xk - x0)[loc]
            yk = pr.y[loc] if form == "dual" else np.zeros(len(loc))
            scal = torch.tensor([x0[loc] @ dx, dx @ dx, yk @ dx], dtype=torch.float64)
            if protocol == "allreduce":  # NCCL path of scd_aggregate
                delta = torch.from_numpy(sk - s0)
                dist.all_reduce(delta)  # Σ_k Δsv_k
                dist.all_reduce(scal)   # Σ_k scalars (disjoint supports)
                delta = delta.numpy()
                a_sd, a_dd = s0 @ delta, delta @ delta  # replicated vectors: not reduced
            else:  # fused peer-memory path (aggregate.cu k_agg_reduce / k_agg_apply): own shard only
                n = len(s0)
                lo, hi = n * rank // K, n * (rank + 1) // K
                peers = [torch.zeros(n, dtype=torch.float64) for _ in range(K)]
                dist.all_gather(peers, torch.from_numpy(sk))  # the peer reads of every rank's sv
                d_sh = sum(p.numpy()[lo:hi] - s0[lo:hi] for p in peers)
                scal = torch.cat([scal, torch.tensor([s0[lo:hi] @ d_sh, d_sh @ d_sh], dtype=torch.float64)])
                dist.all_reduce(scal)  # model scalars + shard dots: the second barrier
                a_sd, a_dd = float(scal[3]), float(scal[4])
                shards = [torch.zeros(n * (k + 1) // K - n * k // K, dtype=torch.float64) for k in range(K)]
                dist.all_gather(shards, torch.from_numpy(d_sh))  # k_agg_apply's stores of every shard
                delta = torch.cat(shards).numpy()
            lamN = pr.lam * pr.N
            if mode == "average":
                g = 1.0 / K
            elif form == "primal":  # the oracle keeps w (not r): <w0 - y, Δw>
                den = a_dd + lamN * float(scal[1])
                g = -((s0 - pr.y) @ delta + lamN * float(scal[0])) / den if den else 0.0
            else:
                den = a_dd / pr.lam + pr.N * float(scal[1])
                g = (float(scal[2]) - pr.N * float(scal[0]) - a_sd / pr.lam) / den if den else 0.0
            gammas.append(g)
            s0 = s0 + g * delta
            x0[loc] = x0[loc] + g * dx
        full = torch.from_numpy(np.where(owner == rank, x0, 0.0))
        dist.all_reduce(full)
        if rank == 0:
            xr, sr, hist = solver.run_distributed(pr, form, K, mode, rounds, seed=seed, seed_part=seed_part)
            out.put(("ok", float(np.abs(full.numpy() - xr).max() / max(np.abs(xr).max(), 1e-300)),
                     float(np.abs(s0 - sr).max() / max(np.abs(sr).max(), 1e-300)),
                     [abs(a - h["gamma"]) for a, h in zip(gammas, hist)]))
        # NCCL bootstrap as in bench.py: rank 0 makes the id, everybody receives the same bytes
        try:
            import paper_1702_07005_b200 as scd

            uid = scd.nccl_unique_id() if rank == 0 else bytes(128)
        except Exception:
            uid = bytes([7] * 128) if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8)
        dist.broadcast(t, 0)
        got = bytes(t.tolist())
        ref = [None]
        if rank == 0:
            ref = [uid]
        dist.broadcast_object_list(ref, 0)
        if rank == 1:
            out.put(("uid", got == ref[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("protocol", ["allreduce", "sharded"])
@pytest.mark.parametrize("form", ["dual", "primal"])
@pytest.mark.parametrize("mode", ["optimal", "average"])
def test_two_process_aggregation_matches_simulator(form, mode, protocol):
    """Both exchange protocols of scd_aggregate (NCCL all-reduce; fused sharded peer exchange)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, form, mode, q, protocol)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ok = [r for r in res if r[0] == "ok"][0]
    uid = [r for r in res if r[0] == "uid"][0]
    assert ok[1] <= 1e-12 and ok[2] <= 1e-12, ok
    assert max(ok[3]) <= 1e-12, ok
    assert uid[1]
