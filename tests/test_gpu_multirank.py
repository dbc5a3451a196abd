"""GPU: the library's world = 2 path (scd_aggregate / scd_duality_gap / scd_objective / the shared-vector
rebuild over a communicator) with two processes, against the oracle's Alg. 3/4 simulator (P:269-371,
readings c3-c6, c14).

Two transports:
  * hooks (always, ONE GPU): both ranks on cuda:0, the library's collectives going through the
    scd_collectives host hooks (tests/hostcoll.py, torch.distributed gloo) — NCCL refuses two ranks
    on one device.  This runs every line of the library's multi-rank logic except the NCCL calls:
    the sharded active-extent exchange, Δ / scalar all-reduces, γ, the fused peer-memory exchange
    (SCD_P2P_AGG=1: CUDA IPC handles all-gathered, shards reduced from the peer's memory and
    written back into it, the three scalar barriers), the collective gap, recompute_every.
  * nccl (needs 2 GPUs, skipped otherwise): one rank per device over an NCCL communicator.
Each worker runs its local epochs in deterministic mode (exact P_t order over its coordinates), so
the rounds must reproduce the simulator's γ and models (fp32 vs fp64: 1e-4)."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
K, SEED, SEED_PART, ROUNDS = 2, 10, 3, 3
MODES = ("average", "optimal", "add")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(kind):
    import synth
    from oracle import solver

    if kind == "c2":
        d = synth.gen_host(synth.CONFIGS["C2"].with_rows(1500))
    else:  # small random problem with empty trailing columns (dual active extent) and empty rows
        d = synth.random_sparse(300, 500, 0.05, 7, empty_rows=6, empty_cols=120)
    return d, solver.Problem.from_csr(d)


def _shard(d, pr, form, rank):
    import oracle

    owner = oracle.partition(SEED_PART, pr.M if form == "primal" else pr.N, K)
    loc = np.nonzero(owner == rank)[0]
    if form == "primal":
        p = np.concatenate([[0], np.cumsum(np.diff(pr.cptr)[loc])]).astype(np.int64)
        sel = np.concatenate([np.arange(pr.cptr[c], pr.cptr[c + 1]) for c in loc]).astype(np.int64)
        return p, pr.cidx[sel], pr.cval[sel], pr.N, len(loc), d["y"], owner
    p = np.concatenate([[0], np.cumsum(np.diff(pr.rptr)[loc])]).astype(np.int64)
    sel = np.concatenate([np.arange(pr.rptr[r], pr.rptr[r + 1]) for r in loc]).astype(np.int64)
    return p, pr.ridx[sel], pr.rval[sel], len(loc), pr.M, d["y"][loc], owner


def _worker(rank, port, transport, form, kind, q):
    sys.path[:0] = [ROOT, HERE]
    res = {}
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist

        dev = rank if transport == "nccl" else 0
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", rank=rank, world_size=K)
        import paper_1702_07005_b200 as scd
        from hostcoll import HostCollectives

        d, pr = _problem(kind)
        p, i, v, nr, nc, y, owner = _shard(d, pr, form, rank)
        comm, hc = None, None
        if transport == "nccl":
            uid = [scd.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = scd.nccl_comm_init(uid[0], K, rank)
        else:
            hc = HostCollectives()
        runs = [(m, e, 0) for m in MODES for e in ("allreduce", "p2p")] + [("optimal", "allreduce", 1)]
        for mode, exch, rec in runs:
            os.environ["SCD_P2P_AGG"] = "1" if exch == "p2p" else "0"
            s = scd.Solver(p, i, v, nr, nc, y, pr.lam, form, seed=SEED + rank, deterministic=True, n_global=pr.N,
                           rank=rank, world=K, nccl_comm=comm, collectives=None if hc is None else hc.struct,
                           recompute_every=rec)
            gam, gaps = [], []
            rounds = ROUNDS if mode != "add" else 2
            for t in range(1, rounds + 1):
                s.epoch(t)
                gam.append(s.aggregate(mode))
                gaps.append(s.duality_gap())
            P, D = s.objective()
            res[(mode, exch, rec)] = dict(gamma=gam, gaps=gaps, P=P, D=D, x=s.get_model(), sv=s.get_shared(),
                                          info=s.info())
            s.close()
        if kind == "empty" and form == "dual":
            # asynchronous epochs: after rounds with γ != 1 the next epoch must put every empty row back
            # on its fixed point α_n = y_n / N (c17), as the simulator's sequential epochs do
            os.environ["SCD_P2P_AGG"] = "0"
            s = scd.Solver(p, i, v, nr, nc, y, pr.lam, form, seed=SEED + rank, n_global=pr.N, rank=rank, world=K,
                           nccl_comm=comm, collectives=None if hc is None else hc.struct)
            for t in range(1, ROUNDS + 1):
                s.epoch(t)
                s.aggregate("average")
            s.epoch(ROUNDS + 1)
            res["async_empty"] = dict(x=s.get_model(), y=np.asarray(y, np.float64), empty=np.diff(p) == 0, N=pr.N)
            s.close()
        if hc is not None:
            res["calls"] = dict(hc.calls)
            res["errors"] = hc.errors
        if comm:
            scd.nccl_comm_destroy(comm)
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback

        res["exception"] = traceback.format_exc()
    q.put((rank, res))


def _spawn(transport, form, kind):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, port, transport, form, kind, q)) for r in range(K)]
    for p in ps:
        p.start()
    out = {}
    for _ in ps:
        r, res = q.get(timeout=600)
        out[r] = res
    for p in ps:
        p.join(timeout=60)
    for r in range(K):
        assert "exception" not in out[r], out[r]["exception"]
    return out


def _check(out, form, kind):
    import oracle
    from oracle import ridge, solver

    d, pr = _problem(kind)
    A = pr.A()
    owner = oracle.partition(SEED_PART, pr.M if form == "primal" else pr.N, K)
    for key in out[0]:
        if not isinstance(key, tuple):
            continue
        mode, exch, rec = key
        r0, r1 = out[0][key], out[1][key]
        rounds = len(r0["gamma"])
        xo, so, hist = solver.run_distributed(pr, form, K, mode, rounds, seed=SEED, seed_part=SEED_PART)
        for t in range(rounds):
            # every rank derives the same γ, and it is the simulator's (Eq. 7 / γ̄ corrected)
            assert r0["gamma"][t] == r1["gamma"][t], (key, t)
            assert r0["gamma"][t] == pytest.approx(hist[t]["gamma"], rel=1e-4, abs=1e-7), (key, t, r0["gamma"], hist)
            # the collective gap (from scratch, fp64, all-reduced) equals the oracle's on the same model
            assert r0["gaps"][t] == r1["gaps"][t]
        x = np.zeros(len(owner))
        x[owner == 0] = r0["x"]
        x[owner == 1] = r1["x"]
        scale = np.abs(xo).max()
        assert np.abs(x - xo).max() <= 1e-4 * scale, (key, np.abs(x - xo).max() / scale)
        for sv in (r0["sv"], r1["sv"]):  # the shared vector is replicated and equals the simulator's
            assert np.abs(sv - so).max() <= 1e-4 * np.abs(so).max(), key
        gap = ridge.dual_report(A, pr.y, pr.lam, x)[2] if form == "dual" else ridge.primal_report(A, pr.y, pr.lam, x)[2]
        if mode != "add":
            assert r0["gaps"][-1] == pytest.approx(gap, rel=1e-5, abs=1e-12), (key, r0["gaps"][-1], gap)
        if rec:  # recompute_every = 1: the shared vector was rebuilt from the aggregated model in fp64
            u = A @ x if form == "primal" else A.T @ x
            assert np.abs(r0["sv"] - u).max() <= 2e-7 * max(1.0, np.abs(u).max()), key


@pytest.mark.parametrize("form", ["dual", "primal"])
def test_world2_hooks_one_gpu(form):
    out = _spawn("hooks", form, "c2")
    _check(out, form, "c2")
    c = out[0]["calls"]
    assert c["allreduce"] > 0 and c["allgather"] > 0, c  # the P2P runs all-gathered their IPC handles
    assert not out[0]["errors"] and not out[1]["errors"]


def test_world2_hooks_dual_active_extent_and_empty_rows():
    """Dual shards whose last 120 columns are empty on every rank (the exchange covers only the
    max-over-ranks active extent) and empty rows (α_n = y_n/N after every round, also after γ != 1)."""
    out = _spawn("hooks", "dual", "empty")
    _check(out, "dual", "empty")
    for r in range(K):
        a = out[r]["async_empty"]
        assert a["empty"].any()
        np.testing.assert_allclose(a["x"][a["empty"]], a["y"][a["empty"]] / a["N"], rtol=1e-6)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="NCCL needs one GPU per rank (2 devices)")
@pytest.mark.parametrize("form", ["dual", "primal"])
def test_world2_nccl_two_gpus(form):
    out = _spawn("nccl", form, "c2")
    _check(out, form, "c2")


def test_dual_world2_needs_global_n():
    import paper_1702_07005_b200 as scd
    from paper_1702_07005_b200.scd import ScdError

    sys.path.insert(0, HERE)
    from hostcoll import HostCollectives

    hc = HostCollectives()
    ptr = np.array([0, 1, 2], np.int64)
    with pytest.raises(ScdError) as e:
        scd.Solver(ptr, np.array([0, 1], np.int32), np.ones(2, np.float32), 2, 2, np.ones(2, np.float32), 1.0, "dual",
                   rank=0, world=2, collectives=hc.struct)
    assert e.value.status == 1 and "n_global" in str(e.value)
    assert hc.calls == {"allreduce": 0, "allgather": 0}
