"""Probe: can two ranks share ONE GPU through NCCL (and CUDA IPC)?  If so, the library's world >= 2
path (NCCL all-reduce aggregation, the active-extent exchange, the fused peer-memory exchange) can
be exercised on a 1-GPU box with two processes.

  python tools/probe_multirank.py        # spawns 2 ranks on cuda:0, prints one line per step
"""
import os
import sys
import traceback

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, q):
    out = []
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        torch.cuda.set_device(0)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1702_07005_b200 as scd
        uid = scd.nccl_unique_id() if rank == 0 else None
        lst = [uid]
        dist.broadcast_object_list(lst, src=0)
        try:
            comm = scd.nccl_comm_init(lst[0], world, rank)
            out.append(f"rank{rank}: scd_nccl_comm_init ok")
        except Exception as e:  # noqa: BLE001
            out.append(f"rank{rank}: scd_nccl_comm_init FAILED: {e}")
            q.put(out)
            return
        import numpy as np
        import synth
        d = synth.gen_host(synth.CONFIGS["C2"].with_rows(2000))
        lo, hi = 1000 * rank, 1000 * (rank + 1)
        ptr = d["ptr"][lo:hi + 1] - d["ptr"][lo]
        idx = d["idx"][d["ptr"][lo]:d["ptr"][hi]]
        val = d["val"][d["ptr"][lo]:d["ptr"][hi]]
        s = scd.Solver(ptr, idx, val, 1000, d["n_cols"], d["y"][lo:hi], 1e-3, "dual", seed=3 + rank, n_global=2000,
                       rank=rank, world=world, nccl_comm=comm)
        s.epoch(1)
        g = s.aggregate("optimal")
        gap = s.duality_gap()
        out.append(f"rank{rank}: world-2 NCCL aggregate gamma={g:.6f} gap={gap:.3e}")
        s.close()
        os.environ["SCD_P2P_AGG"] = "1"
        s = scd.Solver(ptr, idx, val, 1000, d["n_cols"], d["y"][lo:hi], 1e-3, "dual", seed=3 + rank, n_global=2000,
                       rank=rank, world=world, nccl_comm=comm)
        s.epoch(1)
        g = s.aggregate("optimal")
        gap = s.duality_gap()
        out.append(f"rank{rank}: world-2 P2P aggregate gamma={g:.6f} gap={gap:.3e} p2p_state={s.info().get('p2p', '?')}")
        s.close()
        scd.nccl_comm_destroy(comm)
    except Exception:  # noqa: BLE001
        out.append(f"rank{rank}: EXC " + traceback.format_exc()[-1500:])
    q.put(out)


def main():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, 29511, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = []
    for _ in ps:
        try:
            res.extend(q.get(timeout=240))
        except Exception:  # noqa: BLE001
            res.append("timeout waiting for a rank")
    for p in ps:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    for line in res:
        print(line)


if __name__ == "__main__":
    main()
