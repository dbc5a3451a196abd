"""Host-side collective transport for the library's scd_collectives hooks (TEST INFRASTRUCTURE).

NCCL refuses two ranks on one GPU, so to run the library's world >= 2 code (aggregation rounds over a
communicator, the dual's active-extent exchange, the fused peer-memory exchange with its IPC handle
all-gather and scalar barriers, the collective objective / gap / shared-vector rebuild) with several
processes on a single B200, the tests hand the library these hooks: each one synchronises the
library's stream, moves the device buffer to the host, runs the collective over torch.distributed
(gloo) and copies the result back.  The arithmetic of the method stays in the library's kernels;
the hooks only move and sum buffers, as NCCL would."""
from __future__ import annotations

import traceback

import torch
import torch.distributed as dist

from paper_1702_07005_b200 import scd

_DT = {scd.DT_F32: (torch.float32, "<f4"), scd.DT_F64: (torch.float64, "<f8"), scd.DT_I32: (torch.int32, "<i4"),
       scd.DT_I64: (torch.int64, "<i8"), scd.DT_U8: (torch.uint8, "|u1")}
_OP = {scd.OP_SUM: dist.ReduceOp.SUM, scd.OP_MAX: dist.ReduceOp.MAX, scd.OP_MIN: dist.ReduceOp.MIN}


class _Cai:
    """__cuda_array_interface__ view of a raw device pointer (no copy)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def _dev(ptr: int, n: int, dtype_code: int) -> torch.Tensor:
    return torch.as_tensor(_Cai(ptr, n, _DT[dtype_code][1]), device="cuda")


def _sync(stream):
    torch.cuda.ExternalStream(int(stream)).synchronize() if stream else torch.cuda.synchronize()


class HostCollectives:
    """scd_collectives over the default torch.distributed process group.  ``calls`` counts the hook
    invocations by kind, so a test can check which collectives the library issued."""

    def __init__(self):
        self.calls = {"allreduce": 0, "allgather": 0}
        self.errors: list[str] = []
        self._ar = scd.ALLREDUCE_FN(self._allreduce)
        self._ag = scd.ALLGATHER_FN(self._allgather)
        self.struct = scd.Collectives(None, self._ar, self._ag)

    def _allreduce(self, user, buf, count, dtype, op, stream):
        try:
            self.calls["allreduce"] += 1
            _sync(stream)
            if count > 0:
                d = _dev(buf, count, dtype)
                h = d.cpu()
                dist.all_reduce(h, op=_OP[op])
                d.copy_(h)
                torch.cuda.synchronize()
            return 0
        except Exception:  # noqa: BLE001 - reported to the library as a failed collective
            self.errors.append(traceback.format_exc())
            return 1

    def _allgather(self, user, send, recv, nbytes, stream):
        try:
            self.calls["allgather"] += 1
            _sync(stream)
            world = dist.get_world_size()
            h = _dev(send, nbytes, scd.DT_U8).cpu()
            parts = [torch.empty_like(h) for _ in range(world)]
            dist.all_gather(parts, h)
            _dev(recv, nbytes * world, scd.DT_U8).copy_(torch.cat(parts))
            torch.cuda.synchronize()
            return 0
        except Exception:  # noqa: BLE001
            self.errors.append(traceback.format_exc())
            return 1
