// comm.cu — the collectives of the distributed path (Alg. 3/4 "aggregate updates", and the
// collective objective / gap / shared-vector rebuild): NCCL over NVLink / NVSwitch by default, or the
// caller's host-side hooks (scd_collectives in scd.h: several ranks on one device, where NCCL refuses
// to run).  Every call is ordered on the context stream.
#include "common.cuh"

namespace scd {
namespace {

ncclDataType_t nccl_type(scd_dtype dt) {
  switch (dt) {
    case SCD_DT_F32: return ncclFloat;
    case SCD_DT_F64: return ncclDouble;
    case SCD_DT_I32: return ncclInt32;
    case SCD_DT_I64: return ncclInt64;
    default: return ncclUint8;
  }
}

ncclRedOp_t nccl_op(scd_redop op) { return op == SCD_OP_MAX ? ncclMax : (op == SCD_OP_MIN ? ncclMin : ncclSum); }

}  // namespace

scd_status coll_allreduce(scd_ctx *c, void *buf, size_t count, scd_dtype dt, scd_redop op) {
  if (c->nccl) {
    SCD_NCK(c, ncclAllReduce(buf, buf, count, nccl_type(dt), nccl_op(op), c->nccl, c->stream));
    return SCD_OK;
  }
  if (c->coll && c->coll->allreduce) {
    const int32_t r = c->coll->allreduce(c->coll->user, buf, (int64_t)count, (int32_t)dt, (int32_t)op, (void *)c->stream);
    if (r != 0) return fail(c, SCD_E_NCCL, "collectives->allreduce failed (" + std::to_string(r) + ")");
    return SCD_OK;
  }
  return fail(c, SCD_E_STATE, "no communicator");
}

scd_status coll_allgather(scd_ctx *c, const void *send, void *recv, size_t bytes) {
  if (c->nccl) {
    SCD_NCK(c, ncclAllGather(send, recv, bytes, ncclUint8, c->nccl, c->stream));
    return SCD_OK;
  }
  if (c->coll && c->coll->allgather) {
    const int32_t r = c->coll->allgather(c->coll->user, send, recv, (int64_t)bytes, (void *)c->stream);
    if (r != 0) return fail(c, SCD_E_NCCL, "collectives->allgather failed (" + std::to_string(r) + ")");
    return SCD_OK;
  }
  return fail(c, SCD_E_STATE, "no communicator");
}

scd_status coll_group_start(scd_ctx *c) {
  if (c->nccl) SCD_NCK(c, ncclGroupStart());
  return SCD_OK;
}

scd_status coll_group_end(scd_ctx *c) {
  if (c->nccl) SCD_NCK(c, ncclGroupEnd());
  return SCD_OK;
}

}  // namespace scd
