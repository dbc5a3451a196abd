// api.cu — the extern "C" entry points declared in include/scd.h: argument validation, context
// lifecycle, memory ownership, error reporting.  All compute happens in the kernels of
// epoch.cu / evaluate.cu / aggregate.cu / layout.cu.
#include <cstring>
#include <new>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace scd {

static thread_local std::string g_err;

void set_global_error(const std::string &msg) { g_err = msg; }

scd_status fail(scd_ctx *c, scd_status s, const std::string &msg) {
  if (c)
    c->err = msg;
  else
    g_err = msg;
  return s;
}

scd_status cuda_fail(scd_ctx *c, cudaError_t e, const char *what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  cudaGetLastError();  // clear sticky-free errors
  return fail(c, e == cudaErrorMemoryAllocation ? SCD_E_OOM : SCD_E_CUDA, m);
}

}  // namespace scd

using namespace scd;

namespace {

template <typename T>
scd_status dev_alloc(scd_ctx *c, T **p, int64_t n, const char *what) {
  cudaError_t e = cudaMalloc((void **)p, sizeof(T) * (size_t)(n > 0 ? n : 1));
  if (e != cudaSuccess) return cuda_fail(c, e, what);
  return SCD_OK;
}

void free_ctx(scd_ctx *c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaFree(c->own_ptr);
  cudaFree(c->own_idx);
  cudaFree(c->own_val);
  cudaFree(c->own_y);
  cudaFree(c->x);
  cudaFree(c->x0);
  cudaFree(c->sv_base);
  cudaFree(c->sv0);
  cudaFree(c->svr);
  cudaFree(c->norm);
  cudaFree(c->empty_list);
  for (int i = 0; i < kMaxBins; ++i) {
    cudaFree(c->bins[i].list);
    cudaFree(c->bins[i].bperm);
  }
  cudaFree(c->counters);
  cudaFree(c->hot_idx);
  cudaFree(c->hot_ids);
  cudaFree(c->hot_hc);
  cudaFree(c->acc);
  cudaFree(c->vec64);
  cudaFree(c->comm);
  for (void *p : c->p2p_open) cudaIpcCloseMemHandle(p);
  cudaFree(c->p2p_ptrs);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (auto &p : c->ev_pending) {
    cudaEventDestroy(p.second.first);
    cudaEventDestroy(p.second.second);
  }
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

#define CK_CTX(c)                                     \
  do {                                                \
    if (!(c)) return SCD_E_INVALID_ARG;               \
    c->err.clear();                                   \
  } while (0)

}  // namespace

namespace {
// Matrix-to-matrix utilities (transpose, renumber): stage host inputs / outputs through device
// buffers and run `op(p, i, v, outer, inner, nnz, dp, di, dv, s, err)` on device pointers.
// out_outer = outer length of the output (inner for the transpose, outer for the renumbering).
template <typename Op>
scd_status matrix_op(const scd_matrix *in, int64_t *ptr_out, int32_t *idx_out, float *val_out, scd_mem out_mem,
                     bool transpose_shape, Op op) {
  if (!in || !ptr_out || !in->ptr || (in->nnz > 0 && (!idx_out || !in->idx || (in->val && !val_out))))
    return fail(nullptr, SCD_E_INVALID_ARG, "NULL argument");
  const bool has_val = in->val != nullptr;
  const int64_t outer = in->layout == SCD_CSR ? in->n_rows : in->n_cols;
  const int64_t inner = in->layout == SCD_CSR ? in->n_cols : in->n_rows;
  if (outer < 0 || inner < 1 || in->nnz < 0) return fail(nullptr, SCD_E_INVALID_ARG, "bad shape");
  const int64_t nnz = in->nnz, out_outer = transpose_shape ? inner : outer;
  cudaStream_t s = 0;
  std::string err;
  const int64_t *p = in->ptr;
  const int32_t *i = in->idx;
  const float *v = in->val;
  void *tp = nullptr, *ti = nullptr, *tv = nullptr, *op_ = nullptr, *oi = nullptr, *ov = nullptr;
  scd_status st = SCD_OK;
  auto alloc = [&](void **q, size_t b) {
    if (st != SCD_OK) return;
    if (cudaMalloc(q, b > 0 ? b : 1) != cudaSuccess) st = fail(nullptr, SCD_E_OOM, "matrix op alloc");
  };
  if (in->mem == SCD_MEM_HOST) {
    alloc(&tp, sizeof(int64_t) * (size_t)(outer + 1));
    alloc(&ti, sizeof(int32_t) * (size_t)nnz);
    if (has_val) alloc(&tv, sizeof(float) * (size_t)nnz);
    if (st == SCD_OK) {
      cudaMemcpy(tp, p, sizeof(int64_t) * (size_t)(outer + 1), cudaMemcpyHostToDevice);
      if (nnz) {
        cudaMemcpy(ti, i, sizeof(int32_t) * (size_t)nnz, cudaMemcpyHostToDevice);
        if (has_val) cudaMemcpy(tv, v, sizeof(float) * (size_t)nnz, cudaMemcpyHostToDevice);
      }
      p = (const int64_t *)tp;
      i = (const int32_t *)ti;
      v = (const float *)tv;
    }
  }
  int64_t *dp = ptr_out;
  int32_t *di = idx_out;
  float *dv = has_val ? val_out : nullptr;
  if (out_mem == SCD_MEM_HOST) {
    alloc(&op_, sizeof(int64_t) * (size_t)(out_outer + 1));
    alloc(&oi, sizeof(int32_t) * (size_t)nnz);
    if (has_val) alloc(&ov, sizeof(float) * (size_t)nnz);
    dp = (int64_t *)op_;
    di = (int32_t *)oi;
    dv = (float *)ov;
  }
  if (st == SCD_OK) {
    st = op(p, i, v, outer, inner, nnz, dp, di, dv, s, err);
    if (st != SCD_OK) fail(nullptr, st, err);
  }
  if (st == SCD_OK && cudaStreamSynchronize(s) != cudaSuccess) st = fail(nullptr, SCD_E_CUDA, "matrix op sync");
  if (st == SCD_OK && out_mem == SCD_MEM_HOST) {
    cudaMemcpy(ptr_out, op_, sizeof(int64_t) * (size_t)(out_outer + 1), cudaMemcpyDeviceToHost);
    if (nnz) {
      cudaMemcpy(idx_out, oi, sizeof(int32_t) * (size_t)nnz, cudaMemcpyDeviceToHost);
      if (has_val) cudaMemcpy(val_out, ov, sizeof(float) * (size_t)nnz, cudaMemcpyDeviceToHost);
    }
  }
  cudaFree(tp);
  cudaFree(ti);
  cudaFree(tv);
  cudaFree(op_);
  cudaFree(oi);
  cudaFree(ov);
  return st;
}
}  // namespace

namespace {
// NVTX ranges around the public calls (header-only NVTX 3: free unless a profiler is attached), so
// nsys / ncu timelines show epochs, aggregation rounds and evaluations by name.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

extern "C" {

void scd_default_options(scd_options *o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->world = 1;
  o->validate = 1;
}

void scd_struct_sizes(int64_t *sizes_out) {
  if (!sizes_out) return;
  sizes_out[0] = (int64_t)sizeof(scd_matrix);
  sizes_out[1] = (int64_t)sizeof(scd_options);
  sizes_out[2] = (int64_t)sizeof(scd_info);
  sizes_out[3] = (int64_t)sizeof(scd_collectives);
}

const char *scd_status_string(scd_status s) {
  switch (s) {
    case SCD_OK: return "SCD_OK";
    case SCD_E_INVALID_ARG: return "SCD_E_INVALID_ARG";
    case SCD_E_BAD_MATRIX: return "SCD_E_BAD_MATRIX";
    case SCD_E_OOM: return "SCD_E_OOM";
    case SCD_E_CUDA: return "SCD_E_CUDA";
    case SCD_E_NCCL: return "SCD_E_NCCL";
    case SCD_E_STATE: return "SCD_E_STATE";
    case SCD_E_UNSUPPORTED: return "SCD_E_UNSUPPORTED";
  }
  return "SCD_E_UNKNOWN";
}

const char *scd_last_error(const scd_ctx *c) { return c ? c->err.c_str() : g_err.c_str(); }
const char *scd_last_global_error(void) { return g_err.c_str(); }

scd_status scd_create(const scd_matrix *A, const float *y, scd_mem y_mem, double lambda, scd_form form,
                      const scd_options *opt_in, scd_ctx **out) {
  NvtxRange nvtx_("scd_create");
  g_err.clear();
  if (!out) return fail(nullptr, SCD_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!A || !y) return fail(nullptr, SCD_E_INVALID_ARG, "A or y is NULL");
  if (!(lambda > 0.0)) return fail(nullptr, SCD_E_INVALID_ARG, "lambda must be > 0");
  if (form != SCD_PRIMAL && form != SCD_DUAL) return fail(nullptr, SCD_E_INVALID_ARG, "bad form");
  if (A->n_rows < 1 || A->n_cols < 1 || A->nnz < 0) return fail(nullptr, SCD_E_INVALID_ARG, "need N >= 1, M >= 1, nnz >= 0");
  if ((form == SCD_PRIMAL && A->layout != SCD_CSC) || (form == SCD_DUAL && A->layout != SCD_CSR))
    return fail(nullptr, SCD_E_INVALID_ARG, "primal needs CSC, dual needs CSR");
  if (!A->ptr || (A->nnz > 0 && (!A->idx))) return fail(nullptr, SCD_E_INVALID_ARG, "matrix arrays are NULL");
  if (A->n_rows > INT32_MAX || A->n_cols > INT32_MAX) return fail(nullptr, SCD_E_UNSUPPORTED, "dimension > 2^31-1");
  scd_options opt;
  scd_default_options(&opt);
  if (opt_in) opt = *opt_in;
  if (opt.world < 1 || opt.rank < 0 || opt.rank >= opt.world) return fail(nullptr, SCD_E_INVALID_ARG, "bad rank/world");
  if (opt.world > 1 && !opt.nccl_comm && !opt.collectives)
    return fail(nullptr, SCD_E_STATE, "world > 1 requires nccl_comm or collectives");
  if (opt.collectives && (!opt.collectives->allreduce || !opt.collectives->allgather))
    return fail(nullptr, SCD_E_INVALID_ARG, "collectives needs both allreduce and allgather");
  if (opt.n_global < 0) return fail(nullptr, SCD_E_INVALID_ARG, "n_global < 0");
  // a dual shard needs the global N of λN (c14): a silent fallback to the local row count would
  // change the coordinate update, γ and the objectives
  if (form == SCD_DUAL && opt.world > 1 && opt.n_global == 0)
    return fail(nullptr, SCD_E_INVALID_ARG, "dual with world > 1 needs n_global (global N)");

  scd_ctx *c = new (std::nothrow) scd_ctx();
  if (!c) return fail(nullptr, SCD_E_OOM, "host allocation failed");
  c->form = form;
  c->opt = opt;
  c->n_rows = A->n_rows;
  c->n_cols = A->n_cols;
  c->nnz = A->nnz;
  c->n_coord = form == SCD_PRIMAL ? A->n_cols : A->n_rows;
  c->n_shared = form == SCD_PRIMAL ? A->n_rows : A->n_cols;
  c->lam = lambda;
  c->n_global = form == SCD_PRIMAL ? A->n_rows : (opt.n_global > 0 ? opt.n_global : A->n_rows);
  c->lamN = lambda * (double)c->n_global;
  c->nccl = (ncclComm_t)opt.nccl_comm;
  c->coll = c->nccl ? nullptr : opt.collectives;
  cudaGetDevice(&c->device);
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->device);
  scd_status st = SCD_OK;
  auto bail = [&](scd_status s2) {
    std::string m = c->err;
    free_ctx(c);
    g_err = m;
    return s2;
  };
  if (opt.stream) {
    c->stream = (cudaStream_t)opt.stream;
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return bail(cuda_fail(c, e, "cudaStreamCreate"));
    c->own_stream = true;
  }
  cudaStream_t s = c->stream;
  const int64_t outer = c->n_coord;
  // matrix
  if (A->mem == SCD_MEM_DEVICE) {
    c->ptr = A->ptr;
    c->idx = A->idx;
    c->val = A->val;
  } else {
    int64_t *p;
    int32_t *i;
    float *v;
    if ((st = dev_alloc(c, &p, outer + 1, "alloc ptr")) != SCD_OK) return bail(st);
    c->own_ptr = p;
    if ((st = dev_alloc(c, &i, A->nnz, "alloc idx")) != SCD_OK) return bail(st);
    c->own_idx = i;
    v = nullptr;
    if (A->val) {  // val == NULL: implicit values 1.0f (NEXT-1), nothing to upload
      if ((st = dev_alloc(c, &v, A->nnz, "alloc val")) != SCD_OK) return bail(st);
      c->own_val = v;
    }
    cudaMemcpyAsync(p, A->ptr, sizeof(int64_t) * (size_t)(outer + 1), cudaMemcpyHostToDevice, s);
    if (A->nnz > 0) {
      cudaMemcpyAsync(i, A->idx, sizeof(int32_t) * (size_t)A->nnz, cudaMemcpyHostToDevice, s);
      if (A->val) cudaMemcpyAsync(v, A->val, sizeof(float) * (size_t)A->nnz, cudaMemcpyHostToDevice, s);
    }
    c->ptr = p;
    c->idx = i;
    c->val = v;
  }
  if (y_mem == SCD_MEM_DEVICE) {
    c->y = y;
  } else {
    float *yy;
    if ((st = dev_alloc(c, &yy, c->n_rows, "alloc y")) != SCD_OK) return bail(st);
    c->own_y = yy;
    cudaMemcpyAsync(yy, y, sizeof(float) * (size_t)c->n_rows, cudaMemcpyHostToDevice, s);
    c->y = yy;
  }
  if (cudaGetLastError() != cudaSuccess) return bail(fail(c, SCD_E_CUDA, "upload failed"));
  if (opt.validate) {
    const int64_t inner = form == SCD_PRIMAL ? c->n_rows : c->n_cols;
    if ((st = validate_matrix(c, outer, inner)) != SCD_OK) return bail(st);
  }
  if ((st = dev_alloc(c, &c->x, c->n_coord, "alloc model")) != SCD_OK) return bail(st);
  if ((st = dev_alloc(c, &c->x0, c->n_coord, "alloc model snapshot")) != SCD_OK) return bail(st);
  // the shared vector sits at a tuned offset inside a slightly larger allocation (tune_shared_layout)
  if ((st = dev_alloc(c, &c->sv_base, c->n_shared + kMaxSvOffsetFloats, "alloc shared")) != SCD_OK) return bail(st);
  c->sv = c->sv_base;
  if ((st = dev_alloc(c, &c->sv0, c->n_shared, "alloc shared snapshot")) != SCD_OK) return bail(st);
  if ((st = dev_alloc(c, &c->norm, c->n_coord, "alloc norms")) != SCD_OK) return bail(st);
  if ((st = dev_alloc(c, &c->acc, 32, "alloc acc")) != SCD_OK) return bail(st);
  if ((st = dev_alloc(c, &c->vec64, c->n_shared, "alloc vec64")) != SCD_OK) return bail(st);
  if ((st = dev_alloc(c, &c->comm, c->n_shared, "alloc comm")) != SCD_OK) return bail(st);
  cudaMemsetAsync(c->x, 0, sizeof(float) * (size_t)c->n_coord, s);
  cudaMemsetAsync(c->x0, 0, sizeof(float) * (size_t)c->n_coord, s);
  if ((st = compute_norms(c)) != SCD_OK) return bail(st);
  if ((st = build_schedule(c)) != SCD_OK) return bail(st);
  if (!opt.validate) {
    // the head and hot-set kernels accumulate a row's updates with plain shared-memory
    // read-modify-writes, correct only for unique indices within a coordinate: with validation
    // off, still check the index invariants whenever one of them was selected
    bool combining = false;
    for (int i = 0; i < c->n_bins; ++i) combining |= c->bins[i].head > 0 || c->bins[i].hot > 0;
    const int64_t inner = form == SCD_PRIMAL ? c->n_rows : c->n_cols;
    if (combining && (st = validate_matrix(c, outer, inner)) != SCD_OK) return bail(st);
  }
  {
    // shared-vector placement: SCD_SV_OFFSET (bytes) pins it; otherwise large asynchronous
    // problems are probed (tune_shared_layout); SCD_SV_TUNE=0 disables the probe
    const char *e = getenv("SCD_SV_OFFSET");
    const char *tn = getenv("SCD_SV_TUNE");
    if (e) {
      int64_t off = (atoll(e) / 16) * 4;
      if (off < 0) off = 0;
      if (off > kMaxSvOffsetFloats) off = kMaxSvOffsetFloats;
      c->sv = c->sv_base + off;
      c->sv_offset_bytes = off * 4;
    } else if (!opt.deterministic && c->n_bins > 0 && c->nnz >= (int64_t)20000000 && !(tn && atoi(tn) == 0)) {
      if ((st = tune_shared_layout(c)) != SCD_OK) return bail(st);
    }
  }
  // initial state (Alg. 1/2 "Initialize: β = 0, w = 0"): model 0; primal residual r = y - 0 = y; w̄ = 0
  if (form == SCD_PRIMAL) {
    cudaMemcpyAsync(c->sv, c->y, sizeof(float) * (size_t)c->n_shared, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(c->sv0, c->y, sizeof(float) * (size_t)c->n_shared, cudaMemcpyDeviceToDevice, s);
  } else {
    cudaMemsetAsync(c->sv, 0, sizeof(float) * (size_t)c->n_shared, s);
    cudaMemsetAsync(c->sv0, 0, sizeof(float) * (size_t)c->n_shared, s);
  }
  // the all-zero start is already the fixed point of every empty coordinate (Δ = -β = 0 primal);
  // the dual's empty rows still move (α_n = y_n/N), so they run in the first epoch.
  c->empty_dirty = (form == SCD_DUAL);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return bail(cuda_fail(c, e, "create sync"));
  *out = c;
  return SCD_OK;
}

scd_status scd_epoch_part(scd_ctx *c, uint32_t epoch, int32_t part, int32_t nparts) {
  NvtxRange nvtx_("scd_epoch_part");
  CK_CTX(c);
  if (nparts < 1 || part < 0 || part >= nparts || nparts > 1024)
    return fail(c, SCD_E_INVALID_ARG, "need 0 <= part < nparts <= 1024");
  ++c->model_version;
  return run_epoch(c, epoch, part, nparts);
}

scd_status scd_epoch(scd_ctx *c, uint32_t epoch) {
  NvtxRange nvtx_("scd_epoch");
  CK_CTX(c);
  scd_status st = run_epoch(c, epoch, 0, 1);
  if (st != SCD_OK) return st;
  ++c->epochs_done;
  ++c->model_version;
  // P:164 recomputation scheme.  Without a communicator it runs here, every k epochs;
  // with one (world > 1) the shared vector is the sum over the ranks, so it is rebuilt from the
  // aggregated model at the end of scd_aggregate (every k rounds) instead.
  if (c->opt.recompute_every > 0 && !c->has_comm() && (c->epochs_done % (uint32_t)c->opt.recompute_every) == 0) {
    st = rebuild_shared(c);
    if (st != SCD_OK) return st;
  }
  return SCD_OK;
}

scd_status scd_objective(scd_ctx *c, double *primal, double *dual) {
  NvtxRange nvtx_("scd_objective");
  CK_CTX(c);
  return evaluate(c, primal, dual, nullptr);
}

scd_status scd_duality_gap(scd_ctx *c, double *gap) {
  NvtxRange nvtx_("scd_duality_gap");
  CK_CTX(c);
  if (!gap) return fail(c, SCD_E_INVALID_ARG, "gap is NULL");
  return evaluate(c, nullptr, nullptr, gap);
}

scd_status scd_aggregate(scd_ctx *c, scd_agg mode, double *gamma) {
  NvtxRange nvtx_("scd_aggregate");
  CK_CTX(c);
  if (mode != SCD_AGG_ADD && mode != SCD_AGG_AVERAGE && mode != SCD_AGG_OPTIMAL)
    return fail(c, SCD_E_INVALID_ARG, "bad aggregation mode");
  if (c->opt.world > 1 && !c->has_comm()) return fail(c, SCD_E_STATE, "no communicator");
  scd_status st = aggregate(c, mode, gamma);
  if (st != SCD_OK) return st;
  ++c->model_version;
  ++c->rounds_done;
  if (c->opt.recompute_every > 0 && c->has_comm() && (c->rounds_done % (uint32_t)c->opt.recompute_every) == 0) {
    // rebuild the shared vector from the aggregated model: Σ_k A_k x_k in fp64 over the ranks
    st = rebuild_shared(c);
    if (st != SCD_OK) return st;
    SCD_CK(c, cudaStreamSynchronize(c->stream));
  }
  return SCD_OK;
}

scd_status scd_aggregate_group(scd_ctx *const *cs, int32_t k, scd_agg mode, double *gamma) {
  g_err.clear();
  if (!cs || k < 1) return fail(nullptr, SCD_E_INVALID_ARG, "need k >= 1 contexts");
  if (mode != SCD_AGG_ADD && mode != SCD_AGG_AVERAGE && mode != SCD_AGG_OPTIMAL)
    return fail(nullptr, SCD_E_INVALID_ARG, "bad aggregation mode");
  for (int i = 0; i < k; ++i) {
    if (!cs[i]) return fail(nullptr, SCD_E_INVALID_ARG, "NULL context");
    if (cs[i]->form != cs[0]->form || cs[i]->n_shared != cs[0]->n_shared || cs[i]->lam != cs[0]->lam ||
        cs[i]->device != cs[0]->device || cs[i]->n_global != cs[0]->n_global || cs[i]->opt.world != 1)
      return fail(nullptr, SCD_E_INVALID_ARG, "group contexts must share form, shared length, lambda, N, device; world = 1");
    if (cs[i]->opt.recompute_every > 0)
      return fail(nullptr, SCD_E_UNSUPPORTED, "recompute_every with logical workers (each would rebuild its own shard)");
  }
  scd_status st = aggregate_group(cs, k, mode, gamma);
  for (int i = 0; i < k && st == SCD_OK; ++i) ++cs[i]->model_version;
  if (st != SCD_OK) g_err = cs[0]->err;
  return st;
}

scd_status scd_evaluate_group(scd_ctx *const *cs, int32_t k, double *primal, double *dual, double *gap) {
  g_err.clear();
  if (!cs || k < 1) return fail(nullptr, SCD_E_INVALID_ARG, "need k >= 1 contexts");
  for (int i = 0; i < k; ++i) {
    if (!cs[i]) return fail(nullptr, SCD_E_INVALID_ARG, "NULL context");
    if (cs[i]->form != cs[0]->form || cs[i]->n_shared != cs[0]->n_shared || cs[i]->lam != cs[0]->lam ||
        cs[i]->device != cs[0]->device || cs[i]->n_global != cs[0]->n_global || cs[i]->has_comm())
      return fail(nullptr, SCD_E_INVALID_ARG, "group contexts must share form, shared length, lambda, N, device; no comm");
  }
  scd_status st = evaluate_group(cs, k, primal, dual, gap);
  if (st != SCD_OK) g_err = cs[0]->err;
  return st;
}

scd_status scd_get_model(scd_ctx *c, float *host_out, int64_t len) {
  CK_CTX(c);
  if (!host_out || len != c->n_coord) return fail(c, SCD_E_INVALID_ARG, "model length mismatch");
  SCD_CK(c, cudaMemcpyAsync(host_out, c->x, sizeof(float) * (size_t)len, cudaMemcpyDeviceToHost, c->stream));
  SCD_CK(c, cudaStreamSynchronize(c->stream));
  return SCD_OK;
}

scd_status scd_get_shared(scd_ctx *c, float *host_out, int64_t len) {
  CK_CTX(c);
  if (!host_out || len != c->n_shared) return fail(c, SCD_E_INVALID_ARG, "shared length mismatch");
  scd_status st = shared_to_w(c, c->comm);
  if (st != SCD_OK) return st;
  SCD_CK(c, cudaMemcpyAsync(host_out, c->comm, sizeof(float) * (size_t)len, cudaMemcpyDeviceToHost, c->stream));
  SCD_CK(c, cudaStreamSynchronize(c->stream));
  return SCD_OK;
}

scd_status scd_set_model(scd_ctx *c, const float *host_in, int64_t len) {
  CK_CTX(c);
  if (!host_in || len != c->n_coord) return fail(c, SCD_E_INVALID_ARG, "model length mismatch");
  SCD_CK(c, cudaMemcpyAsync(c->x, host_in, sizeof(float) * (size_t)len, cudaMemcpyHostToDevice, c->stream));
  ++c->model_version;
  scd_status st = rebuild_shared(c);
  if (st != SCD_OK) return st;
  c->empty_dirty = true;
  SCD_CK(c, cudaStreamSynchronize(c->stream));
  return SCD_OK;
}

scd_status scd_recompute_shared(scd_ctx *c) {
  NvtxRange nvtx_("scd_recompute_shared");
  CK_CTX(c);
  scd_status st = rebuild_shared(c);
  if (st != SCD_OK) return st;
  SCD_CK(c, cudaStreamSynchronize(c->stream));
  return SCD_OK;
}

scd_status scd_get_stream(scd_ctx *c, void **stream) {
  CK_CTX(c);
  if (!stream) return fail(c, SCD_E_INVALID_ARG, "stream is NULL");
  *stream = (void *)c->stream;
  return SCD_OK;
}

scd_status scd_get_info(scd_ctx *c, scd_info *info) {
  CK_CTX(c);
  if (!info) return fail(c, SCD_E_INVALID_ARG, "info is NULL");
  std::memset(info, 0, sizeof(*info));
  info->n_coord = c->n_coord;
  info->n_shared = c->n_shared;
  info->nnz = c->nnz;
  info->n_nonempty = c->n_nonempty;
  info->n_bins = c->n_bins;
  for (int i = 0; i < c->n_bins && i < 4; ++i) {
    info->bin_kind[i] = c->bins[i].lanes;
    info->bin_count[i] = c->bins[i].count;
    info->bin_nnz[i] = c->bins[i].nnz;
    info->bin_grid[i] = c->bins[i].grid;
    info->bin_block[i] = c->bins[i].block;
  }
  info->launches = c->launches;
  info->tau_star = c->tau_star;
  info->n_slices = c->n_slices;
  info->sv_offset_bytes = c->sv_offset_bytes;
  info->probe_best_ms = 0.f;
  info->probe_worst_ms = 0.f;
  for (int i = 0; i < c->n_probe; ++i) {
    if (i == 0 || c->probe_ms[i] < info->probe_best_ms) info->probe_best_ms = c->probe_ms[i];
    if (c->probe_ms[i] > info->probe_worst_ms) info->probe_worst_ms = c->probe_ms[i];
  }
  info->hot_cover = c->hot_cover;
  info->tail_snap = c->tail_snap;
  info->tail_tau = c->tail_tau;
  info->tail_roll = c->tail_roll;
  info->head_copy = c->head_copy;
  info->hot_copy = c->hot_copy;
  info->hot_tp = c->hot_tp ? 1 : 0;
  info->hot_hp = (c->hot_hp && c->hot_copy > 0 && c->hot_tp) ? 1 : 0;
  info->hot_tail_tau = c->hot_tail_tau;
  info->sm_head = info->sm_chunk = info->sm_ch = info->sm_rh = 0;
  for (int i = 0; i < c->n_bins && i < 4; ++i)
    if (c->bins[i].sm) {
      info->sm_head = c->bins[i].sm;
      info->sm_chunk = sm_chunk_entries(c->bins[i].sm);
      info->sm_ch = c->bins[i].sm_ch;
      info->sm_rh = c->bins[i].sm_rh;
    }
  info->inflight_cap = 0;
  for (int i = 0; i < c->n_bins && i < 4; ++i) {
    info->bin_cap[i] = c->bins[i].cap;
    info->bin_tau[i] = c->bins[i].tau;
    info->bin_head[i] = c->bins[i].head;
    info->bin_flush[i] = c->bins[i].flush;
    info->bin_hot[i] = c->bins[i].hot;
    info->bin_snap[i] = c->bins[i].snap;
    if (c->bins[i].cap > info->inflight_cap) info->inflight_cap = c->bins[i].cap;
  }
  return SCD_OK;
}

scd_status scd_profile_read(scd_ctx *c, double *ms_out, int64_t *count_out, int32_t n, int32_t *filled) {
  CK_CTX(c);
  scd_status st = profile_collect(c);
  if (st != SCD_OK) return st;
  int m = c->n_bins < n ? c->n_bins : n;
  for (int i = 0; i < m; ++i) {
    if (ms_out) ms_out[i] = c->bins[i].ms;
    if (count_out) count_out[i] = c->bins[i].prof_launches;
    c->bins[i].ms = 0.0;
    c->bins[i].prof_launches = 0;
  }
  if (filled) *filled = m;
  return SCD_OK;
}

void scd_destroy(scd_ctx *c) { free_ctx(c); }

scd_status scd_permutation(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n, int64_t *host_out) {
  g_err.clear();
  if (n < 0 || (n > 0 && !host_out)) return fail(nullptr, SCD_E_INVALID_ARG, "bad n / output");
  if (n == 0) return SCD_OK;
  int64_t *d = nullptr;
  cudaError_t e = cudaMalloc((void **)&d, sizeof(int64_t) * (size_t)n);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "alloc");
  scd_status st = launch_perm_export(seed, epoch, stream, n, d, 0);
  if (st == SCD_OK) {
    e = cudaMemcpy(host_out, d, sizeof(int64_t) * (size_t)n, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = cuda_fail(nullptr, e, "copy");
  } else {
    fail(nullptr, st, "permutation kernel failed");
  }
  cudaFree(d);
  return st;
}

scd_status scd_block_permutation(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n, int64_t blk,
                                 int64_t *host_out) {
  g_err.clear();
  if (n < 0 || blk < 1 || (n > 0 && !host_out)) return fail(nullptr, SCD_E_INVALID_ARG, "bad n / blk / output");
  if (n == 0) return SCD_OK;
  int64_t *d = nullptr;
  cudaError_t e = cudaMalloc((void **)&d, sizeof(int64_t) * (size_t)n);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "alloc");
  scd_status st = launch_block_order_export(seed, epoch, stream, n, blk, d, 0);
  if (st == SCD_OK) {
    e = cudaMemcpy(host_out, d, sizeof(int64_t) * (size_t)n, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = cuda_fail(nullptr, e, "copy");
  } else {
    fail(nullptr, st, "block order kernel failed");
  }
  cudaFree(d);
  return st;
}

scd_status scd_partition(uint64_t seed, int64_t count, int32_t k, int32_t *host_owner_out) {
  g_err.clear();
  if (count < 0 || k < 1 || (count > 0 && !host_owner_out)) return fail(nullptr, SCD_E_INVALID_ARG, "bad count / k");
  if (count == 0) return SCD_OK;
  int32_t *d = nullptr;
  cudaError_t e = cudaMalloc((void **)&d, sizeof(int32_t) * (size_t)count);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "alloc");
  scd_status st = launch_partition_export(seed, count, k, d, 0);
  if (st == SCD_OK) {
    e = cudaMemcpy(host_owner_out, d, sizeof(int32_t) * (size_t)count, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = cuda_fail(nullptr, e, "copy");
  } else {
    fail(nullptr, st, "partition kernel failed");
  }
  cudaFree(d);
  return st;
}


scd_status scd_partition_balanced(const int64_t *ptr, int64_t n, scd_mem ptr_mem, uint64_t seed, int32_t k,
                                  int32_t *host_owner_out) {
  g_err.clear();
  if (!ptr || n < 0 || k < 1 || (n > 0 && !host_owner_out)) return fail(nullptr, SCD_E_INVALID_ARG, "bad ptr / n / k");
  if (n == 0) return SCD_OK;
  if (n > INT32_MAX) return fail(nullptr, SCD_E_UNSUPPORTED, "n > 2^31-1");
  int64_t *dp = const_cast<int64_t *>(ptr);
  int32_t *d_owner = nullptr;
  cudaStream_t s = 0;
  if (ptr_mem == SCD_MEM_HOST) {
    if (cudaMalloc((void **)&dp, sizeof(int64_t) * (size_t)(n + 1)) != cudaSuccess) return fail(nullptr, SCD_E_OOM, "alloc");
    cudaMemcpy(dp, ptr, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyHostToDevice);
  }
  scd_status st = SCD_OK;
  if (cudaMalloc((void **)&d_owner, sizeof(int32_t) * (size_t)n) != cudaSuccess) {
    st = fail(nullptr, SCD_E_OOM, "alloc");
  } else {
    std::string err;
    st = partition_balanced_device(dp, n, seed, k, d_owner, s, err);
    if (st != SCD_OK) fail(nullptr, st, err);
    if (st == SCD_OK && cudaMemcpy(host_owner_out, d_owner, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToHost) != cudaSuccess)
      st = fail(nullptr, SCD_E_CUDA, "copy");
  }
  cudaFree(d_owner);
  if (ptr_mem == SCD_MEM_HOST) cudaFree(dp);
  return st;
}

scd_status scd_transpose(const scd_matrix *in, int64_t *ptr_out, int32_t *idx_out, float *val_out, scd_mem out_mem) {
  g_err.clear();
  // in->val == NULL (implicit values) transposes the pattern only; val_out is then ignored
  return matrix_op(in, ptr_out, idx_out, val_out, out_mem, true,
                   [](const int64_t *p, const int32_t *i, const float *v, int64_t outer, int64_t inner, int64_t nnz,
                      int64_t *dp, int32_t *di, float *dv, cudaStream_t s, std::string &err) {
                     return transpose_device(p, i, v, outer, inner, nnz, dp, di, dv, s, err);
                   });
}

scd_status scd_renumber(const scd_matrix *in, int64_t *ptr_out, int32_t *idx_out, float *val_out,
                        int32_t *new_of_old_out, scd_mem out_mem) {
  g_err.clear();
  if (!new_of_old_out) return fail(nullptr, SCD_E_INVALID_ARG, "NULL argument");
  if (!in) return fail(nullptr, SCD_E_INVALID_ARG, "NULL argument");
  const int64_t inner = in->layout == SCD_CSR ? in->n_cols : in->n_rows;
  if (inner < 1 || inner > INT32_MAX) return fail(nullptr, SCD_E_INVALID_ARG, "bad inner size");
  int32_t *d_map = new_of_old_out;
  if (out_mem == SCD_MEM_HOST && cudaMalloc((void **)&d_map, sizeof(int32_t) * (size_t)inner) != cudaSuccess)
    return fail(nullptr, SCD_E_OOM, "renumber alloc");
  scd_status st = matrix_op(in, ptr_out, idx_out, val_out, out_mem, false,
                            [&](const int64_t *p, const int32_t *i, const float *v, int64_t outer, int64_t inn,
                                int64_t nnz, int64_t *dp, int32_t *di, float *dv, cudaStream_t s, std::string &err) {
                              return renumber_device(p, i, v, outer, inn, nnz, dp, di, dv, d_map, s, err);
                            });
  if (out_mem == SCD_MEM_HOST) {
    if (st == SCD_OK) cudaMemcpy(new_of_old_out, d_map, sizeof(int32_t) * (size_t)inner, cudaMemcpyDeviceToHost);
    cudaFree(d_map);
  }
  return st;
}

scd_status scd_nccl_unique_id(void *id_out_128) {
  g_err.clear();
  if (!id_out_128) return fail(nullptr, SCD_E_INVALID_ARG, "NULL id");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclResult_t r = ncclGetUniqueId((ncclUniqueId *)id_out_128);
  if (r != ncclSuccess) return fail(nullptr, SCD_E_NCCL, ncclGetErrorString(r));
  return SCD_OK;
}

scd_status scd_nccl_comm_init(const void *id_128, int32_t world, int32_t rank, void **comm_out) {
  g_err.clear();
  if (!id_128 || !comm_out || world < 1 || rank < 0 || rank >= world)
    return fail(nullptr, SCD_E_INVALID_ARG, "bad id / world / rank");
  ncclUniqueId id;
  std::memcpy(&id, id_128, sizeof(id));
  ncclComm_t comm;
  ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) return fail(nullptr, SCD_E_NCCL, ncclGetErrorString(r));
  *comm_out = (void *)comm;
  return SCD_OK;
}

scd_status scd_nccl_comm_destroy(void *comm) {
  if (!comm) return SCD_OK;
  ncclResult_t r = ncclCommDestroy((ncclComm_t)comm);
  if (r != ncclSuccess) return fail(nullptr, SCD_E_NCCL, ncclGetErrorString(r));
  return SCD_OK;
}

}  // extern "C"
