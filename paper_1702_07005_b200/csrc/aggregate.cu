// aggregate.cu — one aggregation round of distributed SCD (Alg. 3, Alg. 4).
//
// Every worker k ran a local epoch from the common base point (w₀ or w̄₀ and its model
// snapshot x₀_k).  Then
//   Δ      = Σ_k (sv_k - sv₀)                    NCCL all-reduce over NVLink (world > 1)
//   S_x0dx = Σ_k <x₀_k, Δx_k>,  S_dxdx = Σ_k ||Δx_k||²,  S_ydx = Σ_k <y_k, Δx_k>   (P:364-368,
//            valid because the workers' supports are disjoint)
//   γ      = 1 (add) | 1/K (average, Alg. 3) | optimal:
//     primal (Eq. 7, numerator read as <w - y, Δw> (c3), base-point β (c5); on the
//             residual r = y - w kept by the GPU, <w₀ - y, Δw> = <r₀, Δr>):
//             γ = -(<r₀, Δr> + λN S_x0dx) / (||Δr||² + λN S_dxdx)
//     dual   (denominator read as N||Δα||² (c4)):
//             γ̄ = (S_ydx - N S_x0dx - <Δw̄, w̄₀>/λ) / (||Δw̄||²/λ + N S_dxdx)
//     zero denominator -> γ = 0 (c16)
//   The numerator's shared-vector term is taken at the base point from the coordinates, not from the
//   fp32 vector delta: Δw = Σ_k A_k Δx_k, so <r₀, Δr> = -Σ_m Δβ_m <a_m, r₀> and <Δw̄, w̄₀> =
//   Σ_n Δα_n <ā_n, w̄₀> (k_base_dot, fp64, one gather pass over the local matrix).  Near the optimum
//   the two terms of the numerator nearly cancel (<r₀, Δr> ≈ -λN<β₀, Δβ> when ∇P(β₀) ≈ 0), and the
//   vector delta carries the rounding of every fp32 RED of the epoch at the scale of |r| (~1e-6 per
//   entry on C4), which then dominated the difference and made γ erratic below gap ~1e-5.
//   sv = sv₀ + γΔ ;  x_k = x₀_k + γΔx_k ;  the result becomes the next base point (c6).
//
// Two implementations of the exchange:
//   NCCL   pack Δ_k, ncclAllReduce(Δ) + the worker scalars, dots, γ, apply (default for world > 1)
//   fused  over peer memory (the K logical workers of scd_aggregate_group on one device, and
//          world > 1 with SCD_P2P_AGG=1 through CUDA IPC over NVLink): each rank owns a shard of
//          the shared vector; k_agg_reduce reads every worker's sv for the shard and forms Δ and
//          the shard's <sv₀, Δ>, ||Δ||² in one pass (reduce-scatter fused with the dots);
//          after the scalar all-reduce and γ, k_agg_apply writes sv₀ + γΔ of the shard straight
//          into every worker's sv and sv₀ (all-gather fused with the axpy).
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace scd {
namespace {

constexpr int kT = 256;

// acc[0] += <x0, x - x0>, acc[1] += ||x - x0||², acc[2] += <y, x - x0> (dual only)
__global__ void __launch_bounds__(kT) k_model_dots(const float *x, const float *x0, const float *y, int64_t n,
                                                   int dual, double *acc) {
  double a = 0.0, b = 0.0, c = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)x[i] - (double)x0[i];
    a += (double)x0[i] * d;
    b += d * d;
    if (dual) c += (double)y[i] * d;
  }
  block_sum_atomic<kT>(a, acc + 0);
  block_sum_atomic<kT>(b, acc + 1);
  if (dual) block_sum_atomic<kT>(c, acc + 2);
}

// out = (first ? 0 : out) + (sv - sv0)
__global__ void k_delta(const float *sv, const float *sv0, int64_t n, int first, float *out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float d = sv[i] - sv0[i];
    out[i] = first ? d : out[i] + d;
  }
}

// acc[3] += <sv0, Δ>, acc[4] += ||Δ||²
__global__ void __launch_bounds__(kT) k_shared_dots(const float *sv0, const float *d, int64_t n, double *acc) {
  double a = 0.0, b = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double di = d[i];
    a += (double)sv0[i] * di;
    b += di * di;
  }
  block_sum_atomic<kT>(a, acc + 3);
  block_sum_atomic<kT>(b, acc + 4);
}

// acc[5] += Σ_c (x_c - x0_c) <a_c, sv0>: the base-point term of the optimal γ (fp64, warp per coordinate).
// primal: sv0 = r₀ and the term is -<r₀, Δr>; dual: sv0 = w̄₀ and the term is <Δw̄, w̄₀>.
__global__ void __launch_bounds__(kT) k_base_dot(const int64_t *ptr, const int32_t *idx, const float *val,
                                                 const float *x, const float *x0, const float *sv0, int64_t n,
                                                 double *acc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double s = 0.0;
  for (int64_t o = warp; o < n; o += nwarps) {
    const double dx = (double)x[o] - (double)x0[o];
    if (dx == 0.0) continue;  // warp-uniform
    double c = 0.0;
    for (int64_t k = ptr[o] + lane; k < ptr[o + 1]; k += 32) c += (double)val_at(val, k) * (double)sv0[idx[k]];
    s += dx * c;  // lanes' partials; summed below
  }
  block_sum_atomic<kT>(s, acc + 5);
}

__global__ void k_gamma(double *acc, int mode, int form, double K, double lam, double N) {
  double g;
  if (mode == SCD_AGG_ADD) {
    g = 1.0;
  } else if (mode == SCD_AGG_AVERAGE) {
    g = 1.0 / K;
  } else {
    const double lamN = lam * N;
    double num, den;
    // acc[5] = Σ Δx_c <a_c, sv0> replaces <sv0, Δ> (acc[3]) in the numerator (see the header)
    if (form == SCD_PRIMAL) {
      num = -(-acc[5] + lamN * acc[0]);
      den = acc[4] + lamN * acc[1];
    } else {
      num = acc[2] - N * acc[0] - acc[5] / lam;
      den = acc[4] / lam + N * acc[1];
    }
    g = den != 0.0 ? num / den : 0.0;
  }
  acc[8] = g;
}

__global__ void k_apply_shared(float *sv, float *sv0, const float *d, int64_t n, const double *acc) {
  const float g = (float)acc[8];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = sv0[i] + g * d[i];
    sv[i] = v;
    sv0[i] = v;
  }
}

// Fused reduce-scatter + dots: shard [lo, hi) of Δ = Σ_k (sv_k - sv₀) from every worker's sv
// (peer pointers), acc[3] += <sv₀, Δ>, acc[4] += ||Δ||² over the shard.
__global__ void __launch_bounds__(kT) k_agg_reduce(const float *const *peer_sv, int K, const float *sv0, int64_t lo,
                                                   int64_t hi, float *delta, double *acc) {
  double a = 0.0, b = 0.0;
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    const float base = sv0[i];
    float d = 0.f;
    for (int k = 0; k < K; ++k) d += __ldcg(peer_sv[k] + i) - base;
    delta[i] = d;
    a += (double)base * (double)d;
    b += (double)d * (double)d;
  }
  block_sum_atomic<kT>(a, acc + 3);
  block_sum_atomic<kT>(b, acc + 4);
}

// Fused axpy + all-gather: v = sv₀ + γΔ on shard [lo, hi), written into every worker's sv and sv₀.
__global__ void k_agg_apply(float *const *peer_sv, float *const *peer_sv0, int K, const float *sv0, const float *delta,
                            int64_t lo, int64_t hi, const double *acc) {
  const float g = (float)acc[8];
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = sv0[i] + g * delta[i];
    for (int k = 0; k < K; ++k) {
      __stcg(peer_sv[k] + i, v);
      __stcg(peer_sv0[k] + i, v);
    }
  }
  __threadfence_system();  // peer stores visible to the other GPUs before the next collective
}

__global__ void k_apply_model(float *x, float *x0, int64_t n, const double *acc) {
  const float g = (float)acc[8];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x0[i] + g * (x[i] - x0[i]);
    x[i] = v;
    x0[i] = v;
  }
}

}  // namespace

// Peer tables for the fused exchange across processes (world > 1): CUDA IPC handles of every
// rank's sv allocation (+ the offset of sv in it) and sv₀, exchanged with one ncclAllGather, opened
// with peer access.  Any failure leaves the NCCL path in place.
namespace {
struct IpcRec {
  cudaIpcMemHandle_t sv, sv0;
  int64_t sv_off;
  int32_t pad[2];
};

scd_status p2p_setup(scd_ctx *c) {
  c->p2p_state = -1;
  const int K = c->opt.world, r = c->opt.rank;
  IpcRec mine{};
  if (cudaIpcGetMemHandle(&mine.sv, c->sv_base) != cudaSuccess || cudaIpcGetMemHandle(&mine.sv0, c->sv0) != cudaSuccess) {
    cudaGetLastError();
    return SCD_OK;
  }
  mine.sv_off = (int64_t)(c->sv - c->sv_base);
  IpcRec *d_all = nullptr;
  SCD_CK(c, cudaMalloc((void **)&d_all, sizeof(IpcRec) * (size_t)(K + 1)));
  SCD_CK(c, cudaMemcpyAsync(d_all + K, &mine, sizeof(IpcRec), cudaMemcpyHostToDevice, c->stream));
  SCD_COLL(coll_allgather(c, d_all + K, d_all, sizeof(IpcRec)));
  std::vector<IpcRec> all((size_t)K);
  SCD_CK(c, cudaMemcpyAsync(all.data(), d_all, sizeof(IpcRec) * (size_t)K, cudaMemcpyDeviceToHost, c->stream));
  SCD_CK(c, cudaStreamSynchronize(c->stream));
  cudaFree(d_all);
  std::vector<float *> ptrs(2 * (size_t)K, nullptr);
  bool ok = true;
  for (int k = 0; k < K && ok; ++k) {
    if (k == r) {
      ptrs[(size_t)k] = c->sv;
      ptrs[(size_t)K + k] = c->sv0;
      continue;
    }
    void *a = nullptr, *b = nullptr;
    ok = cudaIpcOpenMemHandle(&a, all[(size_t)k].sv, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess &&
         cudaIpcOpenMemHandle(&b, all[(size_t)k].sv0, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    if (a) c->p2p_open.push_back(a);
    if (b) c->p2p_open.push_back(b);
    if (ok) {
      ptrs[(size_t)k] = reinterpret_cast<float *>(a) + all[(size_t)k].sv_off;
      ptrs[(size_t)K + k] = reinterpret_cast<float *>(b);
    }
  }
  // every rank must succeed, or all use the NCCL path
  int32_t *d_ok = nullptr;
  int32_t h_ok = ok ? 1 : 0;
  SCD_CK(c, cudaMalloc((void **)&d_ok, sizeof(int32_t)));
  SCD_CK(c, cudaMemcpyAsync(d_ok, &h_ok, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  SCD_COLL(coll_allreduce(c, d_ok, 1, SCD_DT_I32, SCD_OP_MIN));
  SCD_CK(c, cudaMemcpyAsync(&h_ok, d_ok, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  SCD_CK(c, cudaStreamSynchronize(c->stream));
  cudaFree(d_ok);
  if (!h_ok) {
    cudaGetLastError();
    for (void *p : c->p2p_open) cudaIpcCloseMemHandle(p);
    c->p2p_open.clear();
    return SCD_OK;
  }
  SCD_CK(c, cudaMalloc((void **)&c->p2p_ptrs, sizeof(float *) * 2 * (size_t)K));
  SCD_CK(c, cudaMemcpy(c->p2p_ptrs, ptrs.data(), sizeof(float *) * 2 * (size_t)K, cudaMemcpyHostToDevice));
  c->p2p_state = 1;
  return SCD_OK;
}
}  // namespace

// world > 1, fused exchange over peer memory (SCD_P2P_AGG=1).  Barriers are the scalar collectives:
// (1) all-reduce of the model scalars — every rank's epoch is done before any rank reads its sv;
// (2) all-reduce of the shard dots — every shard's Δ is formed before any rank overwrites sv/sv₀;
// (3) a one-word all-reduce — every rank's stores into this rank's sv/sv₀ are complete before its
// next epoch.
static scd_status aggregate_p2p(scd_ctx *c, scd_agg mode, double *gamma) {
  cudaStream_t s = c->stream;
  const int dual = c->form == SCD_DUAL;
  const int64_t ns = c->n_shared, nc = c->n_coord;
  const int K = c->opt.world, r = c->opt.rank;
  const int64_t lo = ns * r / K, hi = ns * (r + 1) / K;
  float **peer = c->p2p_ptrs;
  SCD_CK(c, cudaMemsetAsync(c->acc, 0, sizeof(double) * 16, s));
  k_model_dots<<<grid_for(nc, kT), kT, 0, s>>>(c->x, c->x0, c->y, nc, dual, c->acc);
  if (mode == SCD_AGG_OPTIMAL)
    k_base_dot<<<grid_for(nc * 32, kT, 148 * 32), kT, 0, s>>>(c->ptr, c->idx, c->val, c->x, c->x0, c->sv0, nc, c->acc);
  SCD_COLL(coll_allreduce(c, c->acc, 6, SCD_DT_F64, SCD_OP_SUM));  // acc[3..4] are still 0 here
  k_agg_reduce<<<grid_for(hi - lo, kT), kT, 0, s>>>(peer, K, c->sv0, lo, hi, c->comm, c->acc);
  SCD_COLL(coll_allreduce(c, c->acc + 3, 2, SCD_DT_F64, SCD_OP_SUM));
  k_gamma<<<1, 1, 0, s>>>(c->acc, (int)mode, (int)c->form, (double)K, c->lam, (double)c->n_global);
  k_agg_apply<<<grid_for(hi - lo, kT), kT, 0, s>>>(peer, peer + K, K, c->sv0, c->comm, lo, hi, c->acc);
  SCD_COLL(coll_allreduce(c, c->acc + 9, 1, SCD_DT_F64, SCD_OP_SUM));
  k_apply_model<<<grid_for(nc, kT), kT, 0, s>>>(c->x, c->x0, nc, c->acc);
  SCD_CKL(c, "aggregate (fused peer exchange)");
  c->launches += 5 + (mode == SCD_AGG_OPTIMAL ? 1 : 0);
  c->empty_dirty = true;  // x₀ + γΔx moved the empty coordinates off their fixed point (c17)
  double g = 0.0;
  SCD_CK(c, cudaMemcpyAsync(&g, c->acc + 8, sizeof(double), cudaMemcpyDeviceToHost, s));
  SCD_CK(c, cudaStreamSynchronize(s));
  if (gamma) *gamma = g;
  return SCD_OK;
}

scd_status aggregate(scd_ctx *c, scd_agg mode, double *gamma) {
  // (a 1-rank communicator runs the same fused path: IPC export, handle all-gather, barriers)
  if (c->has_comm() && getenv("SCD_P2P_AGG") && atoi(getenv("SCD_P2P_AGG")) == 1) {
    if (c->p2p_state == 0) {
      scd_status st = p2p_setup(c);
      if (st != SCD_OK) return st;
    }
    if (c->p2p_state == 1) return aggregate_p2p(c, mode, gamma);
  }
  cudaStream_t s = c->stream;
  const int dual = c->form == SCD_DUAL;
  // the dual's w̄ is zero beyond the largest inner index of every rank's shard, so Δ is too: the
  // round exchanges [0, sv_active) only (exact; C3: 680 715 of 16.6 M entries), the extent being the
  // max over the ranks, reduced once
  if (dual && c->has_comm() && c->opt.world > 1 && !c->sv_active_global) {
    int64_t *d = nullptr, h = c->sv_active;
    SCD_CK(c, cudaMallocAsync((void **)&d, sizeof(int64_t), s));
    SCD_CK(c, cudaMemcpyAsync(d, &h, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SCD_COLL(coll_allreduce(c, d, 1, SCD_DT_I64, SCD_OP_MAX));
    SCD_CK(c, cudaMemcpyAsync(&h, d, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SCD_CK(c, cudaStreamSynchronize(s));
    cudaFreeAsync(d, s);
    c->sv_active = std::max<int64_t>(1, std::min<int64_t>(h, c->n_shared));
  }
  c->sv_active_global = true;
  const int64_t ns = (dual && c->sv_active > 0) ? c->sv_active : c->n_shared, nc = c->n_coord;
  SCD_CK(c, cudaMemsetAsync(c->acc, 0, sizeof(double) * 16, s));
  k_model_dots<<<grid_for(nc, kT), kT, 0, s>>>(c->x, c->x0, c->y, nc, dual, c->acc);
  if (mode == SCD_AGG_OPTIMAL) {
    k_base_dot<<<grid_for(nc * 32, kT, 148 * 32), kT, 0, s>>>(c->ptr, c->idx, c->val, c->x, c->x0, c->sv0, nc, c->acc);
    ++c->launches;
  }
  k_delta<<<grid_for(ns, kT), kT, 0, s>>>(c->sv, c->sv0, ns, 1, c->comm);
  SCD_CKL(c, "aggregate pack");
  c->launches += 2;
  if (c->has_comm()) {  // collective whenever a communicator is attached (world = 1 exercises the same path)
    // Σ_k Δw_k (Alg. 3/4 "Aggregate updates") and the worker scalars
    SCD_COLL(coll_group_start(c));
    SCD_COLL(coll_allreduce(c, c->comm, (size_t)ns, SCD_DT_F32, SCD_OP_SUM));
    SCD_COLL(coll_allreduce(c, c->acc, 6, SCD_DT_F64, SCD_OP_SUM));  // acc[3..4] are still 0 here
    SCD_COLL(coll_group_end(c));
  }
  {
    // <sv0, Δ> and ||Δ||² over the replicated vectors: each rank sums its 1/K shard and the partial
    // sums are all-reduced, so every rank derives the bit-identical γ (a rank-local sum of the whole
    // vector rounds differently from rank to rank: fp64 atomics in block_sum_atomic)
    const int K = c->has_comm() ? c->opt.world : 1, r = c->has_comm() ? c->opt.rank : 0;
    const int64_t lo = ns * r / K, hi = ns * (r + 1) / K;
    k_shared_dots<<<grid_for(std::max<int64_t>(hi - lo, 1), kT), kT, 0, s>>>(c->sv0 + lo, c->comm + lo, hi - lo, c->acc);
    if (c->has_comm() && K > 1) SCD_COLL(coll_allreduce(c, c->acc + 3, 2, SCD_DT_F64, SCD_OP_SUM));
  }
  k_gamma<<<1, 1, 0, s>>>(c->acc, (int)mode, (int)c->form, (double)c->opt.world, c->lam, (double)c->n_global);
  k_apply_shared<<<grid_for(ns, kT), kT, 0, s>>>(c->sv, c->sv0, c->comm, ns, c->acc);
  k_apply_model<<<grid_for(nc, kT), kT, 0, s>>>(c->x, c->x0, nc, c->acc);
  SCD_CKL(c, "aggregate apply");
  c->launches += 4;
  c->empty_dirty = true;  // x₀ + γΔx moved the empty coordinates off their fixed point (c17)
  double g = 0.0;
  SCD_CK(c, cudaMemcpyAsync(&g, c->acc + 8, sizeof(double), cudaMemcpyDeviceToHost, s));
  SCD_CK(c, cudaStreamSynchronize(s));
  if (gamma) *gamma = g;
  return SCD_OK;
}

// k logical workers on one device: the fused peer-memory kernels with the k contexts as the peers
// and one shard (the whole vector).
scd_status aggregate_group(scd_ctx *const *cs, int32_t k, scd_agg mode, double *gamma) {
  scd_ctx *c0 = cs[0];
  for (int i = 0; i < k; ++i) SCD_CK(cs[i], cudaStreamSynchronize(cs[i]->stream));
  cudaStream_t s = c0->stream;
  const int dual = c0->form == SCD_DUAL;
  const int64_t ns = c0->n_shared;
  std::vector<float *> ptrs(2 * (size_t)k);
  for (int i = 0; i < k; ++i) {
    ptrs[(size_t)i] = cs[i]->sv;
    ptrs[(size_t)k + i] = cs[i]->sv0;
  }
  float **d_ptrs = nullptr;
  SCD_CK(c0, cudaMallocAsync((void **)&d_ptrs, sizeof(float *) * 2 * (size_t)k, s));
  SCD_CK(c0, cudaMemcpyAsync(d_ptrs, ptrs.data(), sizeof(float *) * 2 * (size_t)k, cudaMemcpyHostToDevice, s));
  SCD_CK(c0, cudaMemsetAsync(c0->acc, 0, sizeof(double) * 16, s));
  for (int i = 0; i < k; ++i) {
    scd_ctx *c = cs[i];
    k_model_dots<<<grid_for(c->n_coord, kT), kT, 0, s>>>(c->x, c->x0, c->y, c->n_coord, dual, c0->acc);
    if (mode == SCD_AGG_OPTIMAL) {  // each worker's coordinates against the common base point
      k_base_dot<<<grid_for(c->n_coord * 32, kT, 148 * 32), kT, 0, s>>>(c->ptr, c->idx, c->val, c->x, c->x0, c0->sv0,
                                                                         c->n_coord, c0->acc);
      c->launches += 1;
    }
    c->launches += 1;
  }
  k_agg_reduce<<<grid_for(ns, kT), kT, 0, s>>>(d_ptrs, k, c0->sv0, 0, ns, c0->comm, c0->acc);
  k_gamma<<<1, 1, 0, s>>>(c0->acc, (int)mode, (int)c0->form, (double)k, c0->lam, (double)c0->n_global);
  k_agg_apply<<<grid_for(ns, kT), kT, 0, s>>>(d_ptrs, d_ptrs + k, k, c0->sv0, c0->comm, 0, ns, c0->acc);
  c0->launches += 3;
  for (int i = 0; i < k; ++i) {
    scd_ctx *c = cs[i];
    k_apply_model<<<grid_for(c->n_coord, kT), kT, 0, s>>>(c->x, c->x0, c->n_coord, c0->acc);
    c->launches += 1;
    c->empty_dirty = true;  // x₀ + γΔx moved the empty coordinates off their fixed point (c17)
  }
  SCD_CKL(c0, "aggregate_group kernels");
  cudaFreeAsync(d_ptrs, s);
  double g = 0.0;
  SCD_CK(c0, cudaMemcpyAsync(&g, c0->acc + 8, sizeof(double), cudaMemcpyDeviceToHost, s));
  SCD_CK(c0, cudaStreamSynchronize(s));
  if (gamma) *gamma = g;
  return SCD_OK;
}

}  // namespace scd
