// evaluate.cu — fp64 objective / duality-gap evaluation from scratch (§II.C) and the
// shared-vector rebuild.  Never trusts the incrementally maintained shared vector.
//
// primal (CSC, model β):  u = Aβ (fp64 scatter) [+ all-reduce], res = y - u,
//   P(β)   = ||res||²/(2N) + λ/2 ||β||²                              Eq. (1)
//   D(α̂)   with α̂ = res/N  (Eq. 6), Aᵀα̂ = g/N, g_m = <a_m, res>   Eq. (3)
//   G_P    = ||λβ - g/N||²/(2λ) = ||∇P(β)||²/(2λ)                      (c13)
// dual (CSR, model α):  v = Aᵀα (fp64 scatter) [+ all-reduce], q_n = <ā_n, v>,
//   P(β̂)   with β̂ = v/λ (Eq. 5): ||q/λ - y||²/(2N) + ||v||²/(2λ)
//   D(α)   = -N/2||α||² - ||v||²/(2λ) + αᵀy
//   G_D    = ||y - Nα - q/λ||²/(2N) = ||∇D(α)||²/(2N)                   (c13)
#include <algorithm>

#include "common.cuh"

namespace scd {
namespace {

constexpr int kT = 256;

// out[idx[k]] += val[k] * x[o] for every outer o (fp64 atomics); warp per outer index.
__global__ void k_scatter64(const int64_t *ptr, const int32_t *idx, const float *val, const float *x, int64_t outer,
                            double *out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t o = warp; o < outer; o += nwarps) {
    const double xo = x[o];
    if (xo == 0.0) continue;
    for (int64_t k = ptr[o] + lane; k < ptr[o + 1]; k += 32) atomicAdd(out + idx[k], (double)val_at(val, k) * xo);
  }
}

// primal rows: res_i = y_i - u_i, acc[0] += res², acc[1] += y·res  (u = Aβ is kept: the shared-vector
// rebuild may reuse it, see shared64)
__global__ void __launch_bounds__(kT) k_primal_rows(const float *y, const double *u, int64_t n, double *acc) {
  double s_rr = 0.0, s_yr = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double r = (double)y[i] - u[i];
    s_rr += r * r;
    s_yr += (double)y[i] * r;
  }
  block_sum_atomic<kT>(s_rr, acc + 0);
  block_sum_atomic<kT>(s_yr, acc + 1);
}

// primal columns: g_m = <a_m, res>, res = y - u; acc[2] += (λβ_m - g_m/N)², acc[3] += β_m², acc[4] += g_m²
__global__ void __launch_bounds__(kT) k_primal_cols(const int64_t *ptr, const int32_t *idx, const float *val,
                                                    const float *beta, const float *y, const double *u, int64_t outer,
                                                    double lam, double N, double *acc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double s_gg = 0.0, s_bb = 0.0, s_g2 = 0.0;
  for (int64_t o = warp; o < outer; o += nwarps) {
    double g = 0.0;
    for (int64_t k = ptr[o] + lane; k < ptr[o + 1]; k += 32) {
      const int32_t i = idx[k];
      g += (double)val_at(val, k) * ((double)y[i] - u[i]);
    }
    g = warp_sum(g);
    if (lane == 0) {
      const double b = beta[o];
      const double gr = lam * b - g / N;
      s_gg += gr * gr;
      s_bb += b * b;
      s_g2 += g * g;
    }
  }
  block_sum_atomic<kT>(s_gg, acc + 2);
  block_sum_atomic<kT>(s_bb, acc + 3);
  block_sum_atomic<kT>(s_g2, acc + 4);
}

// acc[slot] += Σ v_i²
__global__ void __launch_bounds__(kT) k_sumsq64(const double *v, int64_t n, double *acc) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += v[i] * v[i];
  block_sum_atomic<kT>(s, acc);
}

// dual rows: q_n = <ā_n, v>; acc[1] += (q_n/λ - y_n)², acc[2] += (y_n - Nα_n - q_n/λ)², acc[3] += α_n², acc[4] += α_n y_n
__global__ void __launch_bounds__(kT) k_dual_rows(const int64_t *ptr, const int32_t *idx, const float *val,
                                                  const float *alpha, const float *y, const double *v, int64_t outer,
                                                  double lam, double N, double *acc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double s_res = 0.0, s_gg = 0.0, s_aa = 0.0, s_ay = 0.0;
  for (int64_t o = warp; o < outer; o += nwarps) {
    double q = 0.0;
    for (int64_t k = ptr[o] + lane; k < ptr[o + 1]; k += 32) q += (double)val_at(val, k) * v[idx[k]];
    q = warp_sum(q);
    if (lane == 0) {
      const double a = alpha[o], yo = y[o];
      const double p = q / lam;
      s_res += (p - yo) * (p - yo);
      const double g = yo - N * a - p;
      s_gg += g * g;
      s_aa += a * a;
      s_ay += a * yo;
    }
  }
  block_sum_atomic<kT>(s_res, acc + 1);
  block_sum_atomic<kT>(s_gg, acc + 2);
  block_sum_atomic<kT>(s_aa, acc + 3);
  block_sum_atomic<kT>(s_ay, acc + 4);
}

__global__ void k_resid_to_f32(const float *y, const double *u, int64_t n, float *r) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = (float)((double)y[i] - u[i]);
}
__global__ void k_f64_to_f32(const double *u, int64_t n, float *r) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = (float)u[i];
}
__global__ void k_w_from_r(const float *y, const float *r, int64_t n, float *w) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = y[i] - r[i];
}

}  // namespace

// u = A x (primal: Aβ over N rows) or v = Aᵀx (dual: over M cols) into c->vec64, summed over ranks
// (collective).  The gap pass and the shared-vector rebuild (NEXT-2) both start from it, so
// the scatter runs once per model: it is skipped while vec64 still belongs to the current model
// (every rank bumps model_version identically, so all skip or none does).
static scd_status shared64(scd_ctx *c) {
  if (c->vec64_version == c->model_version) return SCD_OK;
  cudaStream_t s = c->stream;
  SCD_CK(c, cudaMemsetAsync(c->vec64, 0, sizeof(double) * (size_t)c->n_shared, s));
  k_scatter64<<<grid_for(c->n_coord * 32, kT, 148 * 32), kT, 0, s>>>(c->ptr, c->idx, c->val, c->x, c->n_coord,
                                                                      c->vec64);
  SCD_CKL(c, "k_scatter64");
  ++c->launches;
  if (c->has_comm()) SCD_COLL(coll_allreduce(c, c->vec64, (size_t)c->n_shared, SCD_DT_F64, SCD_OP_SUM));
  c->vec64_version = c->model_version;
  return SCD_OK;
}

scd_status evaluate(scd_ctx *c, double *primal, double *dual, double *gap) {
  cudaStream_t s = c->stream;
  scd_status st = shared64(c);
  if (st != SCD_OK) return st;
  SCD_CK(c, cudaMemsetAsync(c->acc, 0, sizeof(double) * 8, s));
  const double N = (double)c->n_global, lam = c->lam;
  double h[8] = {0};
  if (c->form == SCD_PRIMAL) {
    // rows are replicated across the feature-partitioned workers: each rank sums its 1/K shard of them
    // and everything is all-reduced once (every rank then holds bit-identical results)
    const int K = c->has_comm() ? c->opt.world : 1, r = c->has_comm() ? c->opt.rank : 0;
    const int64_t lo = c->n_shared * r / K, hi = c->n_shared * (r + 1) / K;
    k_primal_rows<<<grid_for(std::max<int64_t>(hi - lo, 1), kT, 148 * 8), kT, 0, s>>>(c->y + lo, c->vec64 + lo, hi - lo,
                                                                                    c->acc);
    k_primal_cols<<<grid_for(c->n_coord * 32, kT, 148 * 32), kT, 0, s>>>(c->ptr, c->idx, c->val, c->x, c->y,
                                                                          c->vec64, c->n_coord, lam, N, c->acc);
    SCD_CKL(c, "primal evaluate kernels");
    c->launches += 2;
    if (c->has_comm()) SCD_COLL(coll_allreduce(c, c->acc, 5, SCD_DT_F64, SCD_OP_SUM));
    SCD_CK(c, cudaMemcpyAsync(h, c->acc, sizeof(double) * 8, cudaMemcpyDeviceToHost, s));
    SCD_CK(c, cudaStreamSynchronize(s));
    const double P = h[0] / (2.0 * N) + 0.5 * lam * h[3];
    const double D = -0.5 * N * (h[0] / (N * N)) - (h[4] / (N * N)) / (2.0 * lam) + h[1] / N;
    if (primal) *primal = P;
    if (dual) *dual = D;
    if (gap) *gap = h[2] / (2.0 * lam);
  } else {
    // v is replicated across the example-partitioned workers: each rank sums ||v||² over its 1/K shard
    const int K = c->has_comm() ? c->opt.world : 1, r = c->has_comm() ? c->opt.rank : 0;
    const int64_t lo = c->n_shared * r / K, hi = c->n_shared * (r + 1) / K;
    k_sumsq64<<<grid_for(std::max<int64_t>(hi - lo, 1), kT, 148 * 8), kT, 0, s>>>(c->vec64 + lo, hi - lo, c->acc + 0);
    k_dual_rows<<<grid_for(c->n_coord * 32, kT, 148 * 32), kT, 0, s>>>(c->ptr, c->idx, c->val, c->x, c->y, c->vec64,
                                                                        c->n_coord, lam, N, c->acc);
    SCD_CKL(c, "dual evaluate kernels");
    c->launches += 2;
    if (c->has_comm()) SCD_COLL(coll_allreduce(c, c->acc, 5, SCD_DT_F64, SCD_OP_SUM));
    SCD_CK(c, cudaMemcpyAsync(h, c->acc, sizeof(double) * 8, cudaMemcpyDeviceToHost, s));
    SCD_CK(c, cudaStreamSynchronize(s));
    const double P = h[1] / (2.0 * N) + h[0] / (2.0 * lam);
    const double D = -0.5 * N * h[3] - h[0] / (2.0 * lam) + h[4];
    if (primal) *primal = P;
    if (dual) *dual = D;
    if (gap) *gap = h[2] / (2.0 * N);
  }
  return SCD_OK;
}

// The same evaluation for k logical workers on one device (scd_aggregate_group's setting): the
// shard scatters are summed into ctx 0's fp64 vector (the all-reduce), per-shard partial sums go
// into ctx 0's accumulators; replicated quantities are computed once.
scd_status evaluate_group(scd_ctx *const *cs, int32_t k, double *primal, double *dual, double *gap) {
  scd_ctx *c0 = cs[0];
  for (int i = 0; i < k; ++i) SCD_CK(cs[i], cudaStreamSynchronize(cs[i]->stream));
  cudaStream_t s = c0->stream;
  SCD_CK(c0, cudaMemsetAsync(c0->vec64, 0, sizeof(double) * (size_t)c0->n_shared, s));
  c0->vec64_version = 0;  // now the group's sum, not ctx 0's own A x
  SCD_CK(c0, cudaMemsetAsync(c0->acc, 0, sizeof(double) * 8, s));
  for (int i = 0; i < k; ++i) {
    scd_ctx *c = cs[i];
    k_scatter64<<<grid_for(c->n_coord * 32, kT, 148 * 32), kT, 0, s>>>(c->ptr, c->idx, c->val, c->x, c->n_coord,
                                                                        c0->vec64);
    ++c->launches;
  }
  const double N = (double)c0->n_global, lam = c0->lam;
  double h[8] = {0};
  if (c0->form == SCD_PRIMAL) {
    k_primal_rows<<<grid_for(c0->n_shared, kT, 148 * 8), kT, 0, s>>>(c0->y, c0->vec64, c0->n_shared, c0->acc);
    for (int i = 0; i < k; ++i) {
      scd_ctx *c = cs[i];
      k_primal_cols<<<grid_for(c->n_coord * 32, kT, 148 * 32), kT, 0, s>>>(c->ptr, c->idx, c->val, c->x, c0->y,
                                                                            c0->vec64, c->n_coord, lam, N, c0->acc);
    }
  } else {
    k_sumsq64<<<grid_for(c0->n_shared, kT, 148 * 8), kT, 0, s>>>(c0->vec64, c0->n_shared, c0->acc + 0);
    for (int i = 0; i < k; ++i) {
      scd_ctx *c = cs[i];
      k_dual_rows<<<grid_for(c->n_coord * 32, kT, 148 * 32), kT, 0, s>>>(c->ptr, c->idx, c->val, c->x, c->y,
                                                                          c0->vec64, c->n_coord, lam, N, c0->acc);
    }
  }
  SCD_CKL(c0, "evaluate_group kernels");
  SCD_CK(c0, cudaMemcpyAsync(h, c0->acc, sizeof(double) * 8, cudaMemcpyDeviceToHost, s));
  SCD_CK(c0, cudaStreamSynchronize(s));
  if (c0->form == SCD_PRIMAL) {
    if (primal) *primal = h[0] / (2.0 * N) + 0.5 * lam * h[3];
    if (dual) *dual = -0.5 * N * (h[0] / (N * N)) - (h[4] / (N * N)) / (2.0 * lam) + h[1] / N;
    if (gap) *gap = h[2] / (2.0 * lam);
  } else {
    if (primal) *primal = h[1] / (2.0 * N) + h[0] / (2.0 * lam);
    if (dual) *dual = -0.5 * N * h[3] - h[0] / (2.0 * lam) + h[4];
    if (gap) *gap = h[2] / (2.0 * N);
  }
  return SCD_OK;
}

// Shared vector from the model (fp64 accumulate, one rounding to fp32); resets the base point.
scd_status rebuild_shared(scd_ctx *c) {
  cudaStream_t s = c->stream;
  scd_status st = shared64(c);
  if (st != SCD_OK) return st;
  if (c->form == SCD_PRIMAL)
    k_resid_to_f32<<<grid_for(c->n_shared, kT), kT, 0, s>>>(c->y, c->vec64, c->n_shared, c->sv);
  else
    k_f64_to_f32<<<grid_for(c->n_shared, kT), kT, 0, s>>>(c->vec64, c->n_shared, c->sv);
  SCD_CKL(c, "rebuild_shared");
  SCD_CK(c, cudaMemcpyAsync(c->sv0, c->sv, sizeof(float) * (size_t)c->n_shared, cudaMemcpyDeviceToDevice, s));
  SCD_CK(c, cudaMemcpyAsync(c->x0, c->x, sizeof(float) * (size_t)c->n_coord, cudaMemcpyDeviceToDevice, s));
  return SCD_OK;
}

// w = y - r (primal) into d_out; the dual's shared vector is w̄ itself.
scd_status shared_to_w(scd_ctx *c, float *d_out) {
  if (c->form == SCD_PRIMAL) {
    k_w_from_r<<<grid_for(c->n_shared, kT), kT, 0, c->stream>>>(c->y, c->sv, c->n_shared, d_out);
    SCD_CKL(c, "k_w_from_r");
  } else {
    SCD_CK(c, cudaMemcpyAsync(d_out, c->sv, sizeof(float) * (size_t)c->n_shared, cudaMemcpyDeviceToDevice, c->stream));
  }
  return SCD_OK;
}

}  // namespace scd
