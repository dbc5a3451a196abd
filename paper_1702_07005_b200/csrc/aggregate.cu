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
//   sv = sv₀ + γΔ ;  x_k = x₀_k + γΔx_k ;  the result becomes the next base point (c6).
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

__global__ void k_gamma(double *acc, int mode, int form, double K, double lam, double N) {
  double g;
  if (mode == SCD_AGG_ADD) {
    g = 1.0;
  } else if (mode == SCD_AGG_AVERAGE) {
    g = 1.0 / K;
  } else {
    const double lamN = lam * N;
    double num, den;
    if (form == SCD_PRIMAL) {
      num = -(acc[3] + lamN * acc[0]);
      den = acc[4] + lamN * acc[1];
    } else {
      num = acc[2] - N * acc[0] - acc[3] / lam;
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

__global__ void k_apply_model(float *x, float *x0, int64_t n, const double *acc) {
  const float g = (float)acc[8];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x0[i] + g * (x[i] - x0[i]);
    x[i] = v;
    x0[i] = v;
  }
}

}  // namespace

scd_status aggregate(scd_ctx *c, scd_agg mode, double *gamma) {
  cudaStream_t s = c->stream;
  const int dual = c->form == SCD_DUAL;
  const int64_t ns = c->n_shared, nc = c->n_coord;
  SCD_CK(c, cudaMemsetAsync(c->acc, 0, sizeof(double) * 16, s));
  k_model_dots<<<grid_for(nc, kT), kT, 0, s>>>(c->x, c->x0, c->y, nc, dual, c->acc);
  k_delta<<<grid_for(ns, kT), kT, 0, s>>>(c->sv, c->sv0, ns, 1, c->comm);
  SCD_CKL(c, "aggregate pack");
  c->launches += 2;
  if (c->nccl) {  // collective whenever a communicator is attached (world = 1 exercises the same path)
    // Σ_k Δw_k (Alg. 3/4 "Aggregate updates") and the worker scalars
    SCD_NCK(c, ncclGroupStart());
    SCD_NCK(c, ncclAllReduce(c->comm, c->comm, (size_t)ns, ncclFloat, ncclSum, c->nccl, s));
    SCD_NCK(c, ncclAllReduce(c->acc, c->acc, 3, ncclDouble, ncclSum, c->nccl, s));
    SCD_NCK(c, ncclGroupEnd());
  }
  k_shared_dots<<<grid_for(ns, kT), kT, 0, s>>>(c->sv0, c->comm, ns, c->acc);
  k_gamma<<<1, 1, 0, s>>>(c->acc, (int)mode, (int)c->form, (double)c->opt.world, c->lam, (double)c->n_global);
  k_apply_shared<<<grid_for(ns, kT), kT, 0, s>>>(c->sv, c->sv0, c->comm, ns, c->acc);
  k_apply_model<<<grid_for(nc, kT), kT, 0, s>>>(c->x, c->x0, nc, c->acc);
  SCD_CKL(c, "aggregate apply");
  c->launches += 4;
  double g = 0.0;
  SCD_CK(c, cudaMemcpyAsync(&g, c->acc + 8, sizeof(double), cudaMemcpyDeviceToHost, s));
  SCD_CK(c, cudaStreamSynchronize(s));
  if (gamma) *gamma = g;
  return SCD_OK;
}

// k logical workers on one device: the "all-reduce" is a device-side sum into ctx[0]'s buffers.
scd_status aggregate_group(scd_ctx *const *cs, int32_t k, scd_agg mode, double *gamma) {
  scd_ctx *c0 = cs[0];
  for (int i = 0; i < k; ++i) SCD_CK(cs[i], cudaStreamSynchronize(cs[i]->stream));
  cudaStream_t s = c0->stream;
  const int dual = c0->form == SCD_DUAL;
  const int64_t ns = c0->n_shared;
  SCD_CK(c0, cudaMemsetAsync(c0->acc, 0, sizeof(double) * 16, s));
  for (int i = 0; i < k; ++i) {
    scd_ctx *c = cs[i];
    k_model_dots<<<grid_for(c->n_coord, kT), kT, 0, s>>>(c->x, c->x0, c->y, c->n_coord, dual, c0->acc);
    k_delta<<<grid_for(ns, kT), kT, 0, s>>>(c->sv, c->sv0, ns, i == 0, c0->comm);
    c->launches += 2;
  }
  k_shared_dots<<<grid_for(ns, kT), kT, 0, s>>>(c0->sv0, c0->comm, ns, c0->acc);
  k_gamma<<<1, 1, 0, s>>>(c0->acc, (int)mode, (int)c0->form, (double)k, c0->lam, (double)c0->n_global);
  for (int i = 0; i < k; ++i) {
    scd_ctx *c = cs[i];
    k_apply_shared<<<grid_for(ns, kT), kT, 0, s>>>(c->sv, c->sv0, c0->comm, ns, c0->acc);
    k_apply_model<<<grid_for(c->n_coord, kT), kT, 0, s>>>(c->x, c->x0, c->n_coord, c0->acc);
    c->launches += 2;
  }
  SCD_CKL(c0, "aggregate_group kernels");
  double g = 0.0;
  SCD_CK(c0, cudaMemcpyAsync(&g, c0->acc + 8, sizeof(double), cudaMemcpyDeviceToHost, s));
  SCD_CK(c0, cudaStreamSynchronize(s));
  if (gamma) *gamma = g;
  return SCD_OK;
}

}  // namespace scd
