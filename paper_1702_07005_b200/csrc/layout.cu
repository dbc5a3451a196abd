// layout.cu — create-time plumbing on the device: matrix validation, squared norms, the
// asynchronous coordinate schedule (length bins), and the stable CSR<->CSC transpose.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>

#include "common.cuh"

namespace scd {
namespace {

// Matrix invariants (SPEC S:29-31 restated in scd.h): ptr[0] = 0, nondecreasing, ptr[outer] = nnz;
// inner indices in range and strictly increasing per outer index.  *bad = first bad outer index.
__global__ void k_validate(const int64_t *ptr, const int32_t *idx, int64_t outer, int64_t inner, int64_t nnz,
                           unsigned long long *bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t o = warp; o < outer; o += nwarps) {
    const int64_t beg = ptr[o], end = ptr[o + 1];
    bool ok = beg <= end && beg >= 0 && end <= nnz;
    if (o == 0 && beg != 0) ok = false;
    if (o == outer - 1 && end != nnz) ok = false;
    if (ok) {
      for (int64_t k = beg + lane; k < end; k += 32) {
        const int32_t i = idx[k];
        if (i < 0 || i >= inner) ok = false;
        if (k > beg && idx[k - 1] >= i) ok = false;
      }
    }
    ok = __all_sync(0xffffffffu, ok);
    if (!ok && lane == 0) atomicMin(bad, (unsigned long long)o);
  }
}

// ||a||² of every outer index: fp64 accumulation in storage order per lane, rounded to fp32 (c9).
__global__ void k_norms(const int64_t *ptr, const float *val, int64_t outer, float *out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t o = warp; o < outer; o += nwarps) {
    double s = 0.0;
    for (int64_t k = ptr[o] + lane; k < ptr[o + 1]; k += 32) {
      const double v = val_at(val, k);
      s += v * v;
    }
    s = warp_sum(s);
    if (lane == 0) out[o] = (float)s;
  }
}

// transpose helpers
__global__ void k_outer_of(const int64_t *ptr, int64_t outer, int32_t *outer_of) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t o = warp; o < outer; o += nwarps)
    for (int64_t k = ptr[o] + lane; k < ptr[o + 1]; k += 32) outer_of[k] = (int32_t)o;
}
__global__ void k_iota64(int64_t *p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = i;
}
__global__ void k_count(const int32_t *keys, int64_t n, unsigned long long *cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + keys[i] + 1, 1ull);
}
__global__ void k_gather_t(const int64_t *perm, const int32_t *outer_of, const float *val, int64_t n, int32_t *oidx,
                           float *oval) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = perm[i];
    oidx[i] = outer_of[e];
    if (val) oval[i] = val[e];  // implicit-value input -> implicit-value output
  }
}

// s[idx[k]] += |val[k]|  (s = |A|ᵀ1 for CSR, |A|1 for CSC), fp64
// s[idx[k]] += |val[k]| over the coordinates of a bin (s = |A_b|ᵀ1 for CSR, |A_b|1 for CSC), fp64;
// acc[1] += Σ_bin ||a||² (from the fp32 norms)
__global__ void k_abs_scatter(const int64_t *ptr, const int32_t *idx, const float *val, const int32_t *list,
                              int64_t count, const float *norm, double *s, double *acc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < count; j += nwarps) {
    const int64_t o = list ? list[j] : j;
    for (int64_t k = ptr[o] + lane; k < ptr[o + 1]; k += 32) atomicAdd(s + idx[k], (double)fabsf(val_at(val, k)));
    if (lane == 0) atomicAdd(acc + 1, (double)norm[o]);
  }
}
// Tail part of the same sum: s[idx[k]] += |val[k]| for idx[k] >= lo only; acc[2] += Σ val² of those
// entries (their diagonal terms), acc[1] += Σ_bin ||a||² as above
__global__ void k_abs_scatter_tail(const int64_t *ptr, const int32_t *idx, const float *val, const int32_t *list,
                                   int64_t count, const float *norm, int32_t lo, double *s, double *acc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double sq = 0.0;
  for (int64_t j = warp; j < count; j += nwarps) {
    const int64_t o = list ? list[j] : j;
    for (int64_t k = ptr[o] + lane; k < ptr[o + 1]; k += 32) {
      const int32_t i = idx[k];
      if (i < lo) continue;
      const double v = (double)val_at(val, k);
      atomicAdd(s + i, fabs(v));
      sq += v * v;
    }
    if (lane == 0) atomicAdd(acc + 1, (double)norm[o]);
  }
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane == 0 && sq != 0.0) atomicAdd(acc + 2, sq);
}
// acc[0] += Σ s_i²
__global__ void __launch_bounds__(256) k_sumsq(const double *s, int64_t n, double *acc) {
  double a = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a += s[i] * s[i];
  block_sum_atomic<256>(a, acc + 0);
}


// number of stored entries with inner index < H (sizing the head-combining kernel)
__global__ void __launch_bounds__(256) k_count_below(const int32_t *idx, int64_t n, int32_t H, unsigned long long *out) {
  unsigned long long cnt = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    cnt += __ldcs(idx + i) < H;
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, cnt);
}

__global__ void __launch_bounds__(256) k_max_idx(const int32_t *idx, int64_t n, int *out) {
  int m = -1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, __ldcs(idx + i));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// sort key of inner index j: occurrences descending, then j ascending (a strict total order)
__global__ void k_rank_keys(const unsigned long long *cnt, int64_t inner, unsigned long long *key) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < inner; j += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long c = cnt[j + 1];  // k_count layout: cnt[j + 1] = occurrences of j
    key[j] = ((0xFFFFFFFFull - (c > 0xFFFFFFFFull ? 0xFFFFFFFFull : c)) << 32) | (unsigned long long)j;
  }
}
__global__ void k_rank_scatter(const unsigned long long *key_sorted, int64_t inner, int32_t *new_of_old) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < inner; r += (int64_t)gridDim.x * blockDim.x)
    new_of_old[key_sorted[r] & 0xFFFFFFFFull] = (int32_t)r;
}
__global__ void k_relabel(const int32_t *idx, int64_t n, const int32_t *new_of_old, int32_t *out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    out[k] = new_of_old[idx[k]];
}

}  // namespace

// Fraction of the estimated staleness bound used as the default in-flight cap;
// SCD_CAP_FRACTION overrides it for tuning experiments (tools/sweep_inflight.py).
double cap_fraction() {
  const char *e = getenv("SCD_CAP_FRACTION");
  double f = e ? atof(e) : 0.5;
  return f > 0 ? f : 0.5;
}

// Renumbering of the inner index space by frequency (SURVEY K8' "feature renumbering by frequency at
// load"): new id = rank of the index by (occurrences descending, index ascending); entries relabelled
// and re-sorted within each outer index (keys are distinct within an outer index, so the order is
// unique).  Output offsets equal the input ones.  Bit-exact (integer work only; values are moved).
scd_status renumber_device(const int64_t *ptr, const int32_t *idx, const float *val, int64_t outer, int64_t inner,
                           int64_t nnz, int64_t *optr, int32_t *oidx, float *oval, int32_t *new_of_old, cudaStream_t s,
                           std::string &err) {
  auto ck = [&](cudaError_t e, const char *what) {
    if (e != cudaSuccess) err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaSuccess;
  };
  unsigned long long *cnt = nullptr, *key = nullptr, *key_sorted = nullptr;
  int32_t *tmp_idx = nullptr;
  float *tmp_val = nullptr;
  void *tmp = nullptr;
  size_t tmp_b = 0;
  bool ok = ck(cudaMallocAsync((void **)&cnt, sizeof(unsigned long long) * (inner + 1), s), "alloc") &&
            ck(cudaMallocAsync((void **)&key, sizeof(unsigned long long) * inner, s), "alloc") &&
            ck(cudaMallocAsync((void **)&key_sorted, sizeof(unsigned long long) * inner, s), "alloc") &&
            ck(cudaMallocAsync((void **)&tmp_idx, sizeof(int32_t) * (nnz > 0 ? nnz : 1), s), "alloc");
  if (ok && val) ok = ck(cudaMallocAsync((void **)&tmp_val, sizeof(float) * (nnz > 0 ? nnz : 1), s), "alloc");
  if (ok) {
    cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (inner + 1), s);
    if (nnz > 0) k_count<<<grid_for(nnz, 256), 256, 0, s>>>(idx, nnz, cnt);
    k_rank_keys<<<grid_for(inner, 256), 256, 0, s>>>(cnt, inner, key);
    cub::DeviceRadixSort::SortKeys(nullptr, tmp_b, key, key_sorted, inner, 0, 64, s);
    ok = ck(cudaMallocAsync(&tmp, tmp_b, s), "alloc sort tmp") &&
         ck(cub::DeviceRadixSort::SortKeys(tmp, tmp_b, key, key_sorted, inner, 0, 64, s), "rank sort");
  }
  if (ok) {
    k_rank_scatter<<<grid_for(inner, 256), 256, 0, s>>>(key_sorted, inner, new_of_old);
    if (tmp) cudaFreeAsync(tmp, s);
    tmp = nullptr;
    ok = ck(cudaMemcpyAsync(optr, ptr, sizeof(int64_t) * (outer + 1), cudaMemcpyDeviceToDevice, s), "copy ptr");
  }
  if (ok && nnz > 0) {
    k_relabel<<<grid_for(nnz, 256), 256, 0, s>>>(idx, nnz, new_of_old, tmp_idx);
    if (val) ok = ck(cudaMemcpyAsync(tmp_val, val, sizeof(float) * nnz, cudaMemcpyDeviceToDevice, s), "copy val");
    tmp_b = 0;
    if (ok && val) {
      cub::DeviceSegmentedSort::SortPairs(nullptr, tmp_b, tmp_idx, oidx, tmp_val, oval, nnz, outer, ptr, ptr + 1, s);
      ok = ck(cudaMallocAsync(&tmp, tmp_b, s), "alloc seg sort") &&
           ck(cub::DeviceSegmentedSort::SortPairs(tmp, tmp_b, tmp_idx, oidx, tmp_val, oval, nnz, outer, ptr, ptr + 1, s),
              "segmented sort");
    } else if (ok) {
      cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_b, tmp_idx, oidx, nnz, outer, ptr, ptr + 1, s);
      ok = ck(cudaMallocAsync(&tmp, tmp_b, s), "alloc seg sort") &&
           ck(cub::DeviceSegmentedSort::SortKeys(tmp, tmp_b, tmp_idx, oidx, nnz, outer, ptr, ptr + 1, s),
              "segmented sort");
    }
  }
  ok = ok && ck(cudaGetLastError(), "renumber kernels");
  if (tmp) cudaFreeAsync(tmp, s);
  if (cnt) cudaFreeAsync(cnt, s);
  if (key) cudaFreeAsync(key, s);
  if (key_sorted) cudaFreeAsync(key_sorted, s);
  if (tmp_idx) cudaFreeAsync(tmp_idx, s);
  if (tmp_val) cudaFreeAsync(tmp_val, s);
  return ok ? SCD_OK : SCD_E_CUDA;
}

// Head of the shared vector combined in shared memory by the CTA kernel (k_epoch_cta_head,
// DESIGN.md §6): H = SCD_HEAD floats (default 8192, 0 = off), used when at least 10% of all
// stored entries fall in [0, H) — the frequency-ranked head of a power-law feature distribution.
static scd_status choose_head(scd_ctx *c, int *head) {
  *head = 0;
  int64_t H = 8192;
  if (const char *e = getenv("SCD_HEAD")) H = atoll(e);
  H = std::min<int64_t>(H, c->n_shared) / 4 * 4;
  if (H < 256 || c->opt.deterministic || c->nnz == 0) return SCD_OK;
  if (((uintptr_t)c->sv & 15) != 0) return SCD_OK;  // v4 flush needs 16-byte alignment
  unsigned long long *d = nullptr, h = 0;
  SCD_CK(c, cudaMallocAsync((void **)&d, sizeof(*d), c->stream));
  SCD_CK(c, cudaMemsetAsync(d, 0, sizeof(*d), c->stream));
  k_count_below<<<grid_for(c->nnz, 256, 148 * 8), 256, 0, c->stream>>>(c->idx, c->nnz, (int32_t)H, d);
  SCD_CKL(c, "k_count_below");
  SCD_CK(c, cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  SCD_CK(c, cudaStreamSynchronize(c->stream));
  cudaFreeAsync(d, c->stream);
  if ((double)h >= 0.10 * (double)c->nnz) *head = (int)H;
  return SCD_OK;
}

// Tail read copy of the head kernel: the gathers of tail entries (ids >= H) are served
// from svr, a copy of sv[H, max id] refreshed before every slice, so the lines that are gathered and
// the lines that take REDs are disjoint.  SCD_TAIL_SNAP = 1 (L2 loads) | 2 (L1-cached loads) | 0.
// Largest inner index + 1 of the local matrix (0 if empty): the dual's w̄ is zero beyond it, so the
// aggregation only exchanges [0, sv_active) (the max over all ranks, taken at the first round).
static scd_status active_extent(scd_ctx *c, int64_t *out) {
  *out = 0;
  if (c->nnz == 0) return SCD_OK;
  int *d = nullptr, h = -1;
  SCD_CK(c, cudaMallocAsync((void **)&d, sizeof(int), c->stream));
  SCD_CK(c, cudaMemsetAsync(d, 0xff, sizeof(int), c->stream));
  k_max_idx<<<grid_for(c->nnz, 256, 148 * 8), 256, 0, c->stream>>>(c->idx, c->nnz, d);
  SCD_CKL(c, "k_max_idx");
  SCD_CK(c, cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  SCD_CK(c, cudaStreamSynchronize(c->stream));
  cudaFreeAsync(d, c->stream);
  *out = (int64_t)h + 1;
  return SCD_OK;
}

static scd_status setup_tail_snap(scd_ctx *c, int head) {
  c->tail_snap = 0;
  const char *e = getenv("SCD_TAIL_SNAP");  // 0 = off, 1 = forced past the staleness rule (tests)
  const int mode = e ? atoi(e) : 1;
  if (head <= 0 || mode != 1 || c->form != SCD_DUAL) return SCD_OK;
  const int64_t h = c->sv_active - 1;
  if (h < head) return SCD_OK;
  c->tail_lo = head;
  c->tail_hi = (int64_t)h + 1;
  c->tail_snap = mode;  // the copy is allocated once the schedule keeps it (build_schedule)
  return SCD_OK;
}

// Staleness bound for one bin of the asynchronous schedule.  With τ coordinates of
// the bin in flight, a coordinate's update misses up to τ-1 concurrent updates.  Treating them as
// one block-Jacobi step, the step stays contractive while τ·c̄ < λN + d̄ (diagonal dominance of the
// coordinate-Hessian block), with d̄ = mean ||a||² and c̄ = mean |<a_i, a_j>| over pairs of the bin,
// obtained from ||(|A_b|ᵀ1)||² = Σ_i Σ_j |<a_i,a_j>| (so c̄ upper-bounds the mean |<a_i,a_j>|).
// Bins run one after another, so only intra-bin concurrency matters.
// One pass for both bounds (lo >= 0): the tail sums are the restriction of the same |A_b|ᵀ1 to
// ids >= lo, plus the tail entries' own squares (acc[2]) — see estimate_tail_tau below.
__global__ void k_abs_scatter2(const int64_t *ptr, const int32_t *idx, const float *val, const int32_t *list,
                               int64_t count, const float *norm, int32_t lo, double *s, double *acc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double sq = 0.0;
  for (int64_t j = warp; j < count; j += nwarps) {
    const int64_t o = list ? list[j] : j;
    for (int64_t k = ptr[o] + lane; k < ptr[o + 1]; k += 32) {
      const int32_t i = idx[k];
      const double v = (double)val_at(val, k);
      atomicAdd(s + i, fabs(v));
      if (i >= lo) sq += v * v;
    }
    if (lane == 0) atomicAdd(acc + 1, (double)norm[o]);
  }
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane == 0 && sq != 0.0) atomicAdd(acc + 2, sq);
}

scd_status estimate_bin_tau(scd_ctx *c, const int32_t *d_list, int64_t count, double *tau, int64_t lo,
                            double *tau_tail) {
  cudaStream_t s = c->stream;
  double *vec = c->vec64;
  c->vec64_version = 0;  // scratch use
  SCD_CK(c, cudaMemsetAsync(vec, 0, sizeof(double) * (size_t)c->n_shared, s));
  SCD_CK(c, cudaMemsetAsync(c->acc, 0, sizeof(double) * 8, s));
  const bool tail = lo >= 0 && lo < c->n_shared && tau_tail;
  if (tail)
    k_abs_scatter2<<<grid_for(count * 32, 256, 148 * 32), 256, 0, s>>>(c->ptr, c->idx, c->val, d_list, count, c->norm,
                                                                       (int32_t)lo, vec, c->acc);
  else
    k_abs_scatter<<<grid_for(count * 32, 256, 148 * 32), 256, 0, s>>>(c->ptr, c->idx, c->val, d_list, count, c->norm,
                                                                      vec, c->acc);
  k_sumsq<<<grid_for(c->n_shared, 256, 148 * 8), 256, 0, s>>>(vec, c->n_shared, c->acc);
  if (tail) k_sumsq<<<grid_for(c->n_shared - lo, 256, 148 * 8), 256, 0, s>>>(vec + lo, c->n_shared - lo, c->acc + 5);
  SCD_CKL(c, "coupling estimate");
  double h[8];
  SCD_CK(c, cudaMemcpyAsync(h, c->acc, sizeof(h), cudaMemcpyDeviceToHost, s));
  SCD_CK(c, cudaStreamSynchronize(s));
  const double n = (double)(count > 1 ? count : 2);
  const double cbar = (h[0] - h[1]) / (n * (n - 1.0));
  const double dbar = h[1] / n + c->lamN;
  *tau = cbar > 0 ? dbar / cbar : 1e18;
  if (tail) {
    const double ct = (h[5] - h[2]) / (n * (n - 1.0));
    *tau_tail = ct > 0 ? dbar / ct : 1e18;
  }
  return SCD_OK;
}

// Staleness bound of the bin's coupling through the shared-vector entries >= lo only (the tail read
// copy of the head kernel): τ_tail = (λN + d̄) / c̄_tail, c̄_tail from ||(|A_b[:, lo:]|ᵀ1)||²
// minus its diagonal terms.
scd_status estimate_tail_tau(scd_ctx *c, const int32_t *d_list, int64_t count, int64_t lo, double *tau,
                             const int32_t *idx) {
  cudaStream_t s = c->stream;
  double *vec = c->vec64;
  c->vec64_version = 0;  // scratch use
  SCD_CK(c, cudaMemsetAsync(vec, 0, sizeof(double) * (size_t)c->n_shared, s));
  SCD_CK(c, cudaMemsetAsync(c->acc, 0, sizeof(double) * 3, s));
  // idx: the entries to count (default the matrix's; the hot-set bin passes its re-encoded copy, whose
  // hot entries are negative and so fall below lo = 0)
  k_abs_scatter_tail<<<grid_for(count * 32, 256, 148 * 32), 256, 0, s>>>(c->ptr, idx ? idx : c->idx, c->val, d_list,
                                                                         count, c->norm, (int32_t)lo, vec, c->acc);
  k_sumsq<<<grid_for(c->n_shared - lo, 256, 148 * 8), 256, 0, s>>>(vec + lo, c->n_shared - lo, c->acc);
  SCD_CKL(c, "tail coupling estimate");
  double h[3];
  SCD_CK(c, cudaMemcpyAsync(h, c->acc, sizeof(h), cudaMemcpyDeviceToHost, s));
  SCD_CK(c, cudaStreamSynchronize(s));
  const double n = (double)(count > 1 ? count : 2);
  const double cbar = (h[0] - h[2]) / (n * (n - 1.0));
  const double dbar = h[1] / n + c->lamN;
  *tau = cbar > 0 ? dbar / cbar : 1e18;
  return SCD_OK;
}

scd_status validate_matrix(scd_ctx *c, int64_t outer, int64_t inner) {
  unsigned long long *d_bad = nullptr;
  SCD_CK(c, cudaMallocAsync((void **)&d_bad, sizeof(unsigned long long), c->stream));
  SCD_CK(c, cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), c->stream));
  k_validate<<<grid_for(outer * 32, 256), 256, 0, c->stream>>>(c->ptr, c->idx, outer, inner, c->nnz, d_bad);
  SCD_CKL(c, "k_validate");
  unsigned long long bad = 0;
  SCD_CK(c, cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, c->stream));
  SCD_CK(c, cudaStreamSynchronize(c->stream));
  cudaFreeAsync(d_bad, c->stream);
  if (bad != ~0ull)
    return fail(c, SCD_E_BAD_MATRIX, "matrix invariant violated at outer index " + std::to_string(bad));
  return SCD_OK;
}

scd_status compute_norms(scd_ctx *c) {
  k_norms<<<grid_for(c->n_coord * 32, 256), 256, 0, c->stream>>>(c->ptr, c->val, c->n_coord, c->norm);
  SCD_CKL(c, "k_norms");
  return SCD_OK;
}

// Device-side binning (create time): bin of every coordinate by its stored-entry count (255 = empty),
// per-bin count / entries / longest coordinate, and each bin's coordinate list in ascending order
// (cub::DeviceSelect, order-preserving).  Only the per-bin totals come back to the host.
constexpr int kNB = 4;
struct BinLimits {
  int64_t lim[kNB];
};

__global__ void k_bin_of(const int64_t *ptr, int64_t n, BinLimits L, uint8_t *bin,
                         unsigned long long *cnt /* [kNB + 1] */, unsigned long long *nnz /* [kNB] */,
                         unsigned long long *mx /* [kNB] */) {
  __shared__ unsigned long long s_c[kNB + 1], s_z[kNB], s_m[kNB];
  if (threadIdx.x < kNB + 1) s_c[threadIdx.x] = 0;
  if (threadIdx.x < kNB) s_z[threadIdx.x] = s_m[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t len = ptr[i + 1] - ptr[i];
    uint8_t b = 255;
    if (len > 0) {
      b = kNB - 1;
      for (int k = 0; k < kNB; ++k)
        if (len <= L.lim[k]) {
          b = (uint8_t)k;
          break;
        }
      atomicAdd(&s_z[b], (unsigned long long)len);
      atomicMax(&s_m[b], (unsigned long long)len);
    }
    bin[i] = b;
    atomicAdd(&s_c[b == 255 ? kNB : b], 1ull);
  }
  __syncthreads();
  if (threadIdx.x < kNB + 1 && s_c[threadIdx.x]) atomicAdd(cnt + threadIdx.x, s_c[threadIdx.x]);
  if (threadIdx.x < kNB && s_z[threadIdx.x]) atomicAdd(nnz + threadIdx.x, s_z[threadIdx.x]);
  if (threadIdx.x < kNB && s_m[threadIdx.x]) atomicMax(mx + threadIdx.x, s_m[threadIdx.x]);
}

struct BinIs {
  const uint8_t *bin;
  uint8_t b;
  __device__ __forceinline__ bool operator()(const int32_t &i) const { return bin[i] == b; }
};

// lists[k] (device, ascending ids) for k in [0, kNB] (kNB = the empty coordinates), allocated with
// cudaMalloc when the bin is non-empty and not the whole index range (then nullptr = identity).
static scd_status device_bins(scd_ctx *c, const int64_t lim[kNB], int32_t *lists[kNB + 1], int64_t count[kNB + 1],
                              int64_t nnz[kNB], int64_t maxlen[kNB]) {
  cudaStream_t s = c->stream;
  const int64_t n = c->n_coord;
  uint8_t *bin = nullptr;
  unsigned long long *st = nullptr;
  SCD_CK(c, cudaMallocAsync((void **)&bin, (size_t)std::max<int64_t>(n, 1), s));
  SCD_CK(c, cudaMallocAsync((void **)&st, sizeof(unsigned long long) * (3 * kNB + 1), s));
  SCD_CK(c, cudaMemsetAsync(st, 0, sizeof(unsigned long long) * (3 * kNB + 1), s));
  BinLimits L;
  for (int k = 0; k < kNB; ++k) L.lim[k] = lim[k];
  k_bin_of<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(c->ptr, n, L, bin, st, st + kNB + 1, st + 2 * kNB + 1);
  SCD_CKL(c, "k_bin_of");
  unsigned long long h[3 * kNB + 1];
  SCD_CK(c, cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
  SCD_CK(c, cudaStreamSynchronize(s));
  for (int k = 0; k <= kNB; ++k) count[k] = (int64_t)h[k];
  for (int k = 0; k < kNB; ++k) {
    nnz[k] = (int64_t)h[kNB + 1 + k];
    maxlen[k] = (int64_t)h[2 * kNB + 1 + k];
  }
  int *d_num = nullptr;
  SCD_CK(c, cudaMallocAsync((void **)&d_num, sizeof(int), s));
  void *tmp = nullptr;
  size_t tmp_b = 0;
  for (int k = 0; k <= kNB; ++k) {
    lists[k] = nullptr;
    if (count[k] == 0 || (count[k] == n && k < kNB)) continue;  // empty bin, or a bin's identity list
    SCD_CK(c, cudaMalloc((void **)&lists[k], sizeof(int32_t) * (size_t)count[k]));
    BinIs op{bin, (uint8_t)(k == kNB ? 255 : k)};
    cub::CountingInputIterator<int32_t> ids(0);
    size_t need = 0;
    cub::DeviceSelect::If(nullptr, need, ids, lists[k], d_num, (int)n, op, s);
    if (need > tmp_b) {
      if (tmp) cudaFreeAsync(tmp, s);
      SCD_CK(c, cudaMallocAsync(&tmp, need, s));
      tmp_b = need;
    }
    SCD_CK(c, cub::DeviceSelect::If(tmp, tmp_b, ids, lists[k], d_num, (int)n, op, s));
  }
  if (tmp) cudaFreeAsync(tmp, s);
  cudaFreeAsync(d_num, s);
  cudaFreeAsync(bin, s);
  cudaFreeAsync(st, s);
  SCD_CK(c, cudaStreamSynchronize(s));
  return SCD_OK;
}

// Asynchronous schedule: coordinates binned by stored-entry count, each bin processed by the
// kernel shape that suits its length.  Empty coordinates go to the empty list.
scd_status build_schedule(scd_ctx *c) {
  const int64_t n = c->n_coord;
  // bin thresholds (entries per coordinate): (0,64] -> 8-lane groups, (64,1024] -> warps,
  // (1024,16384] -> one CTA, > 16384 -> one 8-CTA cluster per coordinate
  constexpr int NB = 4;
  const int lanes[NB] = {8, 32, kLanesCta, kLanesCluster};
  int head = 0;
  if (scd_status st = choose_head(c, &head); st != SCD_OK) return st;
  // with the head-combining CTA kernel the medium rows (64, 1024] join the CTA bin (dual only): a
  // separate warp-bin launch per slice is a latency-bound single wave (C3: 2.5% of the step for 0.7%
  // of the entries)
  const int64_t lim1 = head > 0 && c->form == SCD_DUAL ? 64 : 1024;
  c->n_empty = 0;
  c->empty_list = nullptr;
  c->sv_active = c->n_shared;
  if (c->form == SCD_DUAL) {
    if (scd_status st = active_extent(c, &c->sv_active); st != SCD_OK) return st;
    c->sv_active = std::max<int64_t>(1, std::min(c->sv_active, c->n_shared));
  }
  if (scd_status st = setup_tail_snap(c, head); st != SCD_OK) return st;
  c->head_copy = 0;
  // one binning pass with the medium-row boundary lim1 (launch order: longest coordinates first)
  auto bin_pass = [&](int64_t l1) -> scd_status {
    const int64_t lim[NB] = {64, l1, 16384, INT64_MAX};
    int32_t *lists[NB + 1];
    int64_t cnt[NB + 1], nnzb[NB], maxb[NB];
    if (scd_status st = device_bins(c, lim, lists, cnt, nnzb, maxb); st != SCD_OK) return st;
    // the empty coordinates (the same for every pass)
    cudaFree(c->empty_list);
    c->empty_list = lists[NB];
    c->n_empty = cnt[NB];
    c->n_nonempty = n - c->n_empty;
    c->n_bins = 0;
    c->tau_star = 1e18;
    for (int b = NB - 1; b >= 0; --b) {
      if (cnt[b] == 0) continue;
      Bin &B = c->bins[c->n_bins];
      B = Bin();
      B.lanes = lanes[b];
      B.count = cnt[b];
      B.nnz = nnzb[b];
      B.maxlen = maxb[b];
      B.stream_id = 1u + (uint32_t)c->n_bins;
      B.list = lists[b];  // nullptr = identity: every coordinate is in this bin
      // the CTA bin of the head kernel also gets its tail bound (tail read copy) from the same pass
      const bool want_tail = c->tail_snap && B.lanes == kLanesCta && head > 0;
      scd_status st = estimate_bin_tau(c, B.list, B.count, &B.tau, want_tail ? (int64_t)head : -1, &B.tau_tail);
      if (st != SCD_OK) return st;
      if (B.tau < c->tau_star) c->tau_star = B.tau;
      double cap = cap_fraction() * B.tau;
      B.cap = c->opt.max_inflight > 0 ? (int64_t)c->opt.max_inflight : (int64_t)(cap < 1 ? 1 : (cap > 1e9 ? 1e9 : cap));
      B.head = B.lanes == kLanesCta ? head : 0;
      // block order for the short-coordinate bin (reading c28): 16.7 -> 13.1 ms on a C5 shard.  The
      // same rows of a block are in flight together every epoch, so it is used only while the bin's cap
      // spans >= 32 blocks (with a cap of 15 on strongly coupled rows the fixed co-occurrence stalled the
      // per-epoch rate: profiles/block_order_r2.txt)
      int64_t blk = 1;  // a power of two (the epoch order uses shifts and masks)
      while (blk * 2 <= (c->opt.block_order > 0 ? c->opt.block_order : 32)) blk *= 2;
      B.blk = (B.lanes == 8 && blk > 1 && B.cap >= 32 * blk) ? blk : 0;
      B.blk_shift = 0;
      while ((1ll << (B.blk_shift + 1)) <= B.blk) ++B.blk_shift;
      if (B.blk > 1 && B.count / B.blk > 0)
        SCD_CK(c, cudaMalloc((void **)&B.bperm, sizeof(int32_t) * (size_t)(B.count / B.blk)));
      bin_launch_shape(c, B);
      ++c->n_bins;
    }
    return SCD_OK;
  };
  if (scd_status st = bin_pass(lim1); st != SCD_OK) return st;
  if (lim1 < 1024) {
    // the medium rows only belong in the CTA bin when its head-combining kernel is actually used
    // (its window may not fit the staleness budget): otherwise bin again with the warp bin
    bool head_used = false;
    for (int i = 0; i < c->n_bins; ++i) head_used |= c->bins[i].lanes == kLanesCta && c->bins[i].head > 0;
    if (!head_used) {
      for (int i = 0; i < c->n_bins; ++i) {
        cudaFree(c->bins[i].list);
        cudaFree(c->bins[i].bperm);
        c->bins[i] = Bin();
      }
      if (scd_status st = bin_pass(1024); st != SCD_OK) return st;
    }
  }
  if (scd_status st = setup_hot(c); st != SCD_OK) return st;
  // interleave the bins in slices when more than one bin carries work (reading c24); SCD_SLICES overrides
  int S_env = 0;
  if (const char *e = getenv("SCD_SLICES")) {
    const int v = atoi(e);
    if (v >= 1 && v <= kMaxSlices) S_env = v;
  }
  int S = c->n_bins > 1 ? 8 : 1;
  // tail read copy: refreshed before every slice, so a tail read may miss every update of the current
  // slice; it is kept only while a slice of the head bin (8 slices, or SCD_SLICES) stays within
  // cap_fraction of the tail coupling's staleness bound
  if (c->tail_snap) {
    int bi = -1;
    for (int i = 0; i < c->n_bins; ++i)
      if (c->bins[i].head > 0 && c->bins[i].lanes == kLanesCta) bi = i;
    bool keep = bi >= 0;
    if (keep) {
      const Bin &B = c->bins[bi];
      c->tail_tau = B.tau_tail;
      if (!(c->tail_tau > 0)) {  // not estimated in the binning pass
        if (scd_status st = estimate_tail_tau(c, B.list, B.count, c->tail_lo, &c->tail_tau); st != SCD_OK) return st;
      }
      const double slice_rows = (double)B.count / (double)(S_env ? S_env : 8);
      const bool forced = getenv("SCD_TAIL_SNAP") != nullptr;
      // either refreshed between slices (a slice within the bound) or, with one head bin, in rolling
      // chunks whose full sweep is within the bound (possible with a shorter sweep than a slice)
      const int64_t nch = (c->tail_hi - c->tail_lo + 4 * kLanesCta - 1) / (4 * kLanesCta);
      const bool can_roll = c->n_bins == 1 && S_env == 0 && nch > 0 &&
                            std::min(cap_fraction() * c->tail_tau, (double)B.count / 8.0) >= (double)nch;
      keep = forced || (c->opt.max_inflight == 0 && (slice_rows <= cap_fraction() * c->tail_tau || can_roll));
    }
    if (keep) {
      SCD_CK(c, cudaMalloc((void **)&c->svr, sizeof(float) * (size_t)c->n_shared));
      SCD_CK(c, cudaMemsetAsync(c->svr, 0, sizeof(float) * (size_t)c->n_shared, c->stream));
      S = 8;
      // Rolling refresh (single head bin): the copy is refreshed 1024 floats at a time by every
      // tail_roll-th row, so that one full sweep of the tail takes no more rows than a slice would
      // (cap_fraction · τ_tail and 1/8 of the bin), and the epoch needs no slice boundaries (each
      // costs a drain of the grid behind the longest rows: ~65 µs on C3).
      // With several bins (or SCD_SLICES) the copy is refreshed between slices instead.
      c->tail_roll = 0;
      if (c->n_bins == 1 && S_env == 0 && c->opt.max_inflight == 0) {
        Bin &B = c->bins[bi];
        const int64_t nch = (c->tail_hi - c->tail_lo + 4 * kLanesCta - 1) / (4 * kLanesCta);
        const double sweep = std::min(cap_fraction() * c->tail_tau, (double)B.count / 8.0);
        const int64_t R = nch > 0 ? (int64_t)(sweep / (double)nch) : 0;
        if (R >= 1) {
          c->tail_roll = R;
          S = 1;
          // one launch per epoch with the rolling copy: the SM-shared head kernel when its window fits
          if (!sm_head_shape(c, B) && B.sm) {
            B.sm = 0;
            bin_launch_shape(c, B);
          }
        }
      }
      // Head copy: the head gathers also read svr[0, H), refreshed in rolling 1024-float chunks every
      // P rows, so they too land on lines that take no REDs.  A head read may then miss what was flushed
      // in the last P · nchunks rows: that age joins the combined-update budget (reading c25),
      // rows in flight + deferred + age = grid · (1 + flush) + P · nchunks <= budget; the flush window
      // gives way (down to 2) until P >= 16 fits (a shorter period costs more in refresh traffic than
      // it saves: profiles/head_copy_r1.txt).
      Bin &HB = c->bins[bi];
      if (c->tail_roll > 0 && HB.head > 0 && !HB.sm) {
        const int64_t nchh = (HB.head + 4 * kLanesCta - 1) / (4 * kLanesCta);
        const double budget = combine_budget(c, HB);
        int64_t P = 0;
        int f = HB.flush;
        for (; f >= 2; --f) {
          P = (int64_t)((budget - (double)HB.grid * (1.0 + f)) / (double)nchh);
          if (P >= 16) break;
        }
        if (P >= 16) {
          c->head_copy = P;
          HB.flush = f;
        }
      }
    } else {
      c->tail_snap = 0;
    }
  }
  c->n_slices = S_env ? S_env : S;
  // Snapshot bins: when one slice launch of a bin holds no more coordinates than the bin's in-flight
  // cap (cap_fraction * τ_b), the whole launch may gather from a copy of the shared vector taken
  // just before it — the same block-Jacobi bound as the in-flight cap, with the whole slice counted
  // as in flight — so the lines gathered and the lines reduced are disjoint.  Plain
  // kernels only; the copy refresh must stay small next to the slice's own traffic.
  const bool snap_ok = !c->opt.deterministic && !c->opt.wild && c->opt.max_inflight == 0;
  bool any_snap = false;
  for (int i = 0; i < c->n_bins && snap_ok; ++i) {
    Bin &B = c->bins[i];
    B.snap = 0;
    if (B.head > 0 || B.hot > 0) continue;
    const double slice = (double)B.count / (double)c->n_slices;
    const double refresh_bytes = 8.0 * (double)c->n_shared, slice_bytes = 16.0 * (double)B.nnz / c->n_slices;
    // like the combined-update windows (combine_window, reading c25) a slice may also be at most 1/8
    // of the bin: the bound keeps the step contractive, the 1/8 keeps the per-epoch rate sequential-like
    // (a whole-epoch snapshot is a Jacobi epoch and converges visibly slower per epoch)
    if (slice <= cap_fraction() * B.tau && slice <= (double)B.count / 8.0 + 1.0 && refresh_bytes <= 0.05 * slice_bytes) {
      B.snap = 1;
      any_snap = true;
    }
  }
  if (any_snap && !c->svr) {
    SCD_CK(c, cudaMalloc((void **)&c->svr, sizeof(float) * (size_t)c->n_shared));
    SCD_CK(c, cudaMemsetAsync(c->svr, 0, sizeof(float) * (size_t)c->n_shared, c->stream));
  }
  // one ticket counter per (slice, bin)
  SCD_CK(c, cudaMalloc((void **)&c->counters, sizeof(unsigned int) * kMaxBins * kMaxSlices));
  return SCD_OK;
}

// nnz-balanced partition of the outer coordinates over k workers ("partition the
// coordinates in an intelligent way"; reading c29).  Coordinates in order of decreasing length, ties in
// the order of the partition permutation (stream kPartStream, epoch 0: the random partition of c15),
// dealt to the workers in snake order 0..k-1, k-1..0, ...  Every worker's stored-entry count is then
// within the longest coordinate of every other's (the random partition of c15 balances counts only).
__global__ void k_bal_keys(const int64_t *ptr, int64_t n, Perm p, unsigned long long *keys, int32_t *ids) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = (int64_t)perm_apply(p, (uint64_t)i);
    const int64_t len = ptr[c + 1] - ptr[c];
    const unsigned long long inv = 0xFFFFFFFFull - (unsigned long long)(len < 0xFFFFFFFFll ? len : 0xFFFFFFFFll);
    keys[i] = (inv << 32) | (unsigned long long)i;  // length descending, then position ascending
    ids[i] = (int32_t)c;
  }
}

__global__ void k_bal_deal(const int32_t *ids, int64_t n, int32_t k, int32_t *owner) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / k, j = i % k;
    owner[ids[i]] = (int32_t)((r & 1) ? k - 1 - j : j);
  }
}

scd_status partition_balanced_device(const int64_t *ptr, int64_t n, uint64_t seed, int32_t k, int32_t *d_owner,
                                     cudaStream_t s, std::string &err) {
  auto ck = [&](cudaError_t e, const char *what) {
    if (e != cudaSuccess) err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaSuccess;
  };
  unsigned long long *keys = nullptr, *keys2 = nullptr;
  int32_t *ids = nullptr, *ids2 = nullptr;
  void *tmp = nullptr;
  size_t tb = 0;
  bool ok = ck(cudaMallocAsync((void **)&keys, sizeof(*keys) * n, s), "alloc") &&
            ck(cudaMallocAsync((void **)&keys2, sizeof(*keys2) * n, s), "alloc") &&
            ck(cudaMallocAsync((void **)&ids, sizeof(*ids) * n, s), "alloc") &&
            ck(cudaMallocAsync((void **)&ids2, sizeof(*ids2) * n, s), "alloc");
  if (ok) {
    k_bal_keys<<<grid_for(n, 256), 256, 0, s>>>(ptr, n, make_perm(seed, 0u, kPartStream, n), keys, ids);
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, ids, ids2, n, 0, 64, s);
    ok = ck(cudaMallocAsync(&tmp, tb, s), "alloc sort tmp") &&
         ck(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, ids, ids2, n, 0, 64, s), "sort");
    if (ok) k_bal_deal<<<grid_for(n, 256), 256, 0, s>>>(ids2, n, k, d_owner);
    ok = ok && ck(cudaGetLastError(), "partition kernels");
  }
  for (void *q : {(void *)keys, (void *)keys2, (void *)ids, (void *)ids2, tmp})
    if (q) cudaFreeAsync(q, s);
  return ok ? SCD_OK : SCD_E_CUDA;
}

// Stable transpose on the device: stable radix sort of (inner index -> entry position), then
// gather of the outer index and value.  Equal keys keep input order (increasing outer index).
scd_status transpose_device(const int64_t *ptr, const int32_t *idx, const float *val, int64_t outer, int64_t inner,
                            int64_t nnz, int64_t *optr, int32_t *oidx, float *oval, cudaStream_t s, std::string &err) {
  auto ck = [&](cudaError_t e, const char *what) {
    if (e != cudaSuccess) err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaSuccess;
  };
  int32_t *outer_of = nullptr, *keys_out = nullptr;
  int64_t *pos_in = nullptr, *pos_out = nullptr;
  unsigned long long *cnt = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  const int64_t n1 = nnz > 0 ? nnz : 1;
  bool ok = ck(cudaMallocAsync((void **)&outer_of, sizeof(int32_t) * n1, s), "alloc") &&
            ck(cudaMallocAsync((void **)&keys_out, sizeof(int32_t) * n1, s), "alloc") &&
            ck(cudaMallocAsync((void **)&pos_in, sizeof(int64_t) * n1, s), "alloc") &&
            ck(cudaMallocAsync((void **)&pos_out, sizeof(int64_t) * n1, s), "alloc") &&
            ck(cudaMallocAsync((void **)&cnt, sizeof(unsigned long long) * (inner + 1), s), "alloc");
  if (ok) {
    cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (inner + 1), s);
    if (nnz > 0) {
      k_outer_of<<<grid_for(outer * 32, 256), 256, 0, s>>>(ptr, outer, outer_of);
      k_iota64<<<grid_for(nnz, 256), 256, 0, s>>>(pos_in, nnz);
      k_count<<<grid_for(nnz, 256), 256, 0, s>>>(idx, nnz, cnt);
      int end_bit = 1;
      while (end_bit < 32 && (1ll << end_bit) < inner) ++end_bit;
      cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (const uint32_t *)idx, (uint32_t *)keys_out, pos_in, pos_out,
                                      nnz, 0, end_bit, s);
      ok = ck(cudaMallocAsync(&tmp, tmp_bytes, s), "alloc sort tmp");
      if (ok) {
        ok = ck(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, (const uint32_t *)idx, (uint32_t *)keys_out, pos_in,
                                                pos_out, nnz, 0, end_bit, s),
                "radix sort");
      }
      if (ok) k_gather_t<<<grid_for(nnz, 256), 256, 0, s>>>(pos_out, outer_of, val, nnz, oidx, oval);
    }
    if (ok) {
      // counts (cnt[0] = 0) -> inclusive scan = offsets
      size_t sb = 0;
      cub::DeviceScan::InclusiveSum(nullptr, sb, cnt, (unsigned long long *)optr, inner + 1, s);
      void *tmp2 = nullptr;
      ok = ck(cudaMallocAsync(&tmp2, sb, s), "alloc scan tmp") &&
           ck(cub::DeviceScan::InclusiveSum(tmp2, sb, cnt, (unsigned long long *)optr, inner + 1, s), "scan");
      if (tmp2) cudaFreeAsync(tmp2, s);
    }
    ok = ok && ck(cudaGetLastError(), "transpose kernels");
  }
  if (tmp) cudaFreeAsync(tmp, s);
  if (outer_of) cudaFreeAsync(outer_of, s);
  if (keys_out) cudaFreeAsync(keys_out, s);
  if (pos_in) cudaFreeAsync(pos_in, s);
  if (pos_out) cudaFreeAsync(pos_out, s);
  if (cnt) cudaFreeAsync(cnt, s);
  return ok ? SCD_OK : SCD_E_CUDA;
}

}  // namespace scd
