// hot.cu — hot-set re-encoding for the short-coordinate bin (k_epoch_group_hot, epoch.cu).
//
// On one-hot (criteo-shaped) data a few thousand shared-vector entries carry most stored entries:
// the top values of the small and numeric fields appear in 20-38% of all rows.  At create the K most
// frequent shared-vector indices of the bin get a slot (most frequent first) and a private copy of
// the bin's inner indices is written with hot entries re-encoded as (slot | 0x80000000); the epoch
// kernel then keeps those entries' pending updates in shared memory per CTA.  Which entries are hot
// is a property of the data measured here, not assumed from any generator.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"

namespace scd {
namespace {

// occurrences of each inner index among the stored entries of the coordinates in `list`
__global__ void k_hot_count(const int64_t *ptr, const int32_t *idx, const int32_t *list, int64_t count,
                            unsigned *cnt) {
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t i = w0; i < count; i += nw) {
    const int64_t c = list ? list[i] : i;
    for (int64_t k = ptr[c] + lane; k < ptr[c + 1]; k += 32) atomicAdd(cnt + idx[k], 1u);
  }
}

__global__ void k_iota32(int32_t *p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

__global__ void k_hot_slots(const int32_t *hot_ids, int K, int32_t *slot_of) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x) slot_of[hot_ids[i]] = i;
}

// private re-encoded indices of the bin's coordinates (other coordinates' entries are copied as is)
__global__ void k_hot_encode(const int32_t *idx, int64_t nnz, const int32_t *slot_of, int32_t *out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = idx[k];
    const int32_t s = slot_of[j];
    out[k] = s >= 0 ? (int32_t)(0x80000000u | (uint32_t)s) : j;
  }
}

}  // namespace

// SCD_HOT = K (default 4096, 0 = off): hot slots for the short-coordinate bin; used when the K hottest
// entries hold >= 30% of the bin's stored entries and the private index copy fits in free memory.
scd_status setup_hot(scd_ctx *c) {
  int64_t K = 4096;
  if (const char *e = getenv("SCD_HOT")) K = atoll(e);
  K = std::min<int64_t>(K, c->n_shared) / 4 * 4;
  if (K < 64 || c->opt.deterministic || c->opt.wild || c->nnz == 0) return SCD_OK;
  int bi = -1;
  for (int i = 0; i < c->n_bins; ++i)
    if (c->bins[i].lanes == 8) bi = i;
  if (bi < 0) return SCD_OK;
  Bin &b = c->bins[bi];
  if (b.nnz < 1000000) return SCD_OK;  // small problems: the CTA-combining kernel is fine
  size_t free_b = 0, total_b = 0;
  SCD_CK(c, cudaMemGetInfo(&free_b, &total_b));
  if ((size_t)c->nnz * 4 + (size_t)c->n_shared * 16 + ((size_t)1 << 30) > free_b) return SCD_OK;
  cudaStream_t s = c->stream;
  const int64_t n = c->n_shared;
  unsigned *cnt = nullptr, *cnt_sorted = nullptr;
  int32_t *ids = nullptr, *ids_sorted = nullptr;
  SCD_CK(c, cudaMallocAsync((void **)&cnt, sizeof(unsigned) * n, s));
  SCD_CK(c, cudaMallocAsync((void **)&cnt_sorted, sizeof(unsigned) * n, s));
  SCD_CK(c, cudaMallocAsync((void **)&ids, sizeof(int32_t) * n, s));
  SCD_CK(c, cudaMallocAsync((void **)&ids_sorted, sizeof(int32_t) * n, s));
  SCD_CK(c, cudaMemsetAsync(cnt, 0, sizeof(unsigned) * n, s));
  k_hot_count<<<grid_for(b.count * 32, 256, 148 * 32), 256, 0, s>>>(c->ptr, c->idx, b.list, b.count, cnt);
  k_iota32<<<grid_for(n, 256), 256, 0, s>>>(ids, n);
  SCD_CKL(c, "hot count");
  size_t tmp_b = 0;
  void *tmp = nullptr;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_b, cnt, cnt_sorted, ids, ids_sorted, n, 0, 32, s);
  SCD_CK(c, cudaMallocAsync(&tmp, tmp_b, s));
  SCD_CK(c, cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_b, cnt, cnt_sorted, ids, ids_sorted, n, 0, 32, s));
  std::vector<unsigned> top((size_t)K);
  SCD_CK(c, cudaMemcpyAsync(top.data(), cnt_sorted, sizeof(unsigned) * K, cudaMemcpyDeviceToHost, s));
  SCD_CK(c, cudaStreamSynchronize(s));
  double cover = 0;
  int64_t kk = 0;
  for (; kk < K && top[(size_t)kk] > 1; ++kk) cover += top[(size_t)kk];  // an entry used once cannot combine
  kk = kk / 4 * 4;
  scd_status st = SCD_OK;
  if (kk >= 64 && cover >= 0.30 * (double)b.nnz) {
    if (cudaMalloc((void **)&c->hot_ids, sizeof(int32_t) * kk) != cudaSuccess ||
        cudaMalloc((void **)&c->hot_idx, sizeof(int32_t) * c->nnz) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(c->hot_ids);
      c->hot_ids = nullptr;
    } else {
      int32_t *slot_of = reinterpret_cast<int32_t *>(cnt);  // reuse: n int32
      // slots in shared-vector order, not frequency order: the top values of a frequency-ranked field
      // are consecutive ids, so a warp's flush REDs over 32 consecutive slots coalesce into a few
      // sector operations instead of 32 on the hottest lines (profiles/hot_order_r1.txt)
      std::vector<int32_t> hid((size_t)kk);
      cudaMemcpyAsync(hid.data(), ids_sorted, sizeof(int32_t) * kk, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      std::sort(hid.begin(), hid.end());
      cudaMemcpyAsync(c->hot_ids, hid.data(), sizeof(int32_t) * kk, cudaMemcpyHostToDevice, s);
      cudaMemsetAsync(slot_of, 0xff, sizeof(int32_t) * n, s);
      k_hot_slots<<<grid_for(kk, 256), 256, 0, s>>>(c->hot_ids, (int)kk, slot_of);
      k_hot_encode<<<grid_for(c->nnz, 256, 148 * 16), 256, 0, s>>>(c->idx, c->nnz, slot_of, c->hot_idx);
      if (cudaGetLastError() != cudaSuccess) st = fail(c, SCD_E_CUDA, "hot-set encode");
      c->hot_cover = cover / (double)b.nnz;
      b.hot = (int)kk;
    }
  }
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(cnt, s);
  cudaFreeAsync(cnt_sorted, s);
  cudaFreeAsync(ids, s);
  cudaFreeAsync(ids_sorted, s);
  SCD_CK(c, cudaStreamSynchronize(s));
  if (st != SCD_OK) return st;
  if (b.hot > 0) {
    // Tail prefetch: the next batch's non-hot values are gathered one step early, i.e. up to one more
    // round of the rows in flight old.  Like the webspam tail copy (reading c26), that is allowed when
    // the coupling through the non-hot entries alone bounds it: 2 x rows in flight <= cap_fraction x
    // tau_tail (estimated from the re-encoded indices, hot entries excluded).  The launch shape is
    // computed twice: the rows in flight decide hot_tp, and hot_tp joins the window budget.
    c->hot_tp = false;
    if (scd_status st2 = estimate_tail_tau(c, b.list, b.count, 0, &c->hot_tail_tau, c->hot_idx); st2 != SCD_OK)
      return st2;
    bin_launch_shape(c, b);
    if (b.hot > 0 && c->hot_tail_tau > 0) {
      const double inflight = (double)b.grid * (b.block / 8);
      c->hot_tp = 2.0 * inflight <= cap_fraction() * c->hot_tail_tau;
      if (c->hot_tp) bin_launch_shape(c, b);
    }
  }
  return SCD_OK;
}

}  // namespace scd
