// synth_cuda.cu — device twin of the seeded synthetic input generators (see synth.h).
// Test/bench infrastructure; holds none of the method's arithmetic.  Bit-exact with
// synth_host.c (integer hashing; exact int->float conversion and power-of-two scaling).
#include "synth.h"
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

namespace {

__device__ __forceinline__ uint64_t sx_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t sx_h(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b) {
  return sx_mix64(sx_mix64(sx_mix64(seed ^ (tag * 0xD6E8FEB86659FD93ull)) ^ a) ^ b);
}
__device__ __forceinline__ uint32_t sx_alias_draw(uint64_t u, uint64_t n, const uint32_t *__restrict__ thr,
                                                  const uint32_t *__restrict__ alias) {
  uint32_t b = (uint32_t)(((u >> 32) * n) >> 32);
  uint32_t coin = (uint32_t)u;
  return coin < __ldg(thr + b) ? b : __ldg(alias + b);
}

struct ZipfDev {
  int64_t n_active;
  uint64_t seed;
  int32_t values_one, flip_mask;
  const uint32_t *len_table, *thr, *alias;
};

__global__ void k_zipf_lengths(ZipfDev p, int64_t row0, int64_t nrows, int64_t *len_out) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int64_t k = (int64_t)p.len_table[sx_h(p.seed, SYNTH_TAG_LEN, (uint64_t)(row0 + r), 0) >> 54];
  if (k > p.n_active) k = p.n_active;
  len_out[r] = k;  // written at [r]; exclusive scan turns it into ptr
}

constexpr int kGenThreads = 256;

// One CTA per row; shared-memory bitmap over [0, F).  Draws are taken in batches of
// kGenThreads; the batch that would overshoot k is undone and replayed sequentially so
// the selected set is exactly "the first k distinct draws" (= the host twin's set).
__global__ void __launch_bounds__(kGenThreads) k_zipf_rows(ZipfDev p, int64_t row0, int64_t nrows,
                                                           const int64_t *__restrict__ ptr, int32_t *__restrict__ idx,
                                                           float *__restrict__ val, float *__restrict__ y) {
  extern __shared__ uint32_t bm[];
  __shared__ long long s_red[kGenThreads / 32];
  __shared__ int s_wsum[kGenThreads / 32];
  const int tid = threadIdx.x;
  const int64_t F = p.n_active;
  const int W = (int)((F + 31) / 32);
  for (int i = tid; i < W; i += kGenThreads) bm[i] = 0u;
  __syncthreads();
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t n = row0 + r;
    const int64_t base = ptr[r];
    const int64_t k = ptr[r + 1] - base;
    const uint64_t rowkey = sx_mix64(sx_mix64(p.seed ^ (SYNTH_TAG_DRAW * 0xD6E8FEB86659FD93ull)) ^ (uint64_t)n);
    int64_t cnt = 0;
    uint64_t d0 = 0;
    while (cnt < k) {
      uint32_t f = sx_alias_draw(sx_mix64(rowkey ^ (d0 + tid)), (uint64_t)F, p.thr, p.alias);
      uint32_t bit = 1u << (f & 31);
      uint32_t old = atomicOr(&bm[f >> 5], bit);
      int isnew = !(old & bit);
      int c = __syncthreads_count(isnew);
      if (cnt + c <= k) {
        cnt += c;
        d0 += kGenThreads;
      } else {
        if (isnew) atomicAnd(&bm[f >> 5], ~bit);
        __syncthreads();
        if (tid == 0) {
          int64_t cc = cnt;
          for (int dd = 0; dd < kGenThreads && cc < k; ++dd) {
            uint32_t g = sx_alias_draw(sx_mix64(rowkey ^ (d0 + dd)), (uint64_t)F, p.thr, p.alias);
            uint32_t gb = 1u << (g & 31);
            if (!(bm[g >> 5] & gb)) { bm[g >> 5] |= gb; ++cc; }
          }
        }
        __syncthreads();
        cnt = k;
      }
    }
    // extraction: contiguous word chunks per thread, block exclusive scan of popcounts
    const int chunk = (W + kGenThreads - 1) / kGenThreads;
    const int w0 = tid * chunk;
    const int w1 = min(W, w0 + chunk);
    int mycount = 0;
    for (int w = w0; w < w1; ++w) mycount += __popc(bm[w]);
    // block exclusive scan
    const int lane = tid & 31, wid = tid >> 5;
    int incl = mycount;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_wsum[wid] = incl;
    __syncthreads();
    int woff = 0;
    for (int i = 0; i < wid; ++i) woff += s_wsum[i];
    int pos = woff + incl - mycount;
    const int e = (63 - __clzll((unsigned long long)(k > 0 ? k : 1))) / 2;
    long long score = 0;
    for (int w = w0; w < w1; ++w) {
      uint32_t word = bm[w];
      bm[w] = 0u;
      while (word) {
        int b = __ffs(word) - 1;
        word &= word - 1;
        uint32_t f = (uint32_t)w * 32u + (uint32_t)b;
        uint64_t code = p.values_one ? 1ull : ((sx_h(p.seed, SYNTH_TAG_VAL, (uint64_t)n, f) >> 40) + 1ull);
        idx[base + pos] = (int32_t)f;
        val[base + pos] = p.values_one ? 1.0f : ldexpf((float)code, -24 - e);
        score += ((sx_h(p.seed, SYNTH_TAG_SIGN, f, 0) & 1ull) ? 1ll : -1ll) * (long long)code;
        ++pos;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) score += __shfl_xor_sync(0xffffffffu, score, o);
    if (lane == 0) s_red[wid] = score;
    __syncthreads();
    if (tid == 0) {
      long long s = 0;
      for (int i = 0; i < kGenThreads / 32; ++i) s += s_red[i];
      float lab = s >= 0 ? 1.0f : -1.0f;
      if (p.flip_mask && (sx_h(p.seed, SYNTH_TAG_FLIP, (uint64_t)n, 0) & (uint64_t)p.flip_mask) == 0) lab = -lab;
      y[r] = lab;
    }
    __syncthreads();
  }
}

struct FieldsDev {
  int64_t n_cols;
  int32_t n_fields, flip_mask;
  uint64_t seed;
  const int64_t *off, *card;
  const uint32_t *thr, *alias;
};

__global__ void k_fields_rows(FieldsDev p, int64_t row0, int64_t nrows, int64_t *__restrict__ ptr,
                              int32_t *__restrict__ idx, float *__restrict__ val, float *__restrict__ y) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r > nrows) return;
  const int nf = p.n_fields;
  ptr[r] = r * nf;
  if (r == nrows) return;
  const int64_t n = row0 + r;
  const uint64_t rowkey = sx_mix64(sx_mix64(p.seed ^ (SYNTH_TAG_DRAW * 0xD6E8FEB86659FD93ull)) ^ (uint64_t)n);
  int64_t score = 0;
  for (int i = 0; i < nf; ++i) {
    const int64_t off = p.off[i];
    uint32_t rank = sx_alias_draw(sx_mix64(rowkey ^ (uint64_t)i), (uint64_t)p.card[i], p.thr + off, p.alias + off);
    uint64_t f = (uint64_t)off + rank;
    idx[r * nf + i] = (int32_t)f;
    val[r * nf + i] = 1.0f;
    score += (sx_h(p.seed, SYNTH_TAG_SIGN, f, 0) & 1ull) ? 1 : -1;
  }
  float lab = score >= 0 ? 1.0f : -1.0f;
  if (p.flip_mask && (sx_h(p.seed, SYNTH_TAG_FLIP, (uint64_t)n, 0) & (uint64_t)p.flip_mask) == 0) lab = -lab;
  y[r] = lab;
}

template <typename T>
int upload(const T *h, size_t n, T **d, cudaStream_t s) {
  cudaError_t e = cudaMallocAsync((void **)d, n * sizeof(T), s);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaMemcpyAsync(*d, h, n * sizeof(T), cudaMemcpyHostToDevice, s);
}

}  // namespace

extern "C" int synth_zipf_fill_device(const synth_zipf_rows *p, int64_t row0, int64_t nrows, int64_t *ptr_dev,
                                      int32_t *idx_dev, float *val_dev, float *y_dev, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nrows <= 0) {
    return (int)cudaMemsetAsync(ptr_dev, 0, sizeof(int64_t), s);
  }
  const int64_t F = p->n_active;
  uint32_t *d_len = nullptr, *d_thr = nullptr, *d_alias = nullptr;
  int rc;
  if ((rc = upload(p->len_table, SYNTH_LEN_TABLE, &d_len, s))) return rc;
  if ((rc = upload(p->alias_thr, (size_t)F, &d_thr, s))) return rc;
  if ((rc = upload(p->alias_idx, (size_t)F, &d_alias, s))) return rc;
  ZipfDev dp{F, p->seed, p->values_one, p->flip_mask, d_len, d_thr, d_alias};
  // lengths -> ptr (exclusive scan over nrows+1 entries, last length = 0)
  cudaMemsetAsync(ptr_dev + nrows, 0, sizeof(int64_t), s);
  k_zipf_lengths<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(dp, row0, nrows, ptr_dev);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, ptr_dev, ptr_dev, nrows + 1, s);
  void *tmp = nullptr;
  if (cudaMallocAsync(&tmp, tmp_bytes, s) != cudaSuccess) return (int)cudaErrorMemoryAllocation;
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, ptr_dev, ptr_dev, nrows + 1, s);
  const size_t smem = (size_t)((F + 31) / 32) * sizeof(uint32_t);
  cudaFuncSetAttribute(k_zipf_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_zipf_rows, kGenThreads, smem);
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)nsm * occ;
  if (grid > nrows) grid = nrows;
  k_zipf_rows<<<(unsigned)grid, kGenThreads, smem, s>>>(dp, row0, nrows, ptr_dev, idx_dev, val_dev, y_dev);
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(d_len, s);
  cudaFreeAsync(d_thr, s);
  cudaFreeAsync(d_alias, s);
  return (int)cudaGetLastError();
}

extern "C" int synth_fields_fill_device(const synth_fields *p, int64_t row0, int64_t nrows, int64_t *ptr_dev,
                                        int32_t *idx_dev, float *val_dev, float *y_dev, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int64_t *d_off = nullptr, *d_card = nullptr;
  uint32_t *d_thr = nullptr, *d_alias = nullptr;
  int rc;
  if ((rc = upload(p->field_off, (size_t)p->n_fields, &d_off, s))) return rc;
  if ((rc = upload(p->field_card, (size_t)p->n_fields, &d_card, s))) return rc;
  if ((rc = upload(p->alias_thr, (size_t)p->n_cols, &d_thr, s))) return rc;
  if ((rc = upload(p->alias_idx, (size_t)p->n_cols, &d_alias, s))) return rc;
  FieldsDev dp{p->n_cols, p->n_fields, p->flip_mask, p->seed, d_off, d_card, d_thr, d_alias};
  k_fields_rows<<<(unsigned)((nrows + 1 + 255) / 256), 256, 0, s>>>(dp, row0, nrows, ptr_dev, idx_dev, val_dev, y_dev);
  cudaFreeAsync(d_off, s);
  cudaFreeAsync(d_card, s);
  cudaFreeAsync(d_thr, s);
  cudaFreeAsync(d_alias, s);
  return (int)cudaGetLastError();
}
