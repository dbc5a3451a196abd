// die_pattern.cu — the epoch's access pattern (gather + RED of sv[idx] per stored entry, no
// algorithmic dependencies) split by the home die of sv[idx]: does die-local processing speed up
// the real webspam-shaped index stream?  Used by tools/die_pattern.py.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o tools/libdiepattern.so tools/die_pattern.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int kChunk = 512;

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned atom_lat(float *p) {
  float x = 0.f;
  long long t0 = clock64();
#pragma unroll 1
  for (int r = 0; r < 4; ++r) x = atomicAdd(p + (int)(x * 0.f), 0.f);
  return (unsigned)((clock64() - t0) / 4) + (x == 1.5f);
}
__global__ void k_smlat(float *sv, int np, unsigned *lat) {
  extern __shared__ char pad[];
  if (threadIdx.x) return;
  pad[0] = 0;
  const unsigned s = smid();
  for (int l = 0; l < np; ++l) lat[s * np + l] = atom_lat(sv + (size_t)l * kChunk + (s & 7) * 32);
}
__global__ void k_chlat(float *sv, int64_t nch, const uint8_t *smd, unsigned *ctr, int n0, int n1, unsigned *l0,
                        unsigned *l1) {
  extern __shared__ char pad[];
  __shared__ unsigned rk;
  const int d = smd[smid()];
  if (threadIdx.x == 0) {
    pad[0] = 0;
    rk = atomicAdd(ctr + d, 1u);
  }
  __syncthreads();
  if (threadIdx.x & 31) return;
  const int nw = blockDim.x / 32, w = threadIdx.x / 32;
  const int64_t nd = d ? n1 : n0;
  for (int64_t c = (int64_t)rk * nw + w; c < nch; c += nd * nw) (d ? l1 : l0)[c] = atom_lat(sv + c * kChunk);
}

// chunk_die[nchunk], sm_die[256]; returns SMs on die 0 (or -1)
extern "C" int die_map(float *sv, int64_t n, uint8_t *chunk_die, uint8_t *sm_die_dev) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int np = 64, pad = 160 * 1024;
  unsigned *lat;
  cudaMalloc(&lat, sizeof(unsigned) * 256 * np);
  cudaMemset(lat, 0, sizeof(unsigned) * 256 * np);
  cudaFuncSetAttribute(k_smlat, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
  cudaFuncSetAttribute(k_chlat, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
  k_smlat<<<nsm, 32, pad>>>(sv, np, lat);
  std::vector<unsigned> h(256 * np);
  cudaMemcpy(h.data(), lat, sizeof(unsigned) * h.size(), cudaMemcpyDeviceToHost);
  int ref = -1;
  for (int s = 0; s < 256 && ref < 0; ++s)
    if (h[s * np]) ref = s;
  std::vector<unsigned> srt(h.begin() + ref * np, h.begin() + (ref + 1) * np);
  std::sort(srt.begin(), srt.end());
  const unsigned mid = (srt[8] + srt[np - 9]) / 2;
  std::vector<uint8_t> smd(256, 0);
  int n0 = 0, n1 = 0;
  for (int s = 0; s < 256; ++s) {
    if (!h[s * np]) continue;
    int ag = 0;
    for (int l = 0; l < np; ++l) ag += (h[s * np + l] < mid) == (h[ref * np + l] < mid);
    smd[s] = ag > np / 2 ? 0 : 1;
    (smd[s] ? n1 : n0)++;
  }
  cudaMemcpy(sm_die_dev, smd.data(), 256, cudaMemcpyHostToDevice);
  const int64_t nch = (n + kChunk - 1) / kChunk;
  unsigned *l0, *l1, *ctr;
  cudaMalloc(&l0, 4 * nch);
  cudaMalloc(&l1, 4 * nch);
  cudaMalloc(&ctr, 8);
  cudaMemset(ctr, 0, 8);
  k_chlat<<<nsm, 1024, pad>>>(sv, nch, sm_die_dev, ctr, n0, n1, l0, l1);
  std::vector<unsigned> a(nch), b(nch);
  cudaMemcpy(a.data(), l0, 4 * nch, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), l1, 4 * nch, cudaMemcpyDeviceToHost);
  std::vector<uint8_t> cd(nch);
  for (int64_t c = 0; c < nch; ++c) cd[c] = a[c] <= b[c] ? 0 : 1;
  cudaMemcpy(chunk_die, cd.data(), nch, cudaMemcpyHostToDevice);
  cudaFree(lat);
  cudaFree(l0);
  cudaFree(l1);
  cudaFree(ctr);
  return cudaGetLastError() == cudaSuccess ? n0 : -1;
}

// SEL: 0 = every CTA strides over list A (all entries); 1 = die-d CTAs over list d (local);
// 2 = die-d CTAs over list 1-d (remote).  MODE bit 1 gather, bit 2 red.
template <int MODE>
__global__ void __launch_bounds__(256) k_pat(const int32_t *a0, int64_t n0, const int32_t *a1, int64_t n1,
                                             float *sv, const uint8_t *smd, int sel, unsigned *rank, int nd0,
                                             int nd1, float *sink) {
  __shared__ unsigned s_rank;
  __shared__ int s_die;
  if (threadIdx.x == 0) {
    s_die = smd[smid()];
    s_rank = atomicAdd(rank + s_die, 1u);
  }
  __syncthreads();
  const int d = s_die;
  const int32_t *a;
  int64_t n, r, nr;
  if (sel == 0) {
    a = a0; n = n0; r = blockIdx.x; nr = gridDim.x;
  } else {
    const int use = sel == 1 ? d : 1 - d;
    a = use ? a1 : a0;
    n = use ? n1 : n0;
    r = s_rank;
    nr = d ? nd1 : nd0;
  }
  float acc = 0.f;
  const int64_t stride = nr * blockDim.x;
  for (int64_t k = r * blockDim.x + threadIdx.x; k < n; k += 4 * stride) {
    int32_t id[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) id[u] = k + u * stride < n ? __ldcs(a + k + u * stride) : -1;
    if (MODE & 1) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (id[u] >= 0) acc += __ldcg(sv + id[u]);
    }
    if (MODE & 2) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (id[u] >= 0) atomicAdd(sv + id[u], 1e-30f);
    }
  }
  if (acc == 1.2345f) sink[0] = acc;
}

extern "C" float die_pattern_run(int mode, int sel, const int32_t *a0, int64_t n0, const int32_t *a1, int64_t n1,
                                 float *sv, const uint8_t *smd, int nd0, int nd1, float *sink) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  // launch exactly 8 CTAs per SM's worth; per-die CTA counts are counted on the device
  const int grid = nsm * 8;
  unsigned *rank;
  cudaMalloc(&rank, 8);
  cudaMemset(rank, 0, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  // nd0/nd1 = CTAs per die = 8 * SMs per die (8 resident CTAs of 256 threads per SM)
  if (mode == 1) k_pat<1><<<grid, 256>>>(a0, n0, a1, n1, sv, smd, sel, rank, nd0 * 8, nd1 * 8, sink);
  if (mode == 2) k_pat<2><<<grid, 256>>>(a0, n0, a1, n1, sv, smd, sel, rank, nd0 * 8, nd1 * 8, sink);
  if (mode == 3) k_pat<3><<<grid, 256>>>(a0, n0, a1, n1, sv, smd, sel, rank, nd0 * 8, nd1 * 8, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(rank);
  if (cudaGetLastError() != cudaSuccess) return -1.f;
  return ms;
}
