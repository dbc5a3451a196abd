// pattern_bench.cu — the epoch's memory access pattern without the algorithm's dependencies:
// stream (idx, val), gather sv[idx], red.add sv[idx] for every stored entry, grid-stride over
// all entries in storage order (no per-coordinate reduction, no delta, no ordering).  Its time is
// the ceiling of the access pattern that the epoch kernels are measured against (tools/ only).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o tools/libpattern.so tools/pattern_bench.cu
#include <cstdint>
#include <cuda_runtime.h>

// MODE bit 0: gather, bit 1: RED, bit 2: gather from svr (a second vector: the epoch kernels' tail
// read copy) instead of sv
template <int MODE>
__global__ void __launch_bounds__(256) k_pattern(const int32_t *__restrict__ idx, const float *__restrict__ val,
                                                 int64_t nnz, float *sv, float *sink, const float *svr = nullptr) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += 4 * stride) {
    int32_t id[4];
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t kk = k + u * stride;
      id[u] = kk < nnz ? __ldcs(idx + kk) : -1;
      v[u] = kk < nnz ? __ldcs(val + kk) : 0.f;
    }
    if (MODE & 1) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (id[u] >= 0) acc += __ldcg((MODE & 4 ? svr : sv) + id[u]) * v[u];
    }
    if (MODE & 2) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (id[u] >= 0) atomicAdd(sv + id[u], v[u] * 1e-30f);
    }
  }
  if (acc == 1.2345f) sink[0] = acc;
}

extern "C" float pattern_run2(int mode, const int32_t *idx, const float *val, int64_t nnz, float *sv, const float *svr,
                              float *sink) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = nsm * 8;
  cudaEventRecord(a);
  if (mode == 0) k_pattern<0><<<grid, 256>>>(idx, val, nnz, sv, sink);
  if (mode == 1) k_pattern<1><<<grid, 256>>>(idx, val, nnz, sv, sink);
  if (mode == 2) k_pattern<2><<<grid, 256>>>(idx, val, nnz, sv, sink);
  if (mode == 3) k_pattern<3><<<grid, 256>>>(idx, val, nnz, sv, sink);
  if (mode == 7) k_pattern<7><<<grid, 256>>>(idx, val, nnz, sv, sink, svr);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms;
}

extern "C" float pattern_run(int mode, const int32_t *idx, const float *val, int64_t nnz, float *sv, float *sink) {
  return pattern_run2(mode, idx, val, nnz, sv, nullptr, sink);
}
