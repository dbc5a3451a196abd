// l2_bench.cu — microbenchmark of the L2-resident random access patterns of the TPA-SCD epoch
// (SURVEY §7 hard part 2: "L2 atomic throughput ... must be microbenchmarked first").
// Measures, on an L2-resident fp32 vector of `n` entries, the rate of
//   gather: random 4-byte loads (ld.global.cg, L2-coherent)
//   red   : random 4-byte red.global.add.f32
//   both  : one gather and one red per element (the epoch's inner pattern)
// Indices come from a counter hash, so no HBM traffic is involved.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bench tools/l2_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int MODE, int U>
__global__ void __launch_bounds__(256) k(float *v, unsigned n, unsigned iters, float *sink) {
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  for (unsigned it = 0; it < iters; ++it) {
    unsigned id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) id[u] = hash32(tid * 7919u + (it * U + u) * 104729u) % n;
    if (MODE != 1) {
#pragma unroll
      for (int u = 0; u < U; ++u) acc += __ldcg(v + id[u]);
    }
    if (MODE == 1 || MODE == 2) {
#pragma unroll
      for (int u = 0; u < U; ++u) atomicAdd(v + id[u], 1e-9f);
    }
    if (MODE == 3) {  // gather from v, RED into a second vector (different lines)
#pragma unroll
      for (int u = 0; u < U; ++u) atomicAdd(v + n + id[u], 1e-9f);
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main(int argc, char **argv) {
  unsigned n = argc > 1 ? atoi(argv[1]) : 680715;
  float *v, *sink;
  cudaMalloc(&v, sizeof(float) * n * 2);
  cudaMalloc(&sink, 4);
  cudaMemset(v, 0, sizeof(float) * n * 2);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * 8, block = 256;
  const unsigned iters = 256;
  const double ops = (double)grid * block * iters * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char *names[4] = {"gather", "red", "gather+red", "gather+red(2 vectors)"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0, 8><<<grid, block>>>(v, n, iters, sink);
      if (mode == 1) k<1, 8><<<grid, block>>>(v, n, iters, sink);
      if (mode == 2) k<2, 8><<<grid, block>>>(v, n, iters, sink);
      if (mode == 3) k<3, 8><<<grid, block>>>(v, n, iters, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("%-22s n=%u: %.1f G elements/s (%.3f ms)\n", names[mode], n, ops / ms / 1e6, ms);
    }
  }
  return 0;
}
