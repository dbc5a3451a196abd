// red_bench.cu — cost model of L2 fp32 reductions on B200 (which unit of work an L2 atomic costs:
// an element, a sector or a request), to decide how the epoch's scatter should be shaped.
// Every mode issues the same number of fp32 element additions into an L2-resident vector of n
// floats; only the grouping differs:
//   rand1     : random element per lane (1 element per sector per request)          — the tail
//   line1     : a warp covers one random 128-byte line, scalar red per lane         — dense run
//   line_v4   : a warp covers 4 random consecutive lines with red.global.add.v4.f32 — vector red
//   hot1      : every warp hits one of `hot` fixed lines (the dense head), scalar red
//   hot_v4    : same hot lines, v4 red
//   gat_line  : a warp gathers one random line (coalesced ld.global.cg), for comparison
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_bench tools/red_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ void red_v4(float *p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// each iteration every lane adds 4 elements (so all modes do 4 element-adds per lane-iteration)
template <int MODE>
__global__ void __launch_bounds__(256) k(float *v, unsigned n, unsigned hot, unsigned iters, float *sink) {
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned lane = threadIdx.x & 31, warp = tid >> 5;
  const unsigned nlines = n / 32;
  float acc = 0.f;
  for (unsigned it = 0; it < iters; ++it) {
    const unsigned r = hash32(warp * 7919u + it * 104729u);
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) atomicAdd(v + hash32(tid * 7919u + (it * 4 + u) * 104729u) % n, 1e-9f);
    } else if (MODE == 1) {
#pragma unroll
      for (int u = 0; u < 4; ++u) atomicAdd(v + ((r + u * 977u) % nlines) * 32 + lane, 1e-9f);
    } else if (MODE == 2) {
      const unsigned base = (r % (nlines / 4)) * 128;
      red_v4(v + base + lane * 4, 1e-9f, 1e-9f, 1e-9f, 1e-9f);
    } else if (MODE == 3) {
#pragma unroll
      for (int u = 0; u < 4; ++u) atomicAdd(v + ((r + u) % hot) * 32 + lane, 1e-9f);
    } else if (MODE == 4) {
      const unsigned base = ((r % hot) & ~3u) * 32;
      red_v4(v + base + lane * 4, 1e-9f, 1e-9f, 1e-9f, 1e-9f);
    } else if (MODE == 5) {
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += __ldcg(v + ((r + u * 977u) % nlines) * 32 + lane);
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main(int argc, char **argv) {
  unsigned n = argc > 1 ? atoi(argv[1]) : 680715;
  unsigned hot = argc > 2 ? atoi(argv[2]) : 64;
  n = n / 128 * 128;
  float *v, *sink;
  cudaMalloc(&v, sizeof(float) * n);
  cudaMalloc(&sink, 4);
  cudaMemset(v, 0, sizeof(float) * n);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * 8, block = 256;
  const unsigned iters = 256;
  const double elems = (double)grid * block * iters * 4;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char *names[6] = {"rand1", "line1", "line_v4", "hot1", "hot_v4", "gat_line"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      switch (mode) {
        case 0: k<0><<<grid, block>>>(v, n, hot, iters, sink); break;
        case 1: k<1><<<grid, block>>>(v, n, hot, iters, sink); break;
        case 2: k<2><<<grid, block>>>(v, n, hot, iters, sink); break;
        case 3: k<3><<<grid, block>>>(v, n, hot, iters, sink); break;
        case 4: k<4><<<grid, block>>>(v, n, hot, iters, sink); break;
        case 5: k<5><<<grid, block>>>(v, n, hot, iters, sink); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2)
        printf("%-9s n=%u hot=%u lines: %7.1f G elements/s  %7.2f G sectors/s (%.3f ms)\n", names[mode], n, hot,
               elems / ms / 1e6, (mode == 0 ? elems : elems / 8) / ms / 1e6, ms);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
