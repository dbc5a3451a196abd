// Microbenchmark: random 4-byte gathers from distributed shared memory (a cluster-resident copy of
// a vector) against the same gathers from L2, and DSMEM vs L2 reductions, on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dsmem_bench tools/dsmem_bench.cu && /tmp/dsmem_bench
// Question it answers: can the webspam-shaped dual's tail read copy (2.7 MB) live
// in the shared memory of a thread-block cluster, taking its ~2100 gathers per row off the L2?
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// mode 0: DSMEM gathers, 1: DSMEM red.add, 2: DSMEM gathers + L2 REDs to a separate vector (the
// proposed epoch mix), 3: local-smem gathers only (upper bound)
template <int MODE>
__global__ void k_dsmem(int slice, int iters, float *red_vec, int red_n, float *sink) {
  extern __shared__ float s[];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks();
  for (int i = threadIdx.x; i < slice; i += blockDim.x) s[i] = (float)i;
  cl.sync();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(s);
  float acc = 0.f;
  uint32_t st = hsh(blockIdx.x * 1024u + threadIdx.x);
  const uint32_t n = (uint32_t)slice * (uint32_t)CL;
  for (int it = 0; it < iters; ++it) {
    uint32_t addr[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      st = hsh(st + u);
      const uint32_t id = st % n;
      const uint32_t r = MODE == 3 ? 0u : id / (uint32_t)slice, off = id % (uint32_t)slice;
      if (MODE == 3) {
        addr[u] = base + 4u * off;
      } else {
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr[u]) : "r"(base + 4u * off), "r"(r));
      }
    }
    if (MODE == 1) {
#pragma unroll
      for (int u = 0; u < 8; ++u) asm volatile("red.shared::cluster.add.f32 [%0], %1;" ::"r"(addr[u]), "f"(1.0f) : "memory");
    } else {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (MODE == 3)
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[u]) : "r"(addr[u]));
        else
          asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v[u]) : "r"(addr[u]));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
      if (MODE == 2) {
#pragma unroll
        for (int u = 0; u < 8; ++u) atomicAdd(red_vec + (hsh(st ^ (u * 77u)) % (uint32_t)red_n), 1e-9f);
      }
    }
  }
  cl.sync();
  if (acc == 1.2345f) sink[0] = acc;
}

// the same gathers from global memory (L2-resident vector of slice*CL floats)
__global__ void k_l2(const float *v, int n, int iters, float *red_vec, int red_n, int mode, float *sink) {
  float acc = 0.f;
  uint32_t st = hsh(blockIdx.x * 1024u + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
    float x[8];
    uint32_t id[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      st = hsh(st + u);
      id[u] = st % (uint32_t)n;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldcg(v + id[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += x[u];
    if (mode == 1) {
#pragma unroll
      for (int u = 0; u < 8; ++u) atomicAdd(red_vec + (hsh(st ^ (u * 77u)) % (uint32_t)red_n), 1e-9f);
    }
  }
  if (acc == 1.2345f) sink[0] = acc;
}

template <int MODE>
float run_cluster(int CL, int slice, int iters, float *red, int red_n, float *sink, int *nclusters) {
  auto fn = k_dsmem<MODE>;
  const size_t smem = sizeof(float) * (size_t)slice;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (CL > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(CL);
  int ncl = 0;
  cudaOccupancyMaxActiveClusters(&ncl, (void *)fn, &cfg);
  *nclusters = ncl;
  if (ncl < 1) return -1.f;
  cfg.gridDim = dim3(CL * ncl);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, fn, slice, 2, red, red_n, sink);  // warm-up
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, fn, slice, iters, red, red_n, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return -1.f;
  }
  return ms;
}

int main() {
  const int red_n = 2700000 / 4 * 4;
  float *red, *vec, *sink;
  cudaMalloc(&red, sizeof(float) * red_n);
  cudaMalloc(&vec, sizeof(float) * 16 * 45056);
  cudaMalloc(&sink, 64);
  cudaMemset(red, 0, sizeof(float) * red_n);
  cudaMemset(vec, 0, sizeof(float) * 16 * 45056);
  const int iters = 200;
  const char *names[] = {"dsmem gather", "dsmem red.add", "dsmem gather + L2 RED (2.7 MB)", "local smem gather"};
  for (int CL : {2, 4, 8, 16}) {
    const int slice = CL == 16 ? 43008 : 45056;  // floats per CTA (168 / 176 KB)
    for (int mode = 0; mode < 4; ++mode) {
      int ncl = 0;
      float ms = mode == 0 ? run_cluster<0>(CL, slice, iters, red, red_n, sink, &ncl)
               : mode == 1 ? run_cluster<1>(CL, slice, iters, red, red_n, sink, &ncl)
               : mode == 2 ? run_cluster<2>(CL, slice, iters, red, red_n, sink, &ncl)
                           : run_cluster<3>(CL, slice, iters, red, red_n, sink, &ncl);
      if (ms <= 0) {
        printf("CL=%2d %-32s: not launchable (clusters %d)\n", CL, names[mode], ncl);
        continue;
      }
      const double ops = (double)ncl * CL * 1024.0 * iters * 8;
      printf("CL=%2d clusters=%2d SMs=%3d %-32s: %8.3f ms  %7.1f G ops/s  (%.2f ops/clk/SM at 1.965 GHz)\n", CL, ncl,
             ncl * CL, names[mode], ms, ops / ms / 1e6, ops / ms / 1e6 / (ncl * CL) / 1.965);
    }
  }
  // L2 reference: 148 CTAs x 1024 threads, vector of 2.7 MB
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 2; ++mode) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_l2<<<nsm, 1024>>>(vec, 16 * 42000, 2, red, red_n, mode, sink);
    cudaEventRecord(e0);
    k_l2<<<nsm, 1024>>>(vec, 16 * 42000, iters, red, red_n, mode, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)nsm * 1024.0 * iters * 8;
    printf("L2 (148 CTAs x 1024) %-32s: %8.3f ms  %7.1f G ops/s\n", mode ? "gather + RED (2.7 MB)" : "gather (2.7 MB)", ms,
           ops / ms / 1e6);
  }
  return 0;
}
