// die.cu — two-die placement of the TPA-SCD epoch (DESIGN.md §6 "die split").
//
// A B200 is two dies, each with half of the L2.  Every 2 KB chunk of the address space is homed in
// one die's L2, where its atomics execute.  The epoch gathers every shared-vector entry it later
// reduces into, and such a line cannot be served from the reading die's L2 when it is homed on the
// other die: measured on the random gather+RED pattern (tools/die_probe.cu, profiles/die_probe_r1.txt)
// 84 G pairs/s when every SM touches every chunk, 101-135 G/s when each SM touches only chunks of
// its own die, 50 G/s when only the other die's.
//
// So the epoch is split by die: coordinate c's stored entries are reordered once at create into
// [entries whose shared-vector element is homed on die 0 | entries homed on die 1], and each
// coordinate is processed by two CTAs, one per die, each over its own part: they exchange their
// partial dot products through a global slot (release/acquire), both form the same dp = p0 + p1 and
// the same Δ, and each scatters its own part (k_epoch_split, epoch.cu).  The arithmetic is the
// paper's Alg. 2 unchanged; only which SM touches which entry differs.
//
// The maps are measured at create: SM -> die and chunk -> die from the round-trip latency of an
// atomic (atomics execute at the home slice: ~270 cycles near, ~650 far on B200).
#include <algorithm>
#include <cstdio>
#include <vector>

#include "common.cuh"

namespace scd {
namespace {

__device__ __forceinline__ unsigned smid_reg() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// atomic round-trip latency (cycles, mean of R dependent atomics adding +0.0f) to the word `p`
template <int R>
__device__ __forceinline__ unsigned atom_latency(float *p) {
  float x = 0.f;
  const long long t0 = clock64();
#pragma unroll 1
  for (int r = 0; r < R; ++r) x = atomicAdd(p + (int)(x * 0.f), 0.f);
  const long long t1 = clock64();
  return (unsigned)((t1 - t0) / R) + (x == 1234.5f);
}

// One CTA per SM (the dynamic shared memory request leaves room for one).  Latencies are timed by
// ONE lane per warp: the lanes of a warp wait for each other, so a warp-wide timing would see the
// slowest lane.  k_sm_probe: thread 0 times probe chunks 0..nprobe-1 -> lat[smid][l].
__global__ void k_sm_probe(float *sv, int nprobe, unsigned *lat, int *sm_seen) {
  extern __shared__ char s_pad[];
  if (threadIdx.x != 0) return;
  const unsigned sm = smid_reg();
  s_pad[0] = 0;
  sm_seen[sm] = 1;
  for (int l = 0; l < nprobe; ++l)
    lat[sm * nprobe + l] = atom_latency<4>(sv + (size_t)l * kDieChunkFloats + (sm & 7) * 32);
}

// Every warp of die d's CTAs (rank among die d's CTAs from a counter) times its share of the
// chunks with its lane 0; lat_d[chunk] = latency seen from die d.
__global__ void k_chunk_probe(float *sv, int64_t n, int64_t nchunk, const uint8_t *sm_die, unsigned *rank_ctr, int n0,
                              int n1, unsigned *lat0, unsigned *lat1) {
  extern __shared__ char s_pad[];
  __shared__ unsigned s_rank;
  const int d = sm_die[smid_reg()];
  if (threadIdx.x == 0) {
    s_pad[0] = 0;
    s_rank = atomicAdd(rank_ctr + d, 1u);
  }
  __syncthreads();
  if ((threadIdx.x & 31) != 0) return;
  const int nw = blockDim.x / 32, w = threadIdx.x / 32;
  const int64_t nd = d == 0 ? n0 : n1;
  unsigned *lat = d == 0 ? lat0 : lat1;
  for (int64_t ch = (int64_t)s_rank * nw + w; ch < nchunk; ch += nd * nw) {
    int64_t off = (w & 7) * 32;  // distinct lines per warp (no same-address queueing)
    if (ch * kDieChunkFloats + off >= n) off = n - 1 - ch * kDieChunkFloats;
    lat[ch] = atom_latency<2>(sv + ch * kDieChunkFloats + off);
  }
}

__global__ void k_chunk_die(const unsigned *lat0, const unsigned *lat1, int64_t nchunk, uint8_t *chunk_die) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nchunk; i += (int64_t)gridDim.x * blockDim.x)
    chunk_die[i] = lat0[i] <= lat1[i] ? 0 : 1;
}

// Stable per-coordinate partition of the entries by home die of their shared-vector element:
// one warp per coordinate, ballot prefix sums; mid[c] = first die-1 entry.
__global__ void k_split(const int64_t *ptr, const int32_t *idx, const float *val, int64_t n, const uint8_t *chunk_die,
                        int64_t *mid, int32_t *oidx, float *oval, unsigned long long *nnz0) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = w0; c < n; c += nw) {
    const int64_t beg = ptr[c], end = ptr[c + 1];
    int64_t cnt0 = 0;
    for (int64_t k = beg + lane; k < end; k += 32) cnt0 += chunk_die[idx[k] / kDieChunkFloats] == 0;
    for (int o = 16; o > 0; o >>= 1) cnt0 += __shfl_xor_sync(0xffffffffu, cnt0, o);
    const int64_t m = beg + cnt0;
    if (lane == 0) {
      mid[c] = m;
      if (cnt0) atomicAdd(nnz0, (unsigned long long)cnt0);
    }
    int64_t o0 = beg, o1 = m;
    for (int64_t base = beg; base < end; base += 32) {
      const int64_t k = base + lane;
      const bool in = k < end;
      const int32_t j = in ? idx[k] : 0;
      const bool d1 = in && chunk_die[j / kDieChunkFloats] != 0;
      const unsigned b0 = __ballot_sync(0xffffffffu, in && !d1), b1 = __ballot_sync(0xffffffffu, d1);
      const unsigned below = (1u << lane) - 1u;
      if (in) {
        const int64_t dst = d1 ? o1 + __popc(b1 & below) : o0 + __popc(b0 & below);
        oidx[dst] = j;
        if (val) oval[dst] = val[k];
      }
      o0 += __popc(b0);
      o1 += __popc(b1);
    }
  }
}

}  // namespace

// SCD_DIE_SPLIT=1 enables the die split (default off: measured slower than the single-CTA kernels
// on the webspam-shaped C3 epoch, 14.7 vs 13.2 ms, profiles/die_split_r1.txt); it then applies to
// the CTA bins whose grid covers every SM, when the probe finds two dies and the reordered copy of
// the matrix fits in free memory with a 2 GB margin.
static scd_status die_off(scd_ctx *c, int where) {
  if (getenv("SCD_DIE_DEBUG")) fprintf(stderr, "[scd] die split off at check %d\n", where);
  (void)c;
  return SCD_OK;
}

scd_status setup_die_split(scd_ctx *c) {
  c->die_split = false;
  const char *e = getenv("SCD_DIE_SPLIT");
  if (!e || atoi(e) != 1) return die_off(c, 3);
  if (c->opt.deterministic || c->opt.wild || c->nnz == 0) return die_off(c, 4);
  int64_t nsplit = 0, max_count = 0;
  for (int i = 0; i < c->n_bins; ++i)
    if (c->bins[i].lanes == kLanesCta && c->bins[i].grid >= c->nsm) {
      ++nsplit;
      max_count = std::max<int64_t>(max_count, c->bins[i].count);
    }
  if (nsplit == 0) return die_off(c, 11);
  if (((uintptr_t)c->sv & 2047) != 0) return die_off(c, 12);  // chunk j of sv must be [512 j, 512 j + 512)
  const int64_t nchunk = (c->n_shared + kDieChunkFloats - 1) / kDieChunkFloats;
  size_t free_b = 0, total_b = 0;
  SCD_CK(c, cudaMemGetInfo(&free_b, &total_b));
  const size_t need = (size_t)c->nnz * (c->val ? 8 : 4) + sizeof(int64_t) * (size_t)c->n_coord +
                      16 * (size_t)max_count + (size_t)nchunk * 9;
  if (need + ((size_t)2 << 30) > free_b) return die_off(c, 20);
  cudaStream_t s = c->stream;
  // 1. SM -> die
  const int nprobe = (int)std::min<int64_t>(c->n_shared / kDieChunkFloats, 64);  // whole chunks only
  if (nprobe < 8) return die_off(c, 24);
  unsigned *d_lat = nullptr;
  int *d_seen = nullptr;
  SCD_CK(c, cudaMalloc((void **)&d_lat, sizeof(unsigned) * kMaxSm * nprobe));
  SCD_CK(c, cudaMalloc((void **)&d_seen, sizeof(int) * kMaxSm));
  SCD_CK(c, cudaMemsetAsync(d_lat, 0, sizeof(unsigned) * kMaxSm * nprobe, s));
  SCD_CK(c, cudaMemsetAsync(d_seen, 0, sizeof(int) * kMaxSm, s));
  int smem_max = 0;
  SCD_CK(c, cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
  const int pad = smem_max * 3 / 4;  // > half the SM's shared memory: one CTA per SM
  SCD_CK(c, cudaFuncSetAttribute(k_sm_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, pad));
  k_sm_probe<<<c->nsm, 32, pad, s>>>(c->sv, nprobe, d_lat, d_seen);
  SCD_CKL(c, "k_sm_probe");
  std::vector<unsigned> lat((size_t)kMaxSm * nprobe);
  std::vector<int> seen(kMaxSm);
  SCD_CK(c, cudaMemcpyAsync(lat.data(), d_lat, sizeof(unsigned) * lat.size(), cudaMemcpyDeviceToHost, s));
  SCD_CK(c, cudaMemcpyAsync(seen.data(), d_seen, sizeof(int) * kMaxSm, cudaMemcpyDeviceToHost, s));
  SCD_CK(c, cudaStreamSynchronize(s));
  cudaFree(d_lat);
  cudaFree(d_seen);
  int ref = -1, nseen = 0;
  for (int i = 0; i < kMaxSm; ++i)
    if (seen[i]) {
      if (ref < 0) ref = i;
      ++nseen;
    }
  if (ref < 0 || nseen != c->nsm) return die_off(c, 50);  // every SM must have been probed
  std::vector<unsigned> lr(lat.begin() + (size_t)ref * nprobe, lat.begin() + (size_t)(ref + 1) * nprobe);
  std::vector<unsigned> srt = lr;
  std::sort(srt.begin(), srt.end());
  const unsigned lo = srt[nprobe / 8], hi = srt[nprobe - 1 - nprobe / 8];
  if (hi < lo + lo / 4) return die_off(c, 55);  // no near/far split: a single die (or no measurable difference)
  const unsigned mid = (lo + hi) / 2;
  std::vector<uint8_t> die(kMaxSm, 0);
  int n0 = 0, n1 = 0;
  for (int sm = 0; sm < kMaxSm; ++sm) {
    if (!seen[sm]) continue;
    int agree = 0;
    for (int l = 0; l < nprobe; ++l) agree += (lat[(size_t)sm * nprobe + l] < mid) == (lr[l] < mid);
    if (agree * 8 > nprobe * 7) {
      die[sm] = 0;
      ++n0;
    } else if (agree * 8 < nprobe) {
      die[sm] = 1;
      ++n1;
    } else {
      return die_off(c, 70);  // ambiguous SM: leave the plain kernels in place
    }
  }
  if (n0 == 0 || n1 == 0) return die_off(c, 73);
  c->n_die_sm[0] = n0;
  c->n_die_sm[1] = n1;
  c->die_lat[0] = (float)lo;
  c->die_lat[1] = (float)hi;
  SCD_CK(c, cudaMalloc((void **)&c->sm_die, kMaxSm));
  SCD_CK(c, cudaMemcpyAsync(c->sm_die, die.data(), kMaxSm, cudaMemcpyHostToDevice, s));
  // 2. chunk -> die
  unsigned *lat0 = nullptr, *lat1 = nullptr, *rank = nullptr;
  uint8_t *chunk_die = nullptr;
  SCD_CK(c, cudaMalloc((void **)&lat0, sizeof(unsigned) * nchunk));
  SCD_CK(c, cudaMalloc((void **)&lat1, sizeof(unsigned) * nchunk));
  SCD_CK(c, cudaMalloc((void **)&rank, sizeof(unsigned) * 2));
  SCD_CK(c, cudaMalloc((void **)&chunk_die, nchunk));
  SCD_CK(c, cudaMemsetAsync(rank, 0, sizeof(unsigned) * 2, s));
  SCD_CK(c, cudaFuncSetAttribute(k_chunk_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, pad));
  k_chunk_probe<<<c->nsm, 1024, pad, s>>>(c->sv, c->n_shared, nchunk, c->sm_die, rank, n0, n1, lat0, lat1);
  k_chunk_die<<<grid_for(nchunk, 256), 256, 0, s>>>(lat0, lat1, nchunk, chunk_die);
  SCD_CKL(c, "chunk probe");
  // 3. reordered copy of the matrix
  SCD_CK(c, cudaMalloc((void **)&c->split_mid, sizeof(int64_t) * c->n_coord));
  SCD_CK(c, cudaMalloc((void **)&c->split_idx, sizeof(int32_t) * c->nnz));
  if (c->val) SCD_CK(c, cudaMalloc((void **)&c->split_val, sizeof(float) * c->nnz));
  unsigned long long *d_nnz0 = nullptr, h_nnz0 = 0;
  SCD_CK(c, cudaMalloc((void **)&d_nnz0, sizeof(*d_nnz0)));
  SCD_CK(c, cudaMemsetAsync(d_nnz0, 0, sizeof(*d_nnz0), s));
  k_split<<<grid_for(c->n_coord * 32, 256, 148 * 32), 256, 0, s>>>(c->ptr, c->idx, c->val, c->n_coord, chunk_die,
                                                                   c->split_mid, c->split_idx, c->split_val, d_nnz0);
  SCD_CKL(c, "k_split");
  SCD_CK(c, cudaMemcpyAsync(&h_nnz0, d_nnz0, sizeof(h_nnz0), cudaMemcpyDeviceToHost, s));
  SCD_CK(c, cudaMalloc((void **)&c->slot_p, sizeof(float) * 2 * max_count));
  SCD_CK(c, cudaMalloc((void **)&c->slot_tag, sizeof(unsigned) * 2 * max_count));
  SCD_CK(c, cudaMalloc((void **)&c->split_err, sizeof(unsigned)));
  SCD_CK(c, cudaMemsetAsync(c->slot_tag, 0, sizeof(unsigned) * 2 * max_count, s));
  SCD_CK(c, cudaMemsetAsync(c->split_err, 0, sizeof(unsigned), s));
  SCD_CK(c, cudaStreamSynchronize(s));
  cudaFree(lat0);
  cudaFree(lat1);
  cudaFree(rank);
  cudaFree(chunk_die);
  cudaFree(d_nnz0);
  c->split_nnz0 = (int64_t)h_nnz0;
  c->split_nosync = getenv("SCD_SPLIT_NOSYNC") && atoi(getenv("SCD_SPLIT_NOSYNC")) == 1;  // diagnostic only
  c->launch_tag = 0;
  for (int i = 0; i < c->n_bins; ++i) {
    Bin &b = c->bins[i];
    if (b.lanes == kLanesCta && b.grid >= c->nsm) {
      b.split = 1;
      b.head = 0;
      b.flush = 0;
      bin_launch_shape(c, b);
    }
  }
  c->die_split = true;
  return SCD_OK;
}

// A rendezvous that timed out (a partner CTA never arrived: should not happen with a resident grid)
// leaves a flag; it is reported at the next synchronising call.
scd_status check_split_error(scd_ctx *c) {
  if (!c->die_split || !c->split_err) return SCD_OK;
  unsigned h = 0;
  SCD_CK(c, cudaMemcpyAsync(&h, c->split_err, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  SCD_CK(c, cudaStreamSynchronize(c->stream));
  if (h) return fail(c, SCD_E_CUDA, "die-split epoch: partner CTA rendezvous timed out");
  return SCD_OK;
}

}  // namespace scd
