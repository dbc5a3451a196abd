// epoch.cu — the TPA-SCD epoch kernels (Alg. 2) for sm_100a.
//
// One epoch updates every local coordinate exactly once, in the order of the epoch
// permutation, by the closed-form rule
//   primal (CSC, Eq. 2):  Δβ_m = (<y - w, a_m> - λNβ_m) / (||a_m||² + λN)
//   dual   (CSR, Eq. 4): Δα_n = (λy_n - <w̄, ā_n> - λNα_n) / (λN + ||ā_n||²)
// followed by the shared-vector update w += a_m Δβ / w̄ += ā_n Δα written with
// fp32 atomic adds ("floating point atomic additions", Alg. 2).  The primal keeps
// the residual r = y - w instead of w, so the gather reads one vector (design note).
//
// Kernels:
//   k_epoch_cta<FORM,T,E>    one coordinate per CTA (the paper's "thread block per coordinate",
//                            P:190), persistent grid with a global ticket counter; each thread
//                            keeps E entries of the coordinate in registers between the gather-dot
//                            and the scatter (no HBM re-read), longer coordinates stream extra chunks.
//   k_epoch_group<FORM,G,E>  one coordinate per G-lane sub-warp group (short coordinates: a whole
//                            CTA would idle), warp-shuffle reduction, E entries per lane in registers.
//   k_epoch_debug<FORM>      deterministic mode: one CTA, one coordinate at a time in exact P_t
//                            order, fixed reduction tree -> bitwise repeatable (oracle parity).
//   k_empty_fix<FORM>        coordinates with no stored entry: Δ = -β_m (primal) / y_n/N - α_n (dual)
//                            (c17); only re-run when the model was set externally.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"

namespace scd {
namespace {

struct EpochArgs {
  const int64_t *__restrict__ ptr;
  const int32_t *__restrict__ idx;
  const float *__restrict__ val;
  const float *__restrict__ y;
  const float *__restrict__ norm;
  float *x;
  float *sv;
  const float *svr;  // head kernel with a tail read copy: gathers of ids >= H read svr (else == sv)
  const float *svg;  // gather source of the plain kernels: sv, or svr for a snapshot bin (Bin::snap)
  double lam, lamN;
  int64_t roll_R;          // head kernel, rolling tail copy: every roll_R-th row refreshes one chunk (0 = off)
  int64_t head_P;          // head kernel, head copy in svr[0, H): every head_P-th row refreshes one chunk (0 = off)
  int64_t roll_lo, roll_hi;  // the tail range [roll_lo, roll_hi) kept in svr
};

struct BinArgs {
  const int32_t *list;  // coordinate ids of the bin (ascending); nullptr = identity
  int64_t lo, hi;       // this launch processes permutation positions [lo, hi) of the bin
  unsigned int *counter;
  Perm perm;
  int dry;  // 1 = layout probe: full gather/scatter traffic, model untouched, scatter adds +0.0f
};

// Closed-form coordinate delta (Eq. 2 / Eq. 4), scalar math in fp64 (free), result fp32.
template <int FORM>
__device__ __forceinline__ float coord_delta(float dp, float xc, float nrm, float yc, double lam, double lamN) {
  double num = (FORM == SCD_PRIMAL) ? ((double)dp - lamN * (double)xc)
                                    : (lam * (double)yc - (double)dp - lamN * (double)xc);
  return (float)(num / ((double)nrm + lamN));
}
// primal scatters into r = y - w (so -Δ), dual into w̄ (+Δ)
template <int FORM>
__device__ __forceinline__ float scatter_scale(float d) { return FORM == SCD_PRIMAL ? -d : d; }

// Shared-vector gather: L2-coherent load (bypasses L1) so a hot entry is never served stale
// from L1 while other SMs' atomics land in L2.
__device__ __forceinline__ float ld_sv(const float *p) { return __ldcg(p); }
__device__ __forceinline__ void red_add(float *p, float v) { atomicAdd(p, v); }  // RED.E.ADD.F32

// Scatter of U register-held entries (id < 0 = none).  Atomic: red.global.add.f32.  WILD (the
// PASSCoDe-Wild comparison, options.wild): plain load + store, all loads issued before the stores, so
// a concurrent update of the same entry between the two can be lost.
template <bool WILD, int U>
__device__ __forceinline__ void scatter_regs(float *sv, const int32_t *id, const float *v, float d) {
  if (WILD) {
    float o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) o[u] = id[u] >= 0 ? __ldcg(sv + id[u]) : 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (id[u] >= 0) __stcg(sv + id[u], o[u] + v[u] * d);
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (id[u] >= 0) red_add(sv + id[u], v[u] * d);
  }
}

// Partial dot over the entries k = k0 + j*stride (k < end) of a coordinate, U entries at a time:
// all U (idx, val) loads, then all U gathers, then the FMAs (U independent round trips in flight).
template <int U>
__device__ __forceinline__ float dot_strided(const float *sv, const int32_t *idx, const float *val, int64_t k0,
                                             int64_t end, int64_t stride) {
  float acc = 0.f;
  for (int64_t k = k0; k < end; k += stride * U) {
    int32_t id[U];
    float v[U], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t kk = k + (int64_t)u * stride;
      id[u] = kk < end ? __ldcg(idx + kk) : -1;
      v[u] = kk < end ? val_cg(val, kk) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) w[u] = id[u] >= 0 ? ld_sv(sv + id[u]) : 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u) acc = fmaf(w[u], v[u], acc);
  }
  return acc;
}

// Scatter of the entries k = k0 + j*stride (k < end) of a coordinate, U entries at a time
// with all their (idx, val) loads issued before the REDs (the compiler may not hoist loads above
// a RED it cannot prove does not alias them, which would serialise one L2 round trip per entry).
template <int U, bool WILD = false>
__device__ __forceinline__ void scatter_strided(float *sv, const int32_t *idx, const float *val, int64_t k0,
                                                int64_t end, int64_t stride, float d) {
  for (int64_t k = k0; k < end; k += stride * U) {
    int32_t id[U];
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t kk = k + (int64_t)u * stride;
      id[u] = kk < end ? __ldcg(idx + kk) : -1;
      v[u] = kk < end ? val_cg(val, kk) : 0.f;
    }
    scatter_regs<WILD, U>(sv, id, v, d);
  }
}

__device__ __forceinline__ int64_t bin_coord(const BinArgs &b, uint64_t t) {
  uint64_t j = perm_apply(b.perm, t);
  return b.list ? (int64_t)__ldg(b.list + j) : (int64_t)j;
}

// ----------------------------------------------------------------------------------------------
// Two-pass streaming CTA kernel (one coordinate per CTA).  Pass 1 streams the coordinate's
// (idx, val) from HBM with coalesced loads, U independent gathers in flight per thread; pass 2
// re-reads (idx, val) — now L2-resident — for the atomic scatter.  Holding nothing in registers
// between the passes keeps the kernel at ~32 registers, i.e. full occupancy (64 warps/SM), which
// is what hides the idx -> gather -> reduce -> scatter latency chain (the register-resident
// variant below ran at 50% occupancy and was latency-bound).  Thread 0 software-pipelines the
// schedule: the next ticket's atomic is issued before pass 1 and its coordinate / offsets are
// fetched before pass 2, so neither latency sits on the critical path.
template <int FORM, int T, int U, int MINB>
__global__ void __launch_bounds__(T, MINB) k_epoch_stream(EpochArgs a, BinArgs b) {
  constexpr int NW = T / 32;
  __shared__ float s_red[NW];
  __shared__ float s_delta;
  __shared__ long long s_c, s_beg, s_end;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // thread 0: schedule state for the next coordinate
  long long nc = -1, nbeg = 0, nend = 0;
  if (tid == 0) {
    const int64_t t = b.lo + (int64_t)atomicAdd(b.counter, 1u);
    if (t < b.hi) {
      nc = bin_coord(b, (uint64_t)t);
      nbeg = __ldg(a.ptr + nc);
      nend = __ldg(a.ptr + nc + 1);
    }
  }
  for (;;) {
    unsigned int nticket = 0;
    if (tid == 0) {
      s_c = nc;
      s_beg = nbeg;
      s_end = nend;
      if (nc >= 0) nticket = atomicAdd(b.counter, 1u);  // next ticket, consumed after pass 1
    }
    __syncthreads();
    const long long c = s_c;
    if (c < 0) break;
    const int64_t beg = s_beg, end = s_end;
    float xc = 0.f, nrm = 0.f, yc = 0.f;
    if (tid == 0) {  // consumed after the reduction
      xc = a.x[c];
      nrm = __ldg(a.norm + c);
      if (FORM == SCD_DUAL) yc = __ldg(a.y + c);
    }
    // pass 1: gather-dot
    float acc = 0.f;
    for (int64_t base = beg + tid; base < end; base += (int64_t)T * U) {
      int32_t id[U];
      float v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = base + (int64_t)u * T;
        id[u] = k < end ? __ldcg(a.idx + k) : -1;
        v[u] = k < end ? val_cg(a.val, k) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (id[u] >= 0) acc = fmaf(ld_sv(a.svg + id[u]), v[u], acc);
    }
    if (tid == 0) {  // schedule the next coordinate while the block reduces / scatters
      const int64_t t = b.lo + (int64_t)nticket;
      nc = -1;
      if (t < b.hi) {
        nc = bin_coord(b, (uint64_t)t);
        nbeg = __ldg(a.ptr + nc);
        nend = __ldg(a.ptr + nc + 1);
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) s_red[wid] = acc;
    __syncthreads();
    if (wid == 0) {
      float s = lane < NW ? s_red[lane] : 0.f;
      s = warp_sum(s);
      if (lane == 0) {
        const float d = coord_delta<FORM>(s, xc, nrm, yc, a.lam, a.lamN);
        if (!b.dry) a.x[c] = xc + d;  // single writer per epoch (c10)
        s_delta = b.dry ? 0.f : d;
      }
    }
    __syncthreads();
    const float d = scatter_scale<FORM>(s_delta);
    if (d != 0.f || b.dry) {
      for (int64_t base = beg + tid; base < end; base += (int64_t)T * U) {
        // all U (idx, val) loads first: the REDs may alias them as far as the compiler knows,
        // so interleaving would serialise one L2 round trip per entry
        int32_t id[U];
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t k = base + (int64_t)u * T;
          id[u] = k < end ? __ldcg(a.idx + k) : -1;
          v[u] = k < end ? val_cg(a.val, k) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (id[u] >= 0) red_add(a.sv + id[u], v[u] * d);
      }
    }
  }
}

// ----------------------------------------------------------------------------------------------
// Register-resident CTA kernel (first version, kept for comparison): E entries per thread held
// in registers between the gather-dot and the scatter.
template <int FORM, int T, int E, bool WILD = false>
__global__ void __launch_bounds__(T) k_epoch_cta(EpochArgs a, BinArgs b) {
  constexpr int NW = T / 32;
  __shared__ float s_red[NW];
  __shared__ float s_delta;
  __shared__ unsigned int s_ticket;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (;;) {
    if (tid == 0) s_ticket = atomicAdd(b.counter, 1u);
    __syncthreads();
    const int64_t t = b.lo + (int64_t)s_ticket;
    if (t >= b.hi) break;
    const int64_t c = bin_coord(b, t);
    const int64_t beg = __ldg(a.ptr + c), end = __ldg(a.ptr + c + 1);
    int32_t id[E];
    float v[E];
    float acc = 0.f;
    // first chunk: held in registers until the scatter
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t k = beg + (int64_t)e * T + tid;
      if (k < end) {
        id[e] = __ldcs(a.idx + k);
        v[e] = val_cs(a.val, k);
      } else {
        id[e] = -1;
        v[e] = 0.f;
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (id[e] >= 0) acc = fmaf(ld_sv(a.svg + id[e]), v[e], acc);
    // remaining chunks of a long coordinate (re-read for the scatter; L2-resident by then)
    acc += dot_strided<8>(a.svg, a.idx, a.val, beg + (int64_t)T * E + tid, end, T);
    acc = warp_sum(acc);
    if (lane == 0) s_red[wid] = acc;
    __syncthreads();
    if (wid == 0) {
      float s = lane < NW ? s_red[lane] : 0.f;
      s = warp_sum(s);
      if (lane == 0) {
        const float xc = a.x[c];
        const float d = coord_delta<FORM>(s, xc, __ldg(a.norm + c), FORM == SCD_DUAL ? __ldg(a.y + c) : 0.f,
                                          a.lam, a.lamN);
        if (!b.dry) a.x[c] = xc + d;  // single writer per epoch (c10)
        s_delta = b.dry ? 0.f : d;
      }
    }
    __syncthreads();
    const float d = scatter_scale<FORM>(s_delta);
    if (d != 0.f || b.dry) {  // dry probe: same traffic, adds +0.0f (state unchanged)
      scatter_regs<WILD, E>(a.sv, id, v, d);
      scatter_strided<8, WILD>(a.sv, a.idx, a.val, beg + (int64_t)T * E + tid, end, T, d);
    }
  }
}

// ----------------------------------------------------------------------------------------------
// Head-combining CTA kernel (dense head of a frequency-ranked shared vector, webspam-shaped dual).
// The L2 charges a reduction per 32-byte SECTOR, whatever number of fp32 elements of the sector it
// carries, and a line that every coordinate updates serialises in its slice (tools/red_bench.cu,
// profiles/red_bench_r1.txt).  The head [0, H) of w̄ is such a region: its entries are carried by
// most rows.  So each CTA keeps its own pending updates of the head in shared memory (s_acc[H])
// and flushes them every `flush` coordinates with one 16-byte red.global.add.v4.f32 per touched float4 — one L2 reduction per sector per `flush` rows instead of one per row.
// One coordinate at a time per CTA and unique indices within a coordinate make the shared-memory
// accumulation a plain read-modify-write (sm_100 has no native fp32 shared atomic add).
// The CTA reads the head as L2 value + its own pending value, so a CTA always sees its own
// updates; other CTAs' pending head updates are the extra staleness, at most (CTAs)·flush
// coordinates, which build_schedule keeps under the bin's cap.  Tail entries
// (id >= H) are gathered and reduced in L2 exactly as in k_epoch_cta.
__device__ __forceinline__ void red_add_v4(float *p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

template <int T, bool SNAP>
__device__ __forceinline__ void head_flush(float *sv, float *s_acc, float *s_w, int H, int dry) {
  float4 *a4 = reinterpret_cast<float4 *>(s_acc);
  float4 *w4 = reinterpret_cast<float4 *>(s_w);
  for (int i = threadIdx.x; i < H / 4; i += T) {
    const float4 v = a4[i];
    if (SNAP) {
      // refresh the CTA's view of the head: L2 value (every flushed update) + own pending part,
      // read BEFORE this CTA's RED of the pending part is issued (same thread, same address: ordered)
      const float4 l = __ldcg(reinterpret_cast<const float4 *>(sv) + i);
      w4[i] = make_float4(l.x + v.x, l.y + v.y, l.z + v.z, l.w + v.w);
    }
    // dry probe: the pending array starts at -0.0f and the scatter adds +0.0f (non-negative values),
    // which turns a touched entry into +0.0f, so the probe flushes exactly the touched float4s
    const bool touched = dry ? (__float_as_uint(v.x) != 0x80000000u || __float_as_uint(v.y) != 0x80000000u ||
                                __float_as_uint(v.z) != 0x80000000u || __float_as_uint(v.w) != 0x80000000u)
                             : (v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f);
    if (touched) {
      red_add_v4(sv + 4 * i, v);  // dry: adds +-0.0f, state unchanged
      const float z = dry ? -0.f : 0.f;
      a4[i] = make_float4(z, z, z, z);
    }
  }
}

// Tail read (TS): TS = 0 gathers tail entries from sv itself; TS = 1 / 2 from the
// read copy svr (refreshed before every slice launch, so never written during this kernel) with L2 /
// L1-cached loads.  The lines gathered and the lines reduced are then disjoint, which the L2 serves
// ~35% faster (profiles/mix_bench_r1.txt: 84 -> 114 G gather+RED pairs/s).
template <int TS>
__device__ __forceinline__ float ld_tail(const EpochArgs &a, int32_t j) {
  if (TS == 2) return __ldg(a.svr + j);
  if (TS == 1) return __ldcg(a.svr + j);
  return ld_sv(a.sv + j);
}

// PF: thread 0 prefetches the next coordinate (ticket, permutation, offsets, model, norm, label)
// while the CTA works on the current one and publishes it through shared memory, so the
// ticket -> Feistel -> ptr -> x chain (three dependent round trips) leaves the per-row critical
// path.  The prefetched coordinate reads nothing of the shared vector before its turn, so this adds
// no staleness; x[c'] is current because this CTA is its only writer in the epoch (c10).
template <int FORM, int T, int E, bool SNAP, int TS = 0, bool PF = false, bool HC = false>
__global__ void __launch_bounds__(T, 1024 / T) k_epoch_cta_head(EpochArgs a, BinArgs b, int H, int flush) {
  constexpr int NW = T / 32;
  extern __shared__ float4 s_dyn[];
  float *s_acc = reinterpret_cast<float *>(s_dyn);
  float *s_w = s_acc + H;  // SNAP: the CTA's view of the head (refreshed at every flush)
  __shared__ float s_red[NW];
  __shared__ float s_delta;
  __shared__ unsigned int s_ticket;
  __shared__ int64_t s_cur[4];  // PF: coordinate (-1 = slice done), ptr[c], ptr[c + 1], its position t
  __shared__ float s_cx[3];     // PF: x[c], norm[c], y[c]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < H; i += T) s_acc[i] = b.dry ? -0.f : 0.f;
  if (SNAP) {
    __syncthreads();
    head_flush<T, true>(a.sv, s_acc, s_w, H, 0);  // initial view (nothing pending yet)
  }
  int64_t n_c = -1, n_beg = 0, n_end = 0, n_t = 0;  // PF (thread 0): the next coordinate
  float n_x = 0.f, n_nrm = 0.f, n_y = 0.f;
  unsigned n_tk = 0;
  auto fetch = [&](unsigned tk) {
    const int64_t t = b.lo + (int64_t)tk;
    n_t = t;
    n_c = -1;
    if (t >= b.hi) return;
    n_c = bin_coord(b, t);
    n_beg = __ldg(a.ptr + n_c);
    n_end = __ldg(a.ptr + n_c + 1);
    n_x = a.x[n_c];
    n_nrm = __ldg(a.norm + n_c);
    n_y = FORM == SCD_DUAL ? __ldg(a.y + n_c) : 0.f;
  };
  if (PF && tid == 0) fetch(atomicAdd(b.counter, 1u));
  int since = 0;
  for (;;) {
    int64_t c, beg, end;
    if (PF) {
      if (tid == 0) {
        s_cur[0] = n_c;
        s_cur[1] = n_beg;
        s_cur[2] = n_end;
        s_cur[3] = n_t;
        s_cx[0] = n_x;
        s_cx[1] = n_nrm;
        s_cx[2] = n_y;
        if (n_c >= 0) n_tk = atomicAdd(b.counter, 1u);  // consumed after this row's gathers
      }
      __syncthreads();  // also orders the previous coordinate's s_acc updates before this one's reads
      c = s_cur[0];
      if (c < 0) break;
      beg = s_cur[1];
      end = s_cur[2];
      if (HC && !b.dry && s_cur[3] % a.head_P == 0) {
        // head copy (experiment): row position t refreshes chunk (t / head_P) mod (H / 1024) of svr[0, H)
        const int64_t nchh = ((int64_t)H + T * 4 - 1) / (T * 4);
        const int64_t ih = ((s_cur[3] / a.head_P) % nchh) * (T * 4) + (int64_t)tid * 4;
        if (ih + 3 < H)
          *reinterpret_cast<float4 *>(const_cast<float *>(a.svr) + ih) =
              __ldcg(reinterpret_cast<const float4 *>(a.sv + ih));
      }
      if (TS && a.roll_R > 0 && !b.dry && s_cur[3] % a.roll_R == 0) {
        // rolling tail copy: row position t refreshes chunk (t / roll_R) mod nchunks of
        // svr from sv, so every tail entry of the copy is at most roll_R · nchunks positions old
        // without any slice boundary (plain stores: a concurrent reader sees the old or the new value)
        constexpr int64_t CH = (int64_t)T * 4;
        const int64_t nch = (a.roll_hi - a.roll_lo + CH - 1) / CH;
        const int64_t i = a.roll_lo + ((s_cur[3] / a.roll_R) % nch) * CH + (int64_t)tid * 4;
        float *dst = const_cast<float *>(a.svr);
        if (i + 3 < a.roll_hi)
          *reinterpret_cast<float4 *>(dst + i) = __ldcg(reinterpret_cast<const float4 *>(a.sv + i));
        else
          for (int64_t q = i; q < a.roll_hi && q < i + 4; ++q) dst[q] = __ldcg(a.sv + q);
      }
    } else {
      if (tid == 0) s_ticket = atomicAdd(b.counter, 1u);
      __syncthreads();  // also orders the previous coordinate's s_acc updates before this one's reads
      const int64_t t = b.lo + (int64_t)s_ticket;
      if (t >= b.hi) break;
      c = bin_coord(b, t);
      beg = __ldg(a.ptr + c);
      end = __ldg(a.ptr + c + 1);
    }
    int32_t id[E];
    float v[E];
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t k = beg + (int64_t)e * T + tid;
      if (k < end) {
        id[e] = __ldcs(a.idx + k);
        v[e] = val_cs(a.val, k);
      } else {
        id[e] = -1;
        v[e] = 0.f;
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (id[e] >= 0) {
        float w;
        if (SNAP)
          w = id[e] < H ? s_w[id[e]] + s_acc[id[e]] : ld_tail<TS>(a, id[e]);
        else if (TS)
          w = id[e] < H ? ld_sv((HC ? a.svr : a.sv) + id[e]) + s_acc[id[e]] : ld_tail<TS>(a, id[e]);
        else
          w = ld_sv(a.sv + id[e]) + (id[e] < H ? s_acc[id[e]] : 0.f);
        acc = fmaf(w, v[e], acc);
      }
    for (int64_t base = beg + (int64_t)T * E; base < end; base += (int64_t)T * E) {
#pragma unroll 4
      for (int e = 0; e < E; ++e) {
        const int64_t k = base + (int64_t)e * T + tid;
        if (k < end) {
          const int32_t j = __ldcg(a.idx + k);
          float w;
          if (SNAP)
            w = j < H ? s_w[j] + s_acc[j] : ld_tail<TS>(a, j);
          else if (TS)
            w = j < H ? ld_sv((HC ? a.svr : a.sv) + j) + s_acc[j] : ld_tail<TS>(a, j);
          else
            w = ld_sv(a.sv + j) + (j < H ? s_acc[j] : 0.f);
          acc = fmaf(w, val_cg(a.val, k), acc);
        }
      }
    }
    if (PF && tid == 0 && c >= 0) fetch(n_tk);  // next coordinate's chain overlaps reduce + scatter
    acc = warp_sum(acc);
    if (lane == 0) s_red[wid] = acc;
    __syncthreads();
    if (wid == 0) {
      float s = lane < NW ? s_red[lane] : 0.f;
      s = warp_sum(s);
      if (lane == 0) {
        const float xc = PF ? s_cx[0] : a.x[c];
        const float nc = PF ? s_cx[1] : __ldg(a.norm + c);
        const float yc = PF ? s_cx[2] : (FORM == SCD_DUAL ? __ldg(a.y + c) : 0.f);
        const float d = coord_delta<FORM>(s, xc, nc, yc, a.lam, a.lamN);
        if (!b.dry) a.x[c] = xc + d;  // single writer per epoch (c10)
        s_delta = b.dry ? 0.f : d;
      }
    }
    __syncthreads();
    const float d = scatter_scale<FORM>(s_delta);
    if (d != 0.f || b.dry) {
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (id[e] >= 0) {
          if (id[e] < H)
            s_acc[id[e]] += v[e] * d;  // ids unique within a coordinate: no race
          else
            red_add(a.sv + id[e], v[e] * d);
        }
      for (int64_t k0 = beg + (int64_t)T * E + tid; k0 < end; k0 += (int64_t)T * 4) {
        int32_t jj[4];
        float vv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t kk = k0 + (int64_t)u * T;
          jj[u] = kk < end ? __ldcg(a.idx + kk) : -1;
          vv[u] = kk < end ? val_cg(a.val, kk) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (jj[u] >= 0) {
            if (jj[u] < H)
              s_acc[jj[u]] += vv[u] * d;
            else
              red_add(a.sv + jj[u], vv[u] * d);
          }
      }
    }
    if (++since == flush) {
      since = 0;
      __syncthreads();
      head_flush<T, SNAP>(a.sv, s_acc, s_w, H, b.dry);
    }
  }
  head_flush<T, false>(a.sv, s_acc, s_w, H, b.dry);  // after the exit barrier: every pending update is final
}

// ----------------------------------------------------------------------------------------------
// Die-split CTA kernel (die.cu).  Every coordinate is processed by two CTAs, one on
// each die, each over the part of the coordinate's entries whose shared-vector element is homed in
// its own die's L2 (entries reordered at create: [ptr[c], mid[c]) die 0, [mid[c], ptr[c+1]) die 1).
// CTAs of die d take tickets from die d's counter, so both dies walk the same permutation.  The two
// partial dot products meet in a global slot (release/acquire, tagged with the launch); both CTAs
// form dp = p0 + p1 in that order, hence the same Δ; the die-0 CTA is the single writer of x[c]
// (c10) and each CTA scatters its own part.  The die-1 CTA reads x[c] before publishing its
// partial, i.e. before die 0 can write it.  A CTA publishes before it waits, so the lowest
// outstanding ticket always completes: no deadlock while every CTA is resident (grid <= occupancy).
struct SplitArgs {
  const int64_t *mid;
  const int32_t *idx;
  const float *val;  // nullptr = implicit values
  const uint8_t *sm_die;
  float *slot_p;
  unsigned *slot_tag;
  unsigned *err;
  unsigned *counter1;  // die 1's ticket counter (die 0 uses BinArgs::counter)
  unsigned tag;
  int nosync;          // diagnostic only: no partner exchange (wrong Δ), isolates the rendezvous cost
};

__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned smid_now() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

template <int FORM, int T, int E>
__global__ void __launch_bounds__(T, 4) k_epoch_split(EpochArgs a, BinArgs b, SplitArgs s) {
  constexpr int NW = T / 32;
  __shared__ float s_red[NW];
  __shared__ float s_delta;
  __shared__ unsigned int s_ticket;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int die = s.sm_die[smid_now()];  // a CTA never migrates
  unsigned *counter = die == 0 ? b.counter : s.counter1;
  for (;;) {
    if (tid == 0) s_ticket = atomicAdd(counter, 1u);
    __syncthreads();
    const int64_t t = b.lo + (int64_t)s_ticket;
    if (t >= b.hi) break;
    const int64_t c = bin_coord(b, t);
    const int64_t m = __ldg(s.mid + c);
    const int64_t beg = die == 0 ? __ldg(a.ptr + c) : m;
    const int64_t end = die == 0 ? m : __ldg(a.ptr + c + 1);
    float xc = 0.f;
    if (tid == 0) xc = a.x[c];  // before publishing (see above)
    int32_t id[E];
    float v[E];
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t k = beg + (int64_t)e * T + tid;
      if (k < end) {
        id[e] = __ldcs(s.idx + k);
        v[e] = val_cs(s.val, k);
      } else {
        id[e] = -1;
        v[e] = 0.f;
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (id[e] >= 0) acc = fmaf(ld_sv(a.sv + id[e]), v[e], acc);
    acc += dot_strided<8>(a.sv, s.idx, s.val, beg + (int64_t)T * E + tid, end, T);
    acc = warp_sum(acc);
    if (lane == 0) s_red[wid] = acc;
    __syncthreads();
    if (wid == 0) {
      float p = lane < NW ? s_red[lane] : 0.f;
      p = warp_sum(p);
      if (lane == 0) {
        const int64_t q = 2 * t;
        if (s.nosync) {
          s.slot_p[q + 1 - die] = 0.f;
          s.slot_tag[q + 1 - die] = s.tag;
        }
        s.slot_p[q + die] = p;
        st_release(s.slot_tag + q + die, s.tag);
        unsigned spins = 0;
        while (ld_acquire(s.slot_tag + q + (1 - die)) != s.tag) {
          if (++spins > (1u << 26)) {  // partner never arrived: flag it, do not hang
            atomicExch(s.err, 1u);
            break;
          }
        }
        const float po = __ldcg(s.slot_p + q + (1 - die));
        const float dp = die == 0 ? p + po : po + p;
        const float d = coord_delta<FORM>(dp, xc, __ldg(a.norm + c), FORM == SCD_DUAL ? __ldg(a.y + c) : 0.f,
                                          a.lam, a.lamN);
        if (die == 0 && !b.dry) a.x[c] = xc + d;  // single writer per epoch (c10)
        s_delta = b.dry ? 0.f : d;
      }
    }
    __syncthreads();
    const float d = scatter_scale<FORM>(s_delta);
    if (d != 0.f || b.dry) {
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (id[e] >= 0) red_add(a.sv + id[e], v[e] * d);
      scatter_strided<8>(a.sv, s.idx, s.val, beg + (int64_t)T * E + tid, end, T, d);
    }
  }
}

// ----------------------------------------------------------------------------------------------
template <int FORM, int G, int E, bool WILD = false>
__global__ void __launch_bounds__(256) k_epoch_group(EpochArgs a, BinArgs b) {
  constexpr int CPW = 32 / G;  // coordinates per warp per ticket
  const int lane = threadIdx.x & 31;
  const int sub = lane / G, gl = lane % G;
  for (;;) {
    unsigned int t0 = 0;
    if (lane == 0) t0 = atomicAdd(b.counter, (unsigned)CPW);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    if (b.lo + (int64_t)t0 >= b.hi) break;  // warp-uniform
    // lanes 0..CPW-1 evaluate the permutation for the warp's CPW tickets, then broadcast
    int64_t cl = -1;
    if (lane < CPW && b.lo + (int64_t)t0 + lane < b.hi) cl = bin_coord(b, b.lo + t0 + lane);
    const int64_t c = __shfl_sync(0xffffffffu, cl, sub);
    const bool active = c >= 0;
    int64_t beg = 0, end = 0;
    if (active) {
      beg = __ldg(a.ptr + c);
      end = __ldg(a.ptr + c + 1);
    }
    int32_t id[E];
    float v[E];
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t k = beg + (int64_t)e * G + gl;
      if (k < end) {
        id[e] = __ldcs(a.idx + k);
        v[e] = val_cs(a.val, k);
      } else {
        id[e] = -1;
        v[e] = 0.f;
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (id[e] >= 0) acc = fmaf(ld_sv(a.svg + id[e]), v[e], acc);
    acc += dot_strided<8>(a.svg, a.idx, a.val, beg + (int64_t)G * E + gl, end, G);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    float d = 0.f;
    if (active && gl == 0) {  // group leader: single writer of x[c] (c10)
      const float xc = a.x[c];
      d = coord_delta<FORM>(acc, xc, __ldg(a.norm + c), FORM == SCD_DUAL ? __ldg(a.y + c) : 0.f, a.lam, a.lamN);
      if (!b.dry) a.x[c] = xc + d;
      if (b.dry) d = 0.f;
    }
    d = scatter_scale<FORM>(__shfl_sync(0xffffffffu, d, sub * G));
    if (d != 0.f || b.dry) {
      scatter_regs<WILD, E>(a.sv, id, v, d);
      scatter_strided<8, WILD>(a.sv, a.idx, a.val, beg + (int64_t)G * E + gl, end, G, d);
    }
  }
}

// ----------------------------------------------------------------------------------------------
// Software-pipelined sub-warp kernel for short coordinates (criteo-shaped rows, 39 entries).
// With a short coordinate the epoch is bound by its dependent round trips (ticket -> coordinate
// -> offsets -> entries -> gathers -> delta -> scatter), and the staleness cap limits how many
// coordinates may be in flight.  So each warp overlaps the next batch's loads with the current
// batch's compute: while batch i gathers / reduces / scatters, batch i+1's offsets, scalars and
// entries are already in flight, and batch i+2's coordinates are computed.  Only batch i reads
// the shared vector, so prefetching does not add staleness.  Tickets are taken TB batches at a
// time (one atomic per TB·32/G coordinates).
template <int FORM, int G, int E, int TB>
__global__ void __launch_bounds__(256) k_epoch_group_pipe(EpochArgs a, BinArgs b) {
  constexpr int CPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int sub = lane / G, gl = lane % G;
  const unsigned FULL = 0xffffffffu;
  unsigned int grab = 0, left = 0;
  // warp-uniform: position of the next batch (or -1 when the slice is exhausted)
  auto next_pos = [&]() -> int64_t {
    if (left == 0) {
      unsigned int g = 0;
      if (lane == 0) g = atomicAdd(b.counter, (unsigned)(CPW * TB));
      grab = __shfl_sync(FULL, g, 0);
      left = TB;
    }
    const int64_t t = b.lo + (int64_t)grab + (int64_t)(TB - left) * CPW;
    --left;
    return t < b.hi ? t : -1;
  };
  // coordinate of this lane's group for the batch at position t (lanes < CPW evaluate the permutation)
  auto coord_of = [&](int64_t t) -> int64_t {
    int64_t cl = -1;
    if (t >= 0 && lane < CPW && t + lane < b.hi) cl = bin_coord(b, (uint64_t)(t + lane));
    return __shfl_sync(FULL, cl, sub);
  };
  // batch i (current) and i+1 (next) state
  int64_t c_cur = coord_of(next_pos());
  if (__all_sync(FULL, c_cur < 0)) return;
  int64_t beg = 0, end = 0;
  float xc = 0.f, nrm = 0.f, yc = 0.f;
  if (c_cur >= 0) {
    beg = __ldg(a.ptr + c_cur);
    end = __ldg(a.ptr + c_cur + 1);
    if (gl == 0) {
      xc = a.x[c_cur];
      nrm = __ldg(a.norm + c_cur);
      if (FORM == SCD_DUAL) yc = __ldg(a.y + c_cur);
    }
  }
  int32_t id[E];
  float v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int64_t k = beg + (int64_t)e * G + gl;
    id[e] = k < end ? __ldcs(a.idx + k) : -1;
    v[e] = k < end ? val_cs(a.val, k) : 0.f;
  }
  int64_t c_nxt = coord_of(next_pos());
  while (!__all_sync(FULL, c_cur < 0)) {
    // (a) offsets and scalars of batch i+1
    int64_t nbeg = 0, nend = 0;
    float nxc = 0.f, nnrm = 0.f, nyc = 0.f;
    if (c_nxt >= 0) {
      nbeg = __ldg(a.ptr + c_nxt);
      nend = __ldg(a.ptr + c_nxt + 1);
      if (gl == 0) {
        nxc = a.x[c_nxt];
        nnrm = __ldg(a.norm + c_nxt);
        if (FORM == SCD_DUAL) nyc = __ldg(a.y + c_nxt);
      }
    }
    // (b) gather-dot of batch i
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (id[e] >= 0) acc = fmaf(ld_sv(a.svg + id[e]), v[e], acc);
    acc += dot_strided<8>(a.svg, a.idx, a.val, beg + (int64_t)G * E + gl, end, G);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
    // (c) delta of batch i (group leader is the single writer of x[c], c10)
    float d = 0.f;
    if (c_cur >= 0 && gl == 0) {
      d = coord_delta<FORM>(acc, xc, nrm, yc, a.lam, a.lamN);
      if (!b.dry) a.x[c_cur] = xc + d;
      if (b.dry) d = 0.f;
    }
    d = scatter_scale<FORM>(__shfl_sync(FULL, d, sub * G));
    // (d) entries of batch i+1
    int32_t nid[E];
    float nv[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t k = nbeg + (int64_t)e * G + gl;
      nid[e] = k < nend ? __ldcs(a.idx + k) : -1;
      nv[e] = k < nend ? val_cs(a.val, k) : 0.f;
    }
    // (e) scatter of batch i
    if (d != 0.f || b.dry) {
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (id[e] >= 0) red_add(a.sv + id[e], v[e] * d);
      scatter_strided<8>(a.sv, a.idx, a.val, beg + (int64_t)G * E + gl, end, G, d);
    }
    // (f) coordinates of batch i+2, rotate
    const bool more = __any_sync(FULL, c_nxt >= 0);
    const int64_t c_nn = more ? coord_of(next_pos()) : -1;
    c_cur = c_nxt;
    beg = nbeg;
    end = nend;
    xc = nxc;
    nrm = nnrm;
    yc = nyc;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      id[e] = nid[e];
      v[e] = nv[e];
    }
    c_nxt = c_nn;
  }
}

// ----------------------------------------------------------------------------------------------
// CTA-combining sub-warp kernel for short coordinates with heavily shared entries (one-hot
// criteo-shaped rows: every row carries one of the few values of each small field, so a handful
// of shared-vector entries receive an atomic from a large fraction of all rows and serialise in
// their L2 slice).  A CTA processes T/G coordinates per iteration: their entries are inserted into
// a shared-memory hash table (one slot per distinct index), each distinct entry is gathered ONCE,
// the coordinates compute their deltas from those values, the scatter is summed per slot with
// shared-memory atomics, and each distinct entry receives ONE red.global.add.  The T/G
// coordinates of an iteration are in flight together in every kernel variant (they read before
// any of them writes), so combining changes rounding order only, not the algorithm.
template <int FORM, int G, int T, int S>
__global__ void __launch_bounds__(T) k_epoch_group_comb(EpochArgs a, BinArgs b) {
  constexpr int E = 64 / G;  // entries per lane: the bin holds coordinates of <= 64 entries
  constexpr int CPC = T / G;
  const unsigned FULL = 0xffffffffu;
  __shared__ int32_t s_key[S];
  __shared__ float s_g[S];
  __shared__ float s_r[S];
  __shared__ int32_t s_list[S];
  __shared__ int s_n;
  __shared__ unsigned int s_ticket;
  // coordinate queue: every QI iterations the whole CTA takes CPC*QI tickets at once, each thread
  // evaluates one permutation entry and prefetches that coordinate's offsets and scalars (the
  // single writer of x[c] is this CTA, so the prefetched x[c] is current)
  constexpr int QI = T / CPC;  // refill = one coordinate per thread
  __shared__ long long s_qc[T], s_qb[T], s_qe[T];
  __shared__ float s_qx[T], s_qn[T], s_qy[T];
  const int tid = threadIdx.x, lane = tid & 31;
  const int grp = tid / G, gl = tid % G, sub = lane / G;
  for (int i = tid; i < S; i += T) s_key[i] = -1;
  if (tid == 0) s_n = 0;
  int qpos = QI;  // iterations consumed from the queue
  bool more = true;
  for (;;) {
    if (qpos == QI) {
      if (!more) break;
      if (tid == 0) s_ticket = atomicAdd(b.counter, (unsigned)T);
      __syncthreads();
      const int64_t t = b.lo + (int64_t)s_ticket + tid;
      long long cq = -1, qb = 0, qe = 0;
      float qx = 0.f, qn = 0.f, qy = 0.f;
      if (t < b.hi) {
        cq = bin_coord(b, (uint64_t)t);
        qb = __ldg(a.ptr + cq);
        qe = __ldg(a.ptr + cq + 1);
        qx = a.x[cq];
        qn = __ldg(a.norm + cq);
        if (FORM == SCD_DUAL) qy = __ldg(a.y + cq);
      }
      s_qc[tid] = cq;
      s_qb[tid] = qb;
      s_qe[tid] = qe;
      s_qx[tid] = qx;
      s_qn[tid] = qn;
      s_qy[tid] = qy;
      more = __syncthreads_or(b.lo + (int64_t)s_ticket + T < b.hi);
      qpos = 0;
      if (s_qc[0] < 0) break;  // queue empty (uniform)
    }
    const int qi = qpos * CPC + grp;
    ++qpos;
    const int64_t c = s_qc[qi];
    if (__syncthreads_and(c < 0)) {
      qpos = QI;
      if (!more) break;
      continue;
    }
    int64_t beg = 0, end = 0;
    float xc = 0.f, nrm = 0.f, yc = 0.f;
    if (c >= 0) {
      beg = s_qb[qi];
      end = s_qe[qi];
      xc = s_qx[qi];
      nrm = s_qn[qi];
      yc = s_qy[qi];
    }
    int32_t slot[E];
    float v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t k = beg + (int64_t)e * G + gl;
      const int32_t id = k < end ? __ldcs(a.idx + k) : -1;
      v[e] = k < end ? val_cs(a.val, k) : 0.f;
      slot[e] = -1;
      if (id >= 0) {  // insert (linear probing)
        uint32_t h = ((uint32_t)id * 2654435761u) & (S - 1);
        for (;;) {
          const int32_t old = atomicCAS(&s_key[h], -1, id);
          if (old == -1) {
            s_list[atomicAdd(&s_n, 1)] = (int32_t)h;
            break;
          }
          if (old == id) break;
          h = (h + 1) & (S - 1);
        }
        slot[e] = (int32_t)h;
      }
    }
    __syncthreads();
    const int n = s_n;
    for (int i = tid; i < n; i += T) {  // one gather per distinct entry
      const int h = s_list[i];
      s_g[h] = ld_sv(a.svg + s_key[h]);
      s_r[h] = 0.f;
    }
    __syncthreads();
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (slot[e] >= 0) acc = fmaf(s_g[slot[e]], v[e], acc);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
    float d = 0.f;
    if (c >= 0 && gl == 0) {
      d = coord_delta<FORM>(acc, xc, nrm, yc, a.lam, a.lamN);
      if (!b.dry) a.x[c] = xc + d;  // single writer (c10)
      if (b.dry) d = 0.f;
    }
    d = scatter_scale<FORM>(__shfl_sync(FULL, d, sub * G));
    if (d != 0.f) {
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (slot[e] >= 0) atomicAdd(&s_r[slot[e]], v[e] * d);
    }
    __syncthreads();
    for (int i = tid; i < n; i += T) {  // one atomic per distinct entry
      const int h = s_list[i];
      const float r = s_r[h];
      if (r != 0.f || b.dry) red_add(a.sv + s_key[h], r);
      s_key[h] = -1;
    }
    if (tid == 0) s_n = 0;
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------------------------
// Hot-set sub-warp kernel for short coordinates (criteo-shaped one-hot rows).  A few thousand
// shared-vector entries carry most of the stored entries (C5: the 4096 most frequent features hold
// 79% of them) and every row updates some of them, so their L2 lines serialise.  At create
// (hot.cu) the K most frequent entries get a slot and a private copy of the bin's indices is
// re-encoded: id >= 0 = tail entry (shared-vector index), id < 0 = hot entry (slot = id & 0x7fffffff).
// Each CTA keeps its pending updates of the hot entries in shared memory (s_pend, CAS-loop atomics:
// the CTA's rows update them concurrently) and, with VIEW, a copy of their values refreshed at every
// flush; the warps run their rows without any CTA barrier and meet every F row batches to flush
// (one RED per touched hot entry) — so a hot line takes one RED per CTA per F batches instead of
// one per row.  Pending (and, with VIEW, view age) are extra staleness, bounded by the schedule:
// grid * rows per CTA * (1 + F * (VIEW ? 2 : 1)) <= cap.
struct HotArgs {
  const int32_t *idx;      // re-encoded entries of the bin's coordinates (same offsets as EpochArgs::ptr)
  const int32_t *hot_ids;  // [K]: shared-vector index of each hot slot
  int K;                   // hot slots (multiple of 4)
  int F;                   // row batches per warp between flushes
  float *hc;               // HC: [K] rolling copy of the hot values (slot order), gathered instead of sv
  int P;                   // HC: every P-th warp ticket refreshes 32 slots of hc
};

// hc[s] = sv[hot_ids[s]] for every slot (before each hot-bin launch when the copy is used)
__global__ void k_hot_refresh(const float *sv, const int32_t *hot_ids, int K, float *hc) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x) hc[i] = __ldcg(sv + hot_ids[i]);
}

// HC: the hot values are gathered from h.hc, a copy in slot order refreshed 32 slots at a time by the
// warp whose ticket t has (t / rows per warp) mod P = 0, so the gathers leave the lines that take the
// flush REDs; the copy's age (P · K/32 tickets) is counted in the window budget (hot_launch_shape).
template <int FORM, int G, int E, bool VIEW, bool HC = false, bool TP = false, bool HP = false>
__global__ void __launch_bounds__(512) k_epoch_group_hot(EpochArgs a, BinArgs b, HotArgs h) {
  constexpr int CPW = 32 / G;
  const unsigned FULL = 0xffffffffu;
  extern __shared__ float4 s_dyn[];
  float *s_pend = reinterpret_cast<float *>(s_dyn);  // [K] pending updates of the hot entries
  float *s_aux = s_pend + h.K;                       // [K] VIEW: values; else: int32 shared-vector index
  int32_t *s_hid = reinterpret_cast<int32_t *>(s_aux);
  const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
  for (int i = threadIdx.x; i < h.K; i += blockDim.x) {
    s_pend[i] = b.dry ? -0.f : 0.f;
    const int32_t j = __ldg(h.hot_ids + i);
    if (VIEW)
      s_aux[i] = ld_sv(a.sv + j);
    else
      s_hid[i] = j;
  }
  __syncthreads();
  // Software pipeline (as in k_epoch_group_pipe): while batch i gathers, reduces and scatters, the
  // coordinates, offsets, scalars and entries of batch i+1 are already loaded.  Only batch i reads
  // the shared vector, so the prefetch adds no staleness.
  auto take = [&]() -> int64_t {  // warp-uniform: this lane's coordinate of the next batch, -1 = none
    unsigned int t0 = 0;
    if (lane == 0) t0 = atomicAdd(b.counter, (unsigned)CPW);
    t0 = __shfl_sync(FULL, t0, 0);
    if (b.lo + (int64_t)t0 >= b.hi) return -2;  // slice exhausted (uniform)
    if (HC && !b.dry) {
      const int64_t tk = (b.lo + (int64_t)t0) / CPW;
      if (tk % h.P == 0) {
        const int nch = (h.K + 31) / 32;
        const int sl = (int)((tk / h.P) % nch) * 32 + lane;
        if (sl < h.K) h.hc[sl] = __ldcg(a.sv + s_hid[sl]);
      }
    }
    int64_t cl = -1;
    if (lane < CPW && b.lo + (int64_t)t0 + lane < b.hi) cl = bin_coord(b, b.lo + t0 + lane);
    return __shfl_sync(FULL, cl, sub);
  };
  struct Batch {
    int64_t c;
    int32_t id[E];
    float v[E];
    float tw[E];  // TP: tail values gathered one step ahead
    unsigned valid;
    float xc, nrm, yc;
  };
  auto tail_prefetch = [&](Batch &q) {
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (q.valid >> e & 1) {
        if (q.id[e] >= 0)
          q.tw[e] = ld_sv(a.sv + q.id[e]);
        else if (HP)
          q.tw[e] = __ldcg(h.hc + (q.id[e] & 0x7fffffff));  // HP: hot copy value one step early too
      }
  };
  auto load = [&](Batch &q, int64_t c) {
    q.c = c;
    q.valid = 0;
    q.xc = q.nrm = q.yc = 0.f;
    int64_t beg = 0, end = 0;
    if (c >= 0) {
      beg = __ldg(a.ptr + c);
      end = __ldg(a.ptr + c + 1);
      if (gl == 0) {
        q.xc = a.x[c];  // this warp is the single writer of x[c]: the prefetched value is current
        q.nrm = __ldg(a.norm + c);
        if (FORM == SCD_DUAL) q.yc = __ldg(a.y + c);
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t k = beg + (int64_t)e * G + gl;
      q.id[e] = 0;
      q.v[e] = 0.f;
      if (k < end) {
        q.id[e] = __ldcs(h.idx + k);
        q.v[e] = val_cs(a.val, k);
        q.valid |= 1u << e;
      }
    }
  };
  Batch cur, nxt;
  int64_t cn = take();
  bool more = cn != -2;  // warp-uniform: the warp holds a batch
  if (more) load(cur, cn);
  if (TP && more) tail_prefetch(cur);
  for (;;) {
    for (int it = 0; it < h.F && more; ++it) {
      // next batch: ticket + coordinates + entries (no shared-vector access)
      cn = take();
      const bool have_next = cn != -2;
      if (have_next) load(nxt, cn);
      // current batch: gather-dot
      float w[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        w[e] = 0.f;
        if (cur.valid >> e & 1) {
          if (cur.id[e] >= 0) {
            w[e] = TP ? cur.tw[e] : ld_sv(a.sv + cur.id[e]);
          } else {
            const int sl = cur.id[e] & 0x7fffffff;
            w[e] = (VIEW ? s_aux[sl] : (HP ? cur.tw[e] : (HC ? __ldcg(h.hc + sl) : ld_sv(a.sv + s_hid[sl])))) + s_pend[sl];
          }
        }
      }
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) acc = fmaf(w[e], cur.v[e], acc);
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
      float d = 0.f;
      if (cur.c >= 0 && gl == 0) {  // group leader: single writer of x[c] (c10)
        d = coord_delta<FORM>(acc, cur.xc, cur.nrm, cur.yc, a.lam, a.lamN);
        if (!b.dry) a.x[cur.c] = cur.xc + d;
        if (b.dry) d = 0.f;
      }
      d = scatter_scale<FORM>(__shfl_sync(FULL, d, sub * G));
      if (d != 0.f || b.dry) {  // dry probe: same traffic, adds +0.0f
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (cur.valid >> e & 1) {
            if (cur.id[e] >= 0)
              red_add(a.sv + cur.id[e], cur.v[e] * d);
            else
              atomicAdd(s_pend + (cur.id[e] & 0x7fffffff), cur.v[e] * d);
          }
      }
      more = have_next;
      if (have_next) {
        cur = nxt;
        if (TP) tail_prefetch(cur);  // the next batch's tail values, one step early
      }
    }
    const bool any = __syncthreads_or(more);
    for (int i = threadIdx.x; i < h.K; i += blockDim.x) {  // flush (and refresh the view)
      const float p = s_pend[i];
      const int32_t j = VIEW ? __ldg(h.hot_ids + i) : s_hid[i];
      if (VIEW) s_aux[i] = ld_sv(a.sv + j) + p;  // read before this CTA's RED: own pending counted once
      // dry probe: pending starts at -0.0f and a touched slot becomes +0.0f (non-negative values)
      if (b.dry ? __float_as_uint(p) != 0x80000000u : p != 0.f) {
        red_add(a.sv + j, p);
        s_pend[i] = b.dry ? -0.f : 0.f;
      }
    }
    __syncthreads();
    if (!any) break;
  }
}

// ----------------------------------------------------------------------------------------------
// Deterministic (debug) epoch: exactly Alg. 1's order with Alg. 2's arithmetic, one coordinate
// at a time, fixed reduction tree (strided per-thread partials -> xor-shuffle tree -> 8 warp
// partials summed in order).  Plain read-modify-write scatter: one coordinate in flight and
// unique indices within a coordinate, so there is no race.
constexpr int kDbgT = 256;
template <int FORM>
__global__ void __launch_bounds__(kDbgT) k_epoch_debug(EpochArgs a, Perm perm, int64_t j0, int64_t j1) {
  __shared__ float s_red[kDbgT / 32];
  __shared__ float s_delta;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int64_t j = j0; j < j1; ++j) {
    const int64_t c = (int64_t)perm_apply(perm, (uint64_t)j);
    const int64_t beg = a.ptr[c], end = a.ptr[c + 1];
    float acc = 0.f;
    for (int64_t k = beg + tid; k < end; k += kDbgT) acc = fmaf(a.sv[a.idx[k]], val_at(a.val, k), acc);
    acc = warp_sum(acc);
    if (lane == 0) s_red[wid] = acc;
    __syncthreads();
    if (tid == 0) {
      float s = 0.f;
      for (int w = 0; w < kDbgT / 32; ++w) s += s_red[w];
      const float xc = a.x[c];
      const float d = coord_delta<FORM>(s, xc, a.norm[c], FORM == SCD_DUAL ? a.y[c] : 0.f, a.lam, a.lamN);
      a.x[c] = xc + d;
      s_delta = d;
    }
    __syncthreads();
    const float d = scatter_scale<FORM>(s_delta);
    for (int64_t k = beg + tid; k < end; k += kDbgT) a.sv[a.idx[k]] += val_at(a.val, k) * d;
    __syncthreads();
  }
}

// Tail read copy refresh: svr[lo, hi) = sv[lo, hi) (lo multiple of 4, both 16-byte aligned at lo).
__global__ void __launch_bounds__(256) k_tail_refresh(const float *__restrict__ sv, float *__restrict__ svr, int64_t lo,
                                                      int64_t hi) {
  const int64_t n4 = (hi - lo) / 4;
  const float4 *src = reinterpret_cast<const float4 *>(sv + lo);
  float4 *dst = reinterpret_cast<float4 *>(svr + lo);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) dst[i] = __ldcg(src + i);
  for (int64_t i = lo + n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += stride) svr[i] = __ldcg(sv + i);
}

template <int FORM>
__global__ void k_empty_fix(EpochArgs a, const int32_t *list, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = list[i];
    const float xc = a.x[c];
    a.x[c] = xc + coord_delta<FORM>(0.f, xc, 0.f, FORM == SCD_DUAL ? a.y[c] : 0.f, a.lam, a.lamN);
  }
}

__global__ void k_perm_export(Perm p, int64_t n, int64_t *out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    out[j] = (int64_t)perm_apply(p, (uint64_t)j);
}

__global__ void k_partition_export(Perm p, int64_t count, int32_t k, int32_t *owner) {
  const int64_t base = count / k, rem = count % k;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = (int64_t)perm_apply(p, (uint64_t)i);
    const int64_t blk = (i < rem * (base + 1)) ? i / (base + 1) : rem + (i - rem * (base + 1)) / base;
    owner[c] = (int32_t)blk;
  }
}

// ----------------------------------------------------------------------------------------------
// Very long coordinates (> 16384 entries: the dense head of a power-law feature distribution in
// the primal) are strongly coupled to one another, so only a few may be in flight.
// To keep the GPU busy anyway, each one is split across a cluster of CL CTAs: every CTA takes a
// contiguous slice, partial dots meet in CTA 0's shared memory over DSMEM, CTA 0 computes Δ, and
// every CTA scatters its slice.  Two cluster barriers per coordinate.
template <int FORM, int CL, int T, int E, bool WILD = false>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(T) k_epoch_cluster(EpochArgs a, BinArgs b) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int NW = T / 32;
  __shared__ float s_red[NW];
  __shared__ float s_part[CL];
  __shared__ float s_delta;
  __shared__ unsigned int s_ticket;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned int r = cluster.block_rank();
  unsigned int *ticket0 = cluster.map_shared_rank(&s_ticket, 0);
  float *part0 = cluster.map_shared_rank(s_part, 0);
  float *delta0 = cluster.map_shared_rank(&s_delta, 0);
  for (;;) {
    if (r == 0 && tid == 0) s_ticket = atomicAdd(b.counter, 1u);
    cluster.sync();
    const int64_t t = b.lo + (int64_t)*ticket0;
    if (t >= b.hi) {
      cluster.sync();  // nobody leaves while another CTA may still read CTA 0's shared memory
      break;
    }
    const int64_t c = bin_coord(b, t);
    const int64_t beg0 = __ldg(a.ptr + c), end0 = __ldg(a.ptr + c + 1);
    const int64_t slice = (end0 - beg0 + CL - 1) / CL;
    const int64_t beg = beg0 + (int64_t)r * slice;
    const int64_t end = min(end0, beg + slice);
    int32_t id[E];
    float v[E];
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t k = beg + (int64_t)e * T + tid;
      if (k < end) {
        id[e] = __ldcs(a.idx + k);
        v[e] = val_cs(a.val, k);
      } else {
        id[e] = -1;
        v[e] = 0.f;
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (id[e] >= 0) acc = fmaf(ld_sv(a.svg + id[e]), v[e], acc);
    acc += dot_strided<8>(a.svg, a.idx, a.val, beg + (int64_t)T * E + tid, end, T);
    acc = warp_sum(acc);
    if (lane == 0) s_red[wid] = acc;
    __syncthreads();
    if (wid == 0) {
      float s = lane < NW ? s_red[lane] : 0.f;
      s = warp_sum(s);
      if (lane == 0) part0[r] = s;
    }
    cluster.sync();
    if (r == 0 && tid == 0) {
      float s = 0.f;
      for (int i = 0; i < CL; ++i) s += s_part[i];
      const float xc = a.x[c];
      const float d = coord_delta<FORM>(s, xc, __ldg(a.norm + c), FORM == SCD_DUAL ? __ldg(a.y + c) : 0.f, a.lam,
                                        a.lamN);
      a.x[c] = xc + d;
      s_delta = d;
    }
    cluster.sync();
    const float d = scatter_scale<FORM>(*delta0);
    if (d != 0.f) {
      scatter_regs<WILD, E>(a.sv, id, v, d);
      scatter_strided<8, WILD>(a.sv, a.idx, a.val, beg + (int64_t)T * E + tid, end, T, d);
    }
  }
}

// kernel table ---------------------------------------------------------------------------------
constexpr int kCtaT = kLanesCta, kCtaE = 16, kStreamU = 4;
constexpr int kGrpE8 = 8, kGrpE32 = 16;
constexpr int kClE = 8;

// 8-lane bins: 0 = plain, 1 = software-pipelined, 2 = CTA-combining (default); SCD_GROUP_KERNEL
constexpr int kCombT = 128, kCombS = 2048;
inline int group_kind() {
  static const int k = [] {
    const char *e = getenv("SCD_GROUP_KERNEL");
    if (!e) return 2;
    std::string s(e);
    return s == "plain" ? 0 : (s == "pipe" ? 1 : 2);
  }();
  return k;
}

template <int FORM>
void *kernel_for(int lanes, int plain) {
  switch (lanes) {
    case 8:
      if (!plain && group_kind() == 2) return (void *)k_epoch_group_comb<FORM, 8, kCombT, kCombS>;
      return (!plain && group_kind() == 1) ? (void *)k_epoch_group_pipe<FORM, 8, kGrpE8, 4> : (void *)k_epoch_group<FORM, 8, kGrpE8>;
    case 16:
      return group_kind() == 1 ? (void *)k_epoch_group_pipe<FORM, 16, 4, 4> : (void *)k_epoch_group<FORM, 16, 4>;
    case 32: return (void *)k_epoch_group<FORM, 32, kGrpE32>;
    case kLanesCluster: return nullptr;  // cluster_kernel(): depends on the bin's cluster size
    default: {
      // register-resident kernel by default (measured equal-or-faster and half the coordinates in
      // flight); SCD_CTA_KERNEL=stream selects the two-pass streaming variant
      // read once per process (the launch shape at create and every launch must agree)
      static const bool stream = getenv("SCD_CTA_KERNEL") && std::string(getenv("SCD_CTA_KERNEL")) == "stream";
      return stream ? (void *)k_epoch_stream<FORM, kCtaT, kStreamU, 8> : (void *)k_epoch_cta<FORM, kCtaT, kCtaE>;
    }
  }
}

// options.wild: the plain kernel of each bin with the non-atomic scatter (PASSCoDe-Wild comparison)
template <int FORM>
void *kernel_wild(int lanes) {
  switch (lanes) {
    case 8: return (void *)k_epoch_group<FORM, 8, kGrpE8, true>;
    case 16: return (void *)k_epoch_group<FORM, 16, 4, true>;
    case 32: return (void *)k_epoch_group<FORM, 32, kGrpE32, true>;
    case kLanesCluster: return nullptr;
    default: return (void *)k_epoch_cta<FORM, kCtaT, kCtaE, true>;
  }
}

template <int FORM, bool WILD>
void *cluster_kernel(int cl) {
  switch (cl) {
    case 2: return (void *)k_epoch_cluster<FORM, 2, kClusterThreads, kClE, WILD>;
    case 4: return (void *)k_epoch_cluster<FORM, 4, kClusterThreads, kClE, WILD>;
    case 16: {  // non-portable cluster size: opt in once per instantiation
      void *fn = (void *)k_epoch_cluster<FORM, 16, kClusterThreads, kClE, WILD>;
      cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      return fn;
    }
    default: return (void *)k_epoch_cluster<FORM, 8, kClusterThreads, kClE, WILD>;
  }
}

void *bin_kernel(const scd_ctx *c, const Bin &b) {
  if (b.hot > 0 && b.lanes == 8 && !c->opt.wild && c->hot_copy > 0 && !c->hot_view && c->hot_tp && c->hot_hp)
    return c->form == SCD_PRIMAL ? (void *)k_epoch_group_hot<SCD_PRIMAL, 8, 8, false, true, true, true>
                                 : (void *)k_epoch_group_hot<SCD_DUAL, 8, 8, false, true, true, true>;
  if (b.hot > 0 && b.lanes == 8 && !c->opt.wild && c->hot_copy > 0 && !c->hot_view && c->hot_tp)
    return c->form == SCD_PRIMAL ? (void *)k_epoch_group_hot<SCD_PRIMAL, 8, 8, false, true, true>
                                 : (void *)k_epoch_group_hot<SCD_DUAL, 8, 8, false, true, true>;
  if (b.hot > 0 && b.lanes == 8 && !c->opt.wild && c->hot_copy > 0 && !c->hot_view)
    return c->form == SCD_PRIMAL ? (void *)k_epoch_group_hot<SCD_PRIMAL, 8, 8, false, true>
                                 : (void *)k_epoch_group_hot<SCD_DUAL, 8, 8, false, true>;
  if (b.hot > 0 && b.lanes == 8 && !c->opt.wild) {
    if (c->form == SCD_PRIMAL)
      return c->hot_view ? (void *)k_epoch_group_hot<SCD_PRIMAL, 8, 8, true> : (void *)k_epoch_group_hot<SCD_PRIMAL, 8, 8, false>;
    return c->hot_view ? (void *)k_epoch_group_hot<SCD_DUAL, 8, 8, true> : (void *)k_epoch_group_hot<SCD_DUAL, 8, 8, false>;
  }
  if (b.lanes == kLanesCluster) {
    if (c->form == SCD_PRIMAL)
      return c->opt.wild ? cluster_kernel<SCD_PRIMAL, true>(b.cl) : cluster_kernel<SCD_PRIMAL, false>(b.cl);
    return c->opt.wild ? cluster_kernel<SCD_DUAL, true>(b.cl) : cluster_kernel<SCD_DUAL, false>(b.cl);
  }
  if (c->opt.wild) return c->form == SCD_PRIMAL ? kernel_wild<SCD_PRIMAL>(b.lanes) : kernel_wild<SCD_DUAL>(b.lanes);
  if (b.split && b.lanes == kLanesCta)
    return c->form == SCD_PRIMAL ? (void *)k_epoch_split<SCD_PRIMAL, kCtaT, kCtaE>
                                 : (void *)k_epoch_split<SCD_DUAL, kCtaT, kCtaE>;
  if (b.head > 0 && b.lanes == kLanesCta && c->tail_snap && c->head_snap && c->form == SCD_DUAL)
    return c->tail_snap == 2 ? (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, true, 2>
                             : (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, true, 1>;
  if (b.head > 0 && b.lanes == kLanesCta && c->tail_snap && !c->head_snap && c->form == SCD_DUAL) {
    if (c->head_pf && c->head_copy > 0 && c->tail_snap == 1)
      return c->head_T == 512 ? (void *)k_epoch_cta_head<SCD_DUAL, 512, kCtaE, false, 1, true, true>
                              : (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, false, 1, true, true>;
    if (c->head_pf)
      return c->tail_snap == 2 ? (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, false, 2, true>
                               : (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, false, 1, true>;
    return c->tail_snap == 2 ? (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, false, 2>
                             : (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, false, 1>;
  }
  if (b.head > 0 && b.lanes == kLanesCta)
    return c->head_snap ? (c->form == SCD_PRIMAL ? (void *)k_epoch_cta_head<SCD_PRIMAL, kCtaT, kCtaE, true>
                                                 : (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, true>)
                        : (c->form == SCD_PRIMAL ? (void *)k_epoch_cta_head<SCD_PRIMAL, kCtaT, kCtaE, false>
                                                 : (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, false>);
  return c->form == SCD_PRIMAL ? kernel_for<SCD_PRIMAL>(b.lanes, b.plain) : kernel_for<SCD_DUAL>(b.lanes, b.plain);
}

EpochArgs make_args(scd_ctx *c) {
  EpochArgs a;
  a.ptr = c->ptr;
  a.idx = c->idx;
  a.val = c->val;
  a.y = c->y;
  a.norm = c->norm;
  a.x = c->x;
  a.sv = c->sv;
  a.svr = c->tail_snap ? c->svr : c->sv;
  a.svg = c->sv;
  a.roll_R = c->tail_roll;
  a.head_P = c->head_copy;
  a.roll_lo = c->tail_lo;
  a.roll_hi = c->tail_hi;
  a.lam = c->lam;
  a.lamN = c->lamN;
  return a;
}

cudaEvent_t get_event(scd_ctx *c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

}  // namespace

// Combined (deferred) updates — the head kernel's pending head, the hot-set kernel's pending hot
// entries — are missed by other CTAs' reads for a whole window, so their windows are sized against
// the bin's staleness bound itself: `inflight` coordinates in flight plus `inflight` * window * k
// deferred ones <= SCD_COMBINE_BUDGET * τ_b (default 1.0; an explicit max_inflight replaces τ_b).
// The in-flight cap keeps its 0.5 safety factor.  Measured (profiles/hot_sweep_r1.txt,
// head_sweep_r1.txt): per-epoch gaps unchanged within 3% up to 2 τ, divergence beyond ~4 τ.
//
// The per-epoch rate also depends on how large a fraction of the epoch is stale at once: on a
// 20 000-row C3 prefix a window of 5 rows per CTA (3 500 of 19 400 coordinates deferred) left the
// gap 15x behind the sequential one after 4 epochs, so the deferred total is also kept <= 1/8 of the
// bin's coordinates (never binding on the full-size configs).
double combine_budget(const scd_ctx *c, const Bin &b) {
  const double frac = getenv("SCD_COMBINE_BUDGET") ? atof(getenv("SCD_COMBINE_BUDGET")) : 1.0;
  const double budget = c->opt.max_inflight > 0 ? (double)b.cap : frac * b.tau;
  return std::min(budget, (double)b.count / 8.0);
}

int64_t combine_window(const scd_ctx *c, const Bin &b, int64_t inflight, int64_t k) {
  const double budget = combine_budget(c, b);
  if (inflight < 1 || budget <= 0) return 0;
  return (int64_t)((budget / (double)inflight - 1.0) / (double)k);
}

// Hot-set bin (k_epoch_group_hot): 512-thread CTAs (64 rows in flight per CTA, one CTA per SM),
// window F batches.  At a fixed budget the rows a CTA combines per flush (rows per CTA x F) is what
// counts: 512 threads at F = 7 beat 256 threads at F = 7 with twice the CTAs (26.9 vs 31.9 ms on a
// C5 shard).  The grid is lowered (in steps of one CTA per SM, not below one per SM) until F >= 6
// fits the budget.  SCD_HOT_T=256, SCD_HOT_F, SCD_HOT_CTAS (CTAs per SM) override (experiments).
void hot_launch_shape(scd_ctx *c, Bin &b) {
  void *fn = bin_kernel(c, b);
  const size_t smem = 8 * (size_t)b.hot;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  const int T0 = getenv("SCD_HOT_T") && atoi(getenv("SCD_HOT_T")) == 256 ? 256 : 512;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, T0, smem);
  if (occ < 1) occ = 1;
  if (const char *e = getenv("SCD_HOT_CTAS")) occ = std::max(1, std::min(occ, atoi(e)));
  const int T = getenv("SCD_HOT_T") && atoi(getenv("SCD_HOT_T")) == 256 ? 256 : 512;
  const int64_t k = c->hot_view ? 2 : 1, rows = T / 8;
  const int64_t need = (b.count + rows - 1) / rows;
  int64_t grid = std::min<int64_t>((int64_t)c->nsm * occ, std::max<int64_t>(need, 1));
  const char *fe = getenv("SCD_HOT_F");
  const int64_t min_grid = (int64_t)c->nsm * (T == 512 ? 1 : 2);
  while (!fe && combine_window(c, b, grid * rows, k) < 6 && grid > min_grid) grid -= c->nsm;
  int64_t F = std::max<int64_t>(1, std::min<int64_t>(64, combine_window(c, b, grid * rows, k)));
  if (fe) F = std::max(1, atoi(fe));
  if (!fe && F < 4) {  // too short a window to beat the CTA-combining kernel: use that instead
    b.hot = 0;
    bin_launch_shape(c, b);
    return;
  }
  b.grid = (int)std::max<int64_t>(grid, 1);
  b.block = T;
  b.flush = (int)F;
  // Hot copy: the copy's age, P · K/32 warp tickets of rows/warp rows each, joins the window budget:
  // rows in flight · (1 + F + hp) + age <= budget, hp = 1 when the hot values are also gathered one
  // step early (hot_hp: one more round of the rows in flight); F gives way (down to 4) until P >= 8
  // fits.  SCD_HOT_COPY=0: off, =P: forced period; SCD_HOT_HP=0: no early hot gathers.
  c->hot_copy = 0;
  c->hot_hp = !(getenv("SCD_HOT_HP") && atoi(getenv("SCD_HOT_HP")) == 0);
  const char *hce = getenv("SCD_HOT_COPY");
  if (!c->hot_view && !(hce && atoll(hce) == 0) && T == 512) {
    const double budget = combine_budget(c, b);
    const int64_t inflight = (int64_t)b.grid * rows, nch = (b.hot + 31) / 32, cpw = 32 / 8;
    const double hp = c->hot_hp ? 1.0 : 0.0;
    int64_t P = 0, f = F;
    for (; f >= 4; --f) {
      P = (int64_t)((budget - (double)inflight * (1.0 + hp + f)) / (double)(nch * cpw));
      if (P >= 8) break;
    }
    if (hce) P = atoll(hce);
    if (P >= 8 || hce) {
      if (!c->hot_hc && cudaMalloc((void **)&c->hot_hc, sizeof(float) * (size_t)b.hot) != cudaSuccess) {
        cudaGetLastError();
        c->hot_hc = nullptr;
        return;
      }
      c->hot_copy = std::max<int64_t>(1, P);
      if (!hce) b.flush = (int)f;
    }
  }
}

// Grid/block for a bin (used by build_schedule): persistent, sized to the SM count times the
// kernel's residency, capped by max_inflight coordinates in flight.
void bin_launch_shape(scd_ctx *c, Bin &b) {
  // A cap below a kernel's minimum batch must still be honoured (staleness): the
  // combining kernel runs kCombT/8 coordinates per CTA, the 8-lane kernel >= 4 per warp, so small
  // caps fall back to the plain 8-lane kernel, and caps below 4 to one warp per coordinate.
  if (b.lanes == 8 && b.cap > 0 && b.cap < kCombT / 8) b.plain = 1;
  if (b.lanes == 8 && b.cap > 0 && b.cap < 4) b.lanes = 32;
  if (c->opt.wild) {  // plain kernels only (no head / CTA combining, no die split)
    b.plain = 1;
    b.head = b.split = 0;
  }
  if (b.lanes != kLanesCta) b.head = b.split = 0;
  if (b.split) b.head = 0;
  if (b.lanes == kLanesCluster) {
    // cluster size: large clusters split one very long coordinate over more SMs, small ones keep
    // more coordinates in flight; SCD_CLUSTER = 2|4|8 overrides
    const int env_cl = getenv("SCD_CLUSTER") ? atoi(getenv("SCD_CLUSTER")) : 0;
    b.cl = (env_cl == 2 || env_cl == 4 || env_cl == 8 || env_cl == 16) ? env_cl : kClusterCtas;
  }
  if (b.hot > 0 && (b.lanes != 8 || c->opt.wild)) b.hot = 0;
  if (b.hot > 0) {
    hot_launch_shape(c, b);
    return;
  }
  void *fn = bin_kernel(c, b);
  const bool group = (b.lanes <= 32);
  const bool clus = (b.lanes == kLanesCluster);
  const bool comb = (b.lanes == 8 && !b.plain && group_kind() == 2);  // fixed CTA size (kernel template)
  int block = comb ? kCombT : (group ? 256 : (clus ? kClusterThreads : (b.head > 0 ? c->head_T : kCtaT)));
  // sub-warp bins with a small cap shrink the CTA so the cap can be honoured (>= one warp)
  if (group && !comb && b.cap > 0 && b.cap * b.lanes < block) {
    block = (int)(((b.cap * b.lanes) + 31) / 32 * 32);
    if (block < 32) block = 32;
  }
  const size_t smem = b.head > 0 ? sizeof(float) * (size_t)b.head * (c->head_snap ? 2 : 1) : 0;
  if (smem > 0) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, block, smem);
  if (occ < 1) occ = 1;
  const int per_launch_unit = clus ? b.cl : 1;                    // CTAs per coordinate slot
  const int coords_per_cta = group ? block / b.lanes : 1;
  int64_t slots = (int64_t)c->nsm * occ / per_launch_unit;        // resident coordinate slots
  if (clus && slots > (int64_t)c->nsm / b.cl * occ) slots = (int64_t)c->nsm / b.cl * occ;
  int64_t units = slots;                                          // CTAs (or clusters)
  if (b.cap > 0) {  // staleness cap
    int64_t u = (b.cap + coords_per_cta - 1) / coords_per_cta;
    if (u < units) units = u;
  }
  int64_t need = (b.count + coords_per_cta - 1) / coords_per_cta;
  if (units > need) units = need;
  if (units < 1) units = 1;
  b.grid = (int)(units * per_launch_unit);
  b.block = block;
  if (b.head > 0) {
    // Pending head updates of `flush` coordinates per CTA are missed by other CTAs' reads, on top
    // of the grid coordinates in flight: grid * (1 + flush * k) <= combined-update budget, k = 2
    // with the shared-memory view (a read may also miss what others flushed since the CTA's last
    // refresh).  SCD_HEAD_FLUSH overrides (experiments only).
    const int64_t k = c->head_snap ? 2 : 1;
    int64_t f = combine_window(c, b, b.grid, k);
    if (const char *e = getenv("SCD_HEAD_FLUSH")) f = atoi(e);
    if (f > 64) f = 64;
    if (f < 2 && c->head_snap) {  // no room for the view: plain head kernel
      c->head_snap = false;
      bin_launch_shape(c, b);
      return;
    }
    if (f < 2) {  // no combining possible within the budget: plain CTA kernel
      b.head = 0;
      b.flush = 0;
      bin_launch_shape(c, b);
      return;
    }
    b.flush = (int)f;
  }
}

// Launch one bin's kernel over the permutation positions [ba.lo, ba.hi) with `grid` CTAs.
scd_status launch_bin(scd_ctx *c, const Bin &b, EpochArgs &a, BinArgs &ba, int64_t grid, cudaStream_t s) {
  void *fn = bin_kernel(c, b);
  int H = b.head, F = b.flush;
  void *args_head[] = {&a, &ba, &H, &F};
  SplitArgs sa;
  void *args_split[] = {&a, &ba, &sa};
  HotArgs ha;
  void *args_hot[] = {&a, &ba, &ha};
  void **args = args_head;
  if (b.hot > 0 && b.lanes == 8 && !c->opt.wild) {
    ha.idx = c->hot_idx;
    ha.hot_ids = c->hot_ids;
    ha.K = b.hot;
    ha.F = b.flush;
    ha.hc = c->hot_hc;
    ha.P = (int)std::max<int64_t>(1, c->hot_copy);
    args = args_hot;
  }
  if (b.split) {
    sa.mid = c->split_mid;
    sa.idx = c->split_idx;
    sa.val = c->split_val;
    sa.sm_die = c->sm_die;
    sa.slot_p = c->slot_p;
    sa.slot_tag = c->slot_tag;
    sa.err = c->split_err;
    sa.counter1 = ba.counter + kMaxBins * kMaxSlices;    // die 1's counter: same (slice, bin), second half
    if (++c->launch_tag == 0) ++c->launch_tag;                  // 0 = never written
    sa.tag = c->launch_tag;
    sa.nosync = c->split_nosync ? 1 : 0;
    args = args_split;
  }
  const size_t smem = b.hot > 0 ? 8 * (size_t)b.hot
                     : (b.head > 0 ? sizeof(float) * (size_t)b.head * (c->head_snap ? 2 : 1) : 0);
  SCD_CK(c, cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(b.block), args, smem, s));
  return SCD_OK;
}

// Part `part` of `nparts` of epoch `epoch`: permutation positions [n·part/nparts, n·(part+1)/nparts)
// (sub-epoch aggregation rounds; nparts = 1 is a whole epoch).
scd_status run_epoch(scd_ctx *c, uint32_t epoch, int part, int nparts) {
  EpochArgs a = make_args(c);
  cudaStream_t s = c->stream;
  if (c->opt.deterministic) {
    Perm p = make_perm(c->opt.seed, epoch, 0u, c->n_coord);
    const int64_t j0 = c->n_coord * part / nparts, j1 = c->n_coord * (part + 1) / nparts;
    if (c->form == SCD_PRIMAL)
      k_epoch_debug<SCD_PRIMAL><<<1, kDbgT, 0, s>>>(a, p, j0, j1);
    else
      k_epoch_debug<SCD_DUAL><<<1, kDbgT, 0, s>>>(a, p, j0, j1);
    SCD_CKL(c, "k_epoch_debug launch");
    ++c->launches;
    c->empty_dirty = false;
    return SCD_OK;
  }
  if (c->empty_dirty && c->n_empty > 0) {
    const int g = grid_for(c->n_empty, 256);
    if (c->form == SCD_PRIMAL)
      k_empty_fix<SCD_PRIMAL><<<g, 256, 0, s>>>(a, c->empty_list, c->n_empty);
    else
      k_empty_fix<SCD_DUAL><<<g, 256, 0, s>>>(a, c->empty_list, c->n_empty);
    SCD_CKL(c, "k_empty_fix launch");
    ++c->launches;
  }
  c->empty_dirty = false;
  if (c->n_bins == 0) return SCD_OK;
  // The epoch visits each bin in its own random order; the bins are interleaved in S slices so
  // that, at the granularity of a slice, the epoch order stays a random mix of all coordinates
  // (a bin-by-bin order converges much more slowly, DESIGN.md §6 / reading c24).
  const int S = c->n_slices;
  const int64_t Q = (int64_t)S * nparts;  // slices of the whole epoch; this part runs S of them
  SCD_CK(c, cudaMemsetAsync(c->counters, 0, sizeof(unsigned int) * kMaxBins * S, s));
  if (c->die_split)
    SCD_CK(c, cudaMemsetAsync(c->counters + kMaxBins * kMaxSlices, 0, sizeof(unsigned int) * kMaxBins * S, s));
  for (int sl = 0; sl < S; ++sl) {
    const int64_t q = (int64_t)part * S + sl;
    for (int i = 0; i < c->n_bins; ++i) {
      Bin &b = c->bins[i];
      BinArgs ba;
      ba.list = b.list;
      ba.lo = b.count * q / Q;
      ba.hi = b.count * (q + 1) / Q;
      if (ba.hi <= ba.lo) continue;
      ba.counter = c->counters + sl * kMaxBins + i;
      ba.perm = make_perm(c->opt.seed, epoch, b.stream_id, b.count);
      ba.dry = 0;
      const int cpc = b.lanes <= 32 ? b.block / b.lanes : 1;  // coordinates per CTA (or cluster) per round
      const int unit = b.lanes == kLanesCluster ? b.cl : 1;
      const int64_t need = ((ba.hi - ba.lo) + cpc - 1) / cpc;
      int64_t grid = b.grid / unit;
      if (grid > need) grid = need;
      if (grid < 1) grid = 1;
      if (c->tail_snap && b.head > 0 && b.lanes == kLanesCta) {
        k_tail_refresh<<<c->nsm * 4, 256, 0, s>>>(c->sv, c->svr, c->head_copy > 0 ? 0 : c->tail_lo, c->tail_hi);
        SCD_CKL(c, "k_tail_refresh launch");
        ++c->launches;
      }
      if (c->hot_copy > 0 && b.hot > 0 && b.lanes == 8) {
        k_hot_refresh<<<grid_for(b.hot, 256), 256, 0, s>>>(c->sv, c->hot_ids, b.hot, c->hot_hc);
        SCD_CKL(c, "k_hot_refresh launch");
        ++c->launches;
      }
      EpochArgs ab = a;
      if (b.snap) {  // snapshot bin: the whole slice launch gathers from a copy taken just before it
        k_tail_refresh<<<c->nsm * 4, 256, 0, s>>>(c->sv, c->svr, 0, c->n_shared);
        SCD_CKL(c, "k_tail_refresh launch");
        ++c->launches;
        ab.svg = c->svr;
      }
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (c->opt.profile) {
        e0 = get_event(c);
        e1 = get_event(c);
        cudaEventRecord(e0, s);
      }
      scd_status st = launch_bin(c, b, ab, ba, grid * unit, s);
      if (st != SCD_OK) return st;
      ++c->launches;
      if (c->opt.profile) {
        cudaEventRecord(e1, s);
        c->ev_pending.push_back({i, {e0, e1}});
      }
    }
  }
  return SCD_OK;
}

// Shared-vector placement.  The epoch's hottest traffic goes to the head of the shared vector
// (the frequency-ranked features of every row), and how those few lines fall onto L2 slices and
// dies moves the C3 dual epoch between 13.0 and 20.4 ms for byte offsets of the vector within its
// allocation (tools/offset_check.py).  The hash is not documented, so the offset is
// chosen empirically at create: a dry probe of the dominant bin (identical gather/atomic traffic,
// scatter adds +0.0f, model untouched) is timed for each candidate offset and the fastest kept.
scd_status tune_shared_layout(scd_ctx *c) {
  int bi = -1;
  for (int i = 0; i < c->n_bins; ++i)
    if (c->bins[i].lanes != kLanesCluster && (bi < 0 || c->bins[i].nnz > c->bins[bi].nnz)) bi = i;
  if (bi < 0) return SCD_OK;
  Bin &b = c->bins[bi];
  cudaStream_t s = c->stream;
  const int cpc = b.lanes <= 32 ? b.block / b.lanes : 1;
  const int64_t probe = std::min<int64_t>(b.count, (int64_t)b.grid * cpc * 8);  // ~0.14 ms per C3 probe launch
  SCD_CK(c, cudaMemsetAsync(c->sv_base, 0, sizeof(float) * (size_t)(c->n_shared + kMaxSvOffsetFloats), s));
  // all probe launches enqueued back to back between events (one warm-up, then kReps per candidate
  // in round-robin order so slow drifts hit every candidate alike); one synchronisation at the end
  constexpr int kReps = 2;
  const int nl = 1 + kSvCandidates * kReps;
  std::vector<cudaEvent_t> ev(nl + 1);
  for (auto &e : ev) SCD_CK(c, cudaEventCreate(&e));
  SCD_CK(c, cudaMemsetAsync(c->counters, 0, sizeof(unsigned int) * 2 * kMaxBins * kMaxSlices, s));
  SCD_CK(c, cudaEventRecord(ev[0], s));
  for (int l = 0; l < nl; ++l) {
    const int ci = l == 0 ? 0 : (l - 1) % kSvCandidates;
    c->sv = c->sv_base + kSvCandidateBytes[ci] / 4;
    EpochArgs a = make_args(c);
    BinArgs ba;
    ba.list = b.list;
    ba.lo = 0;
    ba.hi = probe;
    ba.perm = make_perm(c->opt.seed ^ 0x5052424Full, 0xFFFFFFFEu, b.stream_id, b.count);
    ba.dry = 1;
    ba.counter = c->counters + l % (kMaxBins * kMaxSlices);
    if (l > 0 && l % (kMaxBins * kMaxSlices) == 0)
      SCD_CK(c, cudaMemsetAsync(c->counters, 0, sizeof(unsigned int) * 2 * kMaxBins * kMaxSlices, s));
    scd_status st = launch_bin(c, b, a, ba, (int64_t)b.grid, s);
    if (st != SCD_OK) return st;
    SCD_CK(c, cudaEventRecord(ev[l + 1], s));
    ++c->launches;
  }
  SCD_CK(c, cudaEventSynchronize(ev[nl]));
  std::vector<float> best_of(kSvCandidates, 1e30f);
  for (int l = 1; l < nl; ++l) {
    float ms = 0.f;
    SCD_CK(c, cudaEventElapsedTime(&ms, ev[l], ev[l + 1]));
    const int ci = (l - 1) % kSvCandidates;
    best_of[ci] = std::min(best_of[ci], ms);
  }
  for (auto &e : ev) cudaEventDestroy(e);
  SCD_CK(c, cudaMemsetAsync(c->counters, 0, sizeof(unsigned int) * 2 * kMaxBins * kMaxSlices, s));
  int best = 0;
  c->n_probe = 0;
  for (int ci = 0; ci < kSvCandidates; ++ci) {
    c->probe_ms[c->n_probe++] = best_of[ci];
    if (best_of[ci] < best_of[best]) best = ci;
  }
  c->sv = c->sv_base + kSvCandidateBytes[best] / 4;
  c->sv_offset_bytes = kSvCandidateBytes[best];
  return SCD_OK;
}

scd_status profile_collect(scd_ctx *c) {
  for (auto &p : c->ev_pending) {
    float ms = 0.f;
    SCD_CK(c, cudaEventSynchronize(p.second.second));
    SCD_CK(c, cudaEventElapsedTime(&ms, p.second.first, p.second.second));
    c->bins[p.first].ms += ms;
    c->bins[p.first].prof_launches += 1;
    c->ev_pool.push_back(p.second.first);
    c->ev_pool.push_back(p.second.second);
  }
  c->ev_pending.clear();
  return SCD_OK;
}

scd_status launch_perm_export(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n, int64_t *d_out,
                              cudaStream_t s) {
  Perm p = make_perm(seed, epoch, stream, n);
  k_perm_export<<<grid_for(n, 256), 256, 0, s>>>(p, n, d_out);
  return cudaGetLastError() == cudaSuccess ? SCD_OK : SCD_E_CUDA;
}

scd_status launch_partition_export(uint64_t seed, int64_t count, int32_t k, int32_t *d_owner, cudaStream_t s) {
  Perm p = make_perm(seed, 0u, kPartStream, count);
  k_partition_export<<<grid_for(count, 256), 256, 0, s>>>(p, count, k, d_owner);
  return cudaGetLastError() == cudaSuccess ? SCD_OK : SCD_E_CUDA;
}

}  // namespace scd
