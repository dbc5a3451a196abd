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
  int64_t nnz;               // stored entries (bound of the bulk copies of k_epoch_cluster_tma)
};

struct BinArgs {
  const int32_t *list;  // coordinate ids of the bin (ascending); nullptr = identity
  int64_t lo, hi;       // this launch processes permutation positions [lo, hi) of the bin
  int64_t blk;          // > 1: block order (reading c28): perm permutes the count / blk full blocks
  int blk_shift;        // log2(blk) (blk is a power of two)
  const int32_t *bperm; // block order: the epoch's block permutation materialised (nullptr: evaluate perm)
  int zero;             // 0 at run time (ticket_async)
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

// Ticket atomic of one lane whose result is consumed later (a prefetch).  ptxas turns an atomicAdd
// on a warp-uniform address into a warp-aggregated one whose result shuffle waits for the atomic right
// away (profiles/ncu_c5_hot_r2b: 16% of the hot kernel's stall samples on that shuffle); an address it
// cannot prove uniform (offset lane * b.zero, b.zero = 0 at run time) keeps the plain ATOMG, so the
// round trip overlaps the work until the ticket is used.
__device__ __forceinline__ unsigned ticket_async(const struct BinArgs &b, unsigned n) {
  unsigned l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));  // opaque to the compiler (it knows the caller's lane)
  return atomicAdd(b.counter + l * (unsigned)b.zero, n);
}

// Position t of the bin's epoch order -> coordinate.  Block order (blk > 1, reading c28): the full
// blocks of blk consecutive coordinates of the bin are visited in the keyed permutation's order and
// the coordinates of a block in turn; the last, partial block (count mod blk) comes last.  A bijection
// on [0, count), so every coordinate is still visited exactly once per epoch.
__device__ __forceinline__ int64_t bin_coord(const BinArgs &b, uint64_t t) {
  uint64_t j;
  if (b.blk > 1) {
    const uint64_t tb = t >> b.blk_shift;
    j = tb < b.perm.n ? (((b.bperm ? (uint64_t)__ldg(b.bperm + tb) : perm_apply(b.perm, tb)) << b.blk_shift) |
                         (t & (uint64_t)(b.blk - 1)))
                      : t;
  } else {
    j = perm_apply(b.perm, t);
  }
  return b.list ? (int64_t)__ldg(b.list + j) : (int64_t)j;
}

// ----------------------------------------------------------------------------------------------
// Register-resident CTA kernel: E entries per thread held in registers between the gather-dot and
// the scatter (longer coordinates re-read the rest from L2 for the scatter).
template <int FORM, int T, int E, bool WILD = false>
__global__ void __launch_bounds__(T) k_epoch_cta(EpochArgs a, BinArgs b) {
  constexpr int NW = T / 32;
  if (blockDim.x != T) __trap();  // the host's launch shape must match the template
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

template <int T>
__device__ __forceinline__ void head_flush(float *sv, float *s_acc, int H, int dry) {
  float4 *a4 = reinterpret_cast<float4 *>(s_acc);
  for (int i = threadIdx.x; i < H / 4; i += T) {
    const float4 v = a4[i];
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

// Shared-vector read of an entry of the row.  Head entries (id < H): L2 value + this
// CTA's pending part, the L2 value from the rolling head copy svr[0, H) with HC, else from sv.  Tail
// entries: from the read copy svr with TS (refreshed in rolling chunks / before every slice, never
// reduced into), else from sv.  Gathered and reduced lines are then disjoint, which the L2 serves
// ~35% faster (profiles/mix_bench_r1.txt: 84 -> 114 G gather+RED pairs/s).
template <int TS, bool HC>
__device__ __forceinline__ float ld_entry(const EpochArgs &a, const float *s_acc, int H, int32_t j) {
  if (j < H) return ld_sv((HC ? a.svr : a.sv) + j) + s_acc[j];
  return ld_sv((TS ? a.svr : a.sv) + j);
}

// Thread 0 prefetches the next coordinate (ticket, permutation, offsets, model, norm, label) while
// the CTA works on the current one and publishes it through shared memory, so the ticket -> Feistel
// -> ptr -> x chain (three dependent round trips) leaves the per-row critical path.  The prefetched
// coordinate reads nothing of the shared vector before its turn, so this adds no staleness; x[c'] is
// current because this CTA is its only writer in the epoch (c10).
template <int FORM, int T, int E, int TS, bool HC>
__global__ void __launch_bounds__(T, 1024 / T) k_epoch_cta_head(EpochArgs a, BinArgs b, int H, int flush) {
  constexpr int NW = T / 32;
  if (blockDim.x != T) __trap();  // the host's launch shape must match the template
  extern __shared__ float4 s_dyn[];
  float *s_acc = reinterpret_cast<float *>(s_dyn);
  __shared__ float s_red[NW];
  __shared__ float s_delta;
  __shared__ int64_t s_cur[4];  // coordinate (-1 = slice done), ptr[c], ptr[c + 1], its position t
  __shared__ float s_cx[3];     // x[c], norm[c], y[c]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < H; i += T) s_acc[i] = b.dry ? -0.f : 0.f;
  int64_t n_c = -1, n_beg = 0, n_end = 0, n_t = 0;  // thread 0: the next coordinate
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
  if (tid == 0) fetch(ticket_async(b, 1u));
  int since = 0;
  for (;;) {
    if (tid == 0) {
      s_cur[0] = n_c;
      s_cur[1] = n_beg;
      s_cur[2] = n_end;
      s_cur[3] = n_t;
      s_cx[0] = n_x;
      s_cx[1] = n_nrm;
      s_cx[2] = n_y;
      if (n_c >= 0) n_tk = ticket_async(b, 1u);  // consumed after this row's gathers
    }
    __syncthreads();  // also orders the previous coordinate's s_acc updates before this one's reads
    const int64_t c = s_cur[0];
    if (c < 0) break;
    const int64_t beg = s_cur[1], end = s_cur[2];
    if (HC && !b.dry && s_cur[3] % a.head_P == 0) {
      // head copy: row position t refreshes chunk (t / head_P) mod (H / 4T) of svr[0, H)
      const int64_t nchh = ((int64_t)H + T * 4 - 1) / (T * 4);
      const int64_t ih = ((s_cur[3] / a.head_P) % nchh) * (T * 4) + (int64_t)tid * 4;
      if (ih + 3 < H)
        *reinterpret_cast<float4 *>(const_cast<float *>(a.svr) + ih) = __ldcg(reinterpret_cast<const float4 *>(a.sv + ih));
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
      if (id[e] >= 0) acc = fmaf(ld_entry<TS, HC>(a, s_acc, H, id[e]), v[e], acc);
    for (int64_t base = beg + (int64_t)T * E; base < end; base += (int64_t)T * E) {
#pragma unroll 4
      for (int e = 0; e < E; ++e) {
        const int64_t k = base + (int64_t)e * T + tid;
        if (k < end) acc = fmaf(ld_entry<TS, HC>(a, s_acc, H, __ldcg(a.idx + k)), val_cg(a.val, k), acc);
      }
    }
    if (tid == 0) fetch(n_tk);  // next coordinate's chain overlaps reduce + scatter
    acc = warp_sum(acc);
    if (lane == 0) s_red[wid] = acc;
    __syncthreads();
    if (wid == 0) {
      float s = lane < NW ? s_red[lane] : 0.f;
      s = warp_sum(s);
      if (lane == 0) {
        const float xc = s_cx[0];
        const float d = coord_delta<FORM>(s, xc, s_cx[1], s_cx[2], a.lam, a.lamN);
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
      head_flush<T>(a.sv, s_acc, H, b.dry);
    }
  }
  head_flush<T>(a.sv, s_acc, H, b.dry);  // after the exit barrier: every pending update is final
}

// mbarrier + 1-D bulk copy (TMA) helpers
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
}

// ----------------------------------------------------------------------------------------------
// SM-shared head kernel with bulk-copied rows (default for the single head bin of a dual with the
// rolling tail copy: C3; DESIGN.md §6 "SM-shared head kernel").
//
// One CTA per SM runs G row groups of T threads (default 6 x 128, kSmG / kSmT); a group does one row at a
// time.  The G rows an SM has in flight share one shared-memory state of the frequency-ranked head:
//   S[0, H)  the SM's snapshot of w̄[0, H)
//   P[0, H)  the SM's pending updates of w̄[0, H) (not yet reduced into w̄)
// A head read is S[j] + P[j] (no L2 access; the head was ~620 L2 sector reads per C3 row), a tail read
// (j >= H) is the rolling tail read copy svr[j].  Head scatters are shared-memory
// compare-and-swap adds into P (the groups of an SM may hit the same entry), tail scatters red.global.add.
// Rolling flush by the SM's row count u: every rh-th row flushes head chunks (u/rh·ch + k) mod nh, k < ch,
// of 4T floats (exchange P with 0, one v4 RED per touched float4, S = the w̄ value loaded before that RED
// plus the flushed part, so S + P stays w̄ + the SM's own pending).  A head read then misses at most
// the other SMs' pending updates and what they flushed since its chunk's refresh, nh/ch·rh rows of every
// other SM each: that joins the combined-update budget (reading c25; sm_head_shape).
//
// The row's entries are not held in registers: each group streams its row through two shared-memory
// buffers of C entries (idx and val) filled by 1-D bulk copies (cp.async.bulk, completion on an mbarrier
// with a transaction count; the row itself is prefetched into L2 by cp.async.bulk.prefetch when it is
// published, a row ahead).  The gather-dot reads chunk i while chunk i + 1 is copied; the scatter walks
// the chunks backwards, so the last two are still resident and only rows longer than 2C re-read chunks
// (L2 hits); the buffers freed at the end of the scatter take the NEXT row's first two chunks, so a row
// starts with its entries on chip.  A buffer is handed back by the last of the group's warps to read it
// (shared-memory counter), which issues the next copy into it; the row descriptors and the partial sums
// are double-buffered by row parity, every warp derives the delta itself: one group barrier per row.
constexpr int kRollChunk = 1024;  // floats per rolling tail-copy refresh (= 4 * kLanesCta, as build_schedule assumes)

struct SmHeadArgs {
  int H;   // head snapshot / pending extent [0, H), a multiple of 4 * T
  int ch;  // head chunks flushed per flushing row
  int rh;  // rows per flushing row
};

template <int T>
__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "n"(T) : "memory");
}

__device__ __forceinline__ float4 exch4_zero(float *p) {
  float4 r;
  r.x = atomicExch(p + 0, 0.f);
  r.y = atomicExch(p + 1, 0.f);
  r.z = atomicExch(p + 2, 0.f);
  r.w = atomicExch(p + 3, 0.f);
  return r;
}

__device__ __forceinline__ bool nonzero4(float4 v) { return v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f; }

// Predicated accesses: the entries of a warp fall in both ranges (head / tail), and per-entry branches
// serialise the warp over the paths and keep the compiler from batching the loads of several entries.
__device__ __forceinline__ void red_if(float *p, float v, bool c) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q red.global.add.f32 [%0], %1; }" ::"l"(p), "f"(v), "r"((unsigned)c)
               : "memory");
}
// shared-memory CAS issued only where c holds; returns the value seen (o itself where c is false)
__device__ __forceinline__ unsigned cas_shared_if(float *p, unsigned o, unsigned n, bool c) {
  unsigned r = o;
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %4, 0; @q atom.shared.cas.b32 %0, [%1], %2, %3; }"
               : "+r"(r)
               : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(o), "r"(n), "r"((unsigned)c)
               : "memory");
  return r;
}

// Shared-vector read of entry j: S[j] + P[j] for j < H, svr[j] beyond; the shared-memory and the L2
// load land in one register under complementary predicates.  j < 0 (no entry) reads S[0] + P[0]; the
// caller gives it a zero weight.
__device__ __forceinline__ float sm_read(const float *S, const float *P, const float *svr, int H, int32_t j) {
  float r, p;
  const unsigned js = (unsigned)max(j, 0) * 4u;
  asm("{ .reg .pred q; setp.lt.s32 q, %2, %3;\n\t"
      "@q ld.shared.f32 %0, [%4];\n\t"
      "@!q ld.global.cg.f32 %0, [%5];\n\t"
      "mov.f32 %1, 0f00000000;\n\t"
      "@q ld.shared.f32 %1, [%6]; }"
      : "=f"(r), "=f"(p)
      : "r"(j), "r"(H), "r"(smem_u32(S) + js), "l"(svr + j), "r"(smem_u32(P) + js));
  return r + p;
}

// Scatter of 4 entries (id < 0 = none): ids < H into the SM's pending P, the rest with red.global.add.
// The pending adds are compare-and-swap rounds issued for all 4 entries at once (an fp32 shared-memory
// atomicAdd compiles to one CAS loop per entry, each waiting out two shared-memory round trips); another
// group of the SM rarely hits the same entry at the same time, so the retry loop almost never runs.
__device__ __forceinline__ void pend_scatter4(float *P, float *sv, int H, const int32_t *id, const float *v, float d) {
  unsigned o[4];
  bool pend[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    pend[q] = id[q] >= 0 && id[q] < H;
    o[q] = __float_as_uint(P[min((unsigned)id[q], (unsigned)H - 1u)]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float dv = v[q] * d;
    const unsigned r = cas_shared_if(P + id[q], o[q], __float_as_uint(__uint_as_float(o[q]) + dv), pend[q]);
    red_if(sv + id[q], dv, id[q] >= H);
    pend[q] = pend[q] && r != o[q];  // lost the race: retry from the value seen
    o[q] = r;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    while (pend[q]) {
      const unsigned n = __float_as_uint(__uint_as_float(o[q]) + v[q] * d);
      const unsigned r = atomicCAS(reinterpret_cast<unsigned *>(P + id[q]), o[q], n);
      pend[q] = r != o[q];
      o[q] = r;
    }
}

struct RowInfo {
  int64_t c, beg, end, t;  // coordinate (-1 = none), its entries [beg, end), its position t
  float x, nrm, y;         // x[c], norm[c], y[c]
  unsigned u;              // SM row index
};

template <int C, int NW>
struct alignas(16) GroupSmem {
  int32_t idx[2][C + 4];
  float val[2][C + 4];
  uint64_t bar[2];
  int64_t a0[2], a1[2];  // buffer b holds the stored entries [a0, a1) (16-byte aligned copy)
  unsigned cnt[2];       // warps done with buffer b
  RowInfo row[2];        // by row parity
  RowInfo stg;           // the next row's loads land here (cp.async) until it is published
  float red[2][NW];      // partial sums by row parity
};

// Prefetch the stored entries [gb, ge) of a row into L2 (bulk prefetch, no shared memory): its chunks'
// bulk copies then hit L2 instead of DRAM.
__device__ __forceinline__ void prefetch_row_l2(const EpochArgs &a, int64_t gb, int64_t ge) {
  const int64_t a0 = gb & ~(int64_t)3;
  int64_t a1 = (ge + 3) & ~(int64_t)3;
  const int64_t lim = a.nnz & ~(int64_t)3;
  if (a1 > lim) a1 = lim;
  if (a1 <= a0) return;
  const unsigned bytes = (unsigned)(a1 - a0) * 4u;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.idx + a0), "r"(bytes) : "memory");
  if (a.val) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.val + a0), "r"(bytes) : "memory");
}

__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Copy the entries [gb, ge) (at most C) into buffer bi (one thread).  The copy covers the 16-byte aligned
// superset [gb & ~3, min(ceil4(ge), floor4(nnz))); entries past it (the last stored entries of the matrix
// only) are read from global memory by the consumer.
template <int C, int NW>
__device__ __forceinline__ void issue_chunk(const EpochArgs &a, GroupSmem<C, NW> *gs, int bi, int64_t gb, int64_t ge) {
  const int64_t a0 = gb & ~(int64_t)3;
  int64_t a1 = (ge + 3) & ~(int64_t)3;
  const int64_t lim = a.nnz & ~(int64_t)3;
  if (a1 > lim) a1 = lim;
  if (a1 < a0) a1 = a0;
  gs->a0[bi] = a0;
  gs->a1[bi] = a1;
  const unsigned bytes = (unsigned)(a1 - a0) * 4u;
  // the buffer was last read through the generic proxy (those reads are ordered before this thread by
  // the hand-back counter and a CTA fence)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(&gs->bar[bi], a.val ? 2u * bytes : bytes);
  if (bytes) {
    bulk_g2s(gs->idx[bi], a.idx + a0, bytes, &gs->bar[bi]);
    if (a.val) bulk_g2s(gs->val[bi], a.val + a0, bytes, &gs->bar[bi]);
  }
}

template <int C, int NW>
__device__ __forceinline__ void issue_row_chunk(const EpochArgs &a, GroupSmem<C, NW> *gs, int bi, const RowInfo &r, int i) {
  const int64_t gb = r.beg + (int64_t)i * C;
  issue_chunk<C, NW>(a, gs, bi, gb, min(r.end, gb + (int64_t)C));
}

// The warp is done reading buffer bi; the last warp of the group to get here issues the next copy into
// it: chunk i + 2 after the gather-dot of chunk i (the last two chunks stay for the scatter), chunk i - 2
// after the scatter of chunk i, the next row's chunk 0 / 1 after the scatter of chunk 1 / 0.
template <int C, int NW>
__device__ __forceinline__ void hand_back(const EpochArgs &a, GroupSmem<C, NW> *gs, int bi, int lane, bool scatter, int i,
                                          int n, int par) {
  __syncwarp();
  if (lane == 0) {
    __threadfence_block();
    if (atomicAdd(&gs->cnt[bi], 1u) == NW - 1) {
      gs->cnt[bi] = 0;
      __threadfence_block();
      const RowInfo &cur = gs->row[par];
      const RowInfo &nxt = gs->row[par ^ 1];
      if (!scatter) {
        if (i + 2 < n) issue_row_chunk<C, NW>(a, gs, bi, cur, i + 2);
      } else if (i >= 2) {
        issue_row_chunk<C, NW>(a, gs, bi, cur, i - 2);
      } else if (nxt.c >= 0) {
        const int nn = (int)((nxt.end - nxt.beg + C - 1) / C);
        if (i == 1) issue_row_chunk<C, NW>(a, gs, bi, nxt, 0);
        else if (nn >= 2) issue_row_chunk<C, NW>(a, gs, bi, nxt, 1);
      }
    }
  }
  __syncwarp();
}

// The U entries of this thread in chunk [cb, cb + ce) held by buffer bi (j = -1 past the chunk).
template <int C, int NW, int T, int U>
__device__ __forceinline__ void chunk_entries(const EpochArgs &a, const GroupSmem<C, NW> *gs, int bi, int64_t cb, int ce,
                                              int gt, int32_t *j, float *v) {
  const int off0 = (int)(cb - gs->a0[bi]), lim = (int)min(gs->a1[bi] - cb, (int64_t)C);
#pragma unroll
  for (int q = 0; q < U; ++q) {
    const int k = q * T + gt;
    j[q] = k < ce ? gs->idx[bi][off0 + k] : -1;
    v[q] = a.val ? gs->val[bi][off0 + min(k, C - 1)] : 1.f;
  }
  if (lim < ce) {  // the chunk runs past the aligned copy: the matrix's last stored entries
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int k = q * T + gt;
      if (k < ce && k >= lim) {
        j[q] = __ldg(a.idx + cb + k);
        v[q] = a.val ? __ldg(a.val + cb + k) : 1.f;
      }
    }
  }
}

template <int FORM, int G, int T, int C>
__global__ void __launch_bounds__(G *T, 1) k_epoch_sm_tma(EpochArgs a, BinArgs b, SmHeadArgs h) {
  constexpr int NW = T / 32;
  if (blockDim.x != G * T) __trap();  // the host's launch shape must match the template
  constexpr int CH = 4 * T;  // floats per flushed chunk (one float4 per thread of a group)
  constexpr int U = C / T;   // entries per thread per chunk
  static_assert(C % T == 0 && U % 4 == 0, "chunk shape");
  extern __shared__ float4 s_dyn[];
  float *S = reinterpret_cast<float *>(s_dyn);
  float *P = S + h.H;
  __shared__ unsigned s_rows;
  const int tid = threadIdx.x, g = tid / T, gt = tid % T, lane = tid & 31, wl = gt >> 5;
  const int H = h.H;
  GroupSmem<C, NW> *gs = reinterpret_cast<GroupSmem<C, NW> *>(P + H) + g;
  for (int i = tid * 4; i < H; i += G * T * 4) {
    *reinterpret_cast<float4 *>(S + i) = __ldcg(reinterpret_cast<const float4 *>(a.sv + i));
    *reinterpret_cast<float4 *>(P + i) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (tid == 0) s_rows = 0;
  __syncthreads();
  // group thread 0: fetch of the next coordinate (ticket taken a row earlier); its offsets, model value,
  // norm and label are copied into gs->stg asynchronously (no registers held across the row)
  int64_t n_c = -1, n_t = 0;
  unsigned n_tk = 0;
  auto fetch = [&](unsigned tk) {
    n_t = b.lo + (int64_t)tk;
    n_c = -1;
    if (n_t >= b.hi) return;
    n_c = bin_coord(b, n_t);
    cp_async8(&gs->stg.beg, a.ptr + n_c);
    cp_async8(&gs->stg.end, a.ptr + n_c + 1);
    cp_async4(&gs->stg.x, a.x + n_c);
    cp_async4(&gs->stg.nrm, a.norm + n_c);
    if (FORM == SCD_DUAL) cp_async4(&gs->stg.y, a.y + n_c);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto publish = [&](int slot) {  // the fetched row becomes gs->row[slot]; its entries go to L2
    asm volatile("cp.async.wait_all;" ::: "memory");
    RowInfo &d = gs->row[slot];
    d.c = n_c;
    d.t = n_t;
    if (n_c >= 0) {
      d.beg = gs->stg.beg;
      d.end = gs->stg.end;
      d.x = gs->stg.x;
      d.nrm = gs->stg.nrm;
      d.y = FORM == SCD_DUAL ? gs->stg.y : 0.f;
      d.u = atomicAdd(&s_rows, 1u);
      prefetch_row_l2(a, d.beg, d.end);
    }
  };
  if (gt == 0) {
    mbar_init(&gs->bar[0], 1);
    mbar_init(&gs->bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    gs->cnt[0] = gs->cnt[1] = 0;
    fetch(ticket_async(b, 1u));
    n_tk = ticket_async(b, 1u);
    publish(0);
    const RowInfo &r0 = gs->row[0];
    if (r0.c >= 0) {
      issue_row_chunk<C, NW>(a, gs, 0, r0, 0);
      if (r0.end - r0.beg > C) issue_row_chunk<C, NW>(a, gs, 1, r0, 1);
    }
  }
  __syncthreads();
  const int nh = H / CH;
  unsigned ph = 0;  // mbarrier phase parity of the two buffers (bit b)
  int b0 = 0;       // buffer holding the current row's first chunk
  for (int par = 0;; par ^= 1) {
    const RowInfo &r = gs->row[par];  // read from shared memory where used
    const int64_t rc = r.c;
    if (rc < 0) break;
    const int64_t beg = r.beg, end = r.end;
    const int n = (int)((end - beg + C - 1) / C);
    if (gt == 0) {  // the next row: its loads overlap this row's gather-dot
      fetch(n_tk);
      n_tk = ticket_async(b, 1u);
    }
    if (a.roll_R > 0 && !b.dry && r.t % a.roll_R == 0) {
      // rolling tail copy: row position t refreshes chunk (t / roll_R) mod nchunks of svr,
      // in the 1024-float chunks build_schedule sized roll_R for (kRollChunk), whatever the group size
      const int64_t nch = (a.roll_hi - a.roll_lo + kRollChunk - 1) / kRollChunk;
      float *dst = const_cast<float *>(a.svr);
#pragma unroll
      for (int q = 0; q < (kRollChunk + 4 * T - 1) / (4 * T); ++q) {
        const int64_t i = a.roll_lo + ((r.t / a.roll_R) % nch) * kRollChunk + (int64_t)(q * T + gt) * 4;
        if (q * T + gt >= kRollChunk / 4) break;
        if (i + 3 < a.roll_hi)
          *reinterpret_cast<float4 *>(dst + i) = __ldcg(reinterpret_cast<const float4 *>(a.sv + i));
        else
          for (int64_t e = i; e < a.roll_hi && e < i + 4; ++e) dst[e] = __ldcg(a.sv + e);
      }
    }
    // the head chunk this row refreshes: its w̄ value is loaded now, consumed after the gather-dot
    const bool hfl = r.u % (unsigned)h.rh == 0;
    const unsigned hq = (r.u / (unsigned)h.rh) * (unsigned)h.ch;
    const int ih = (int)(hq % (unsigned)nh) * CH + gt * 4;
    float4 cur = make_float4(0.f, 0.f, 0.f, 0.f);
    if (hfl) cur = __ldcg(reinterpret_cast<const float4 *>(a.sv + ih));
    // gather-dot over the chunks
    float acc = 0.f;
    for (int i = 0; i < n; ++i) {
      const int bi = (b0 + i) & 1;
      mbar_wait(&gs->bar[bi], (ph >> bi) & 1u);
      ph ^= 1u << bi;
      const int64_t cb = beg + (int64_t)i * C;
      int32_t j[U];
      float v[U], w[U];
      chunk_entries<C, NW, T, U>(a, gs, bi, cb, (int)min((int64_t)C, end - cb), gt, j, v);
      // the entries are in registers: hand the buffer back before the gathers (the next copy into it
      // then overlaps their round trip)
      hand_back<C, NW>(a, gs, bi, lane, false, i, n, par);
#pragma unroll
      for (int q = 0; q < U; ++q) w[q] = sm_read(S, P, a.svr, H, j[q]);
#pragma unroll
      for (int q = 0; q < U; ++q) acc = fmaf(w[q], j[q] >= 0 ? v[q] : 0.f, acc);
    }
    // rolling flush of the SM's pending head; S refreshed from the value loaded before the RED
    if (hfl) {
      for (int k = 0; k < h.ch; ++k) {
        const int ik = (int)((hq + (unsigned)k) % (unsigned)nh) * CH + gt * 4;
        const float4 ck = k == 0 ? cur : __ldcg(reinterpret_cast<const float4 *>(a.sv + ik));
        const float4 pk = exch4_zero(P + ik);
        if (nonzero4(pk)) red_add_v4(a.sv + ik, pk);
        *reinterpret_cast<float4 *>(S + ik) = make_float4(ck.x + pk.x, ck.y + pk.y, ck.z + pk.z, ck.w + pk.w);
      }
    }
    if (gt == 0) publish(par ^ 1);  // the next row (read after the barrier below)
    acc = warp_sum(acc);
    if (lane == 0) gs->red[par][wl] = acc;
    group_sync<T>(g);
    // every warp sums the partials and derives the same delta (no second barrier)
    float sum = lane < NW ? gs->red[par][lane] : 0.f;
    sum = warp_sum(sum);
    float d = 0.f;
    if (lane == 0) d = coord_delta<FORM>(sum, r.x, r.nrm, r.y, a.lam, a.lamN);
    d = __shfl_sync(0xffffffffu, d, 0);
    if (gt == 0 && !b.dry) a.x[rc] = r.x + d;  // single writer per epoch (c10)
    d = b.dry ? 0.f : scatter_scale<FORM>(d);
    // a one-chunk row leaves the other buffer free from here on: the next row's first chunk goes there
    if (n == 1 && gt == 0 && n_c >= 0) issue_row_chunk<C, NW>(a, gs, b0 ^ 1, gs->row[par ^ 1], 0);
    // scatter, chunks in reverse order (the last two are still resident)
    for (int i = n - 1; i >= 0; --i) {
      const int bi = (b0 + i) & 1;
      if (i <= n - 3) {  // re-read (issued when chunk i + 2 was handed back)
        mbar_wait(&gs->bar[bi], (ph >> bi) & 1u);
        ph ^= 1u << bi;
      }
      const int64_t cb = beg + (int64_t)i * C;
      int32_t j[U];
      float v[U];
      chunk_entries<C, NW, T, U>(a, gs, bi, cb, (int)min((int64_t)C, end - cb), gt, j, v);
      hand_back<C, NW>(a, gs, bi, lane, true, i, n, par);
      if (d != 0.f || b.dry) {
#pragma unroll
        for (int q0 = 0; q0 < U; q0 += 4) pend_scatter4(P, a.sv, H, j + q0, v + q0, d);
      }
    }
    b0 ^= 1;  // the next row's first chunk went into the other buffer
  }
  __syncthreads();  // every group has left its loop: the pending updates are final
  for (int i = tid * 4; i < H; i += G * T * 4) {
    const float4 p = *reinterpret_cast<const float4 *>(P + i);
    if (nonzero4(p)) red_add_v4(a.sv + i, p);
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
// the CTA's rows update them concurrently); the warps run their rows without any CTA barrier and
// meet every F row batches to flush (one RED per touched hot entry) — so a hot line takes one RED
// per CTA per F batches instead of one per row.  Pending updates are extra staleness, bounded by the
// schedule: grid * rows per CTA * (1 + F) <= cap (plus the copy age and early gathers, below).
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
// E: entries per lane (5 covers the 39-entry criteo rows at 8 lanes); IMP: implicit values (val =
// NULL, NEXT-1: no value registers); T: threads of the one CTA per SM.
template <int FORM, int G, int E, bool HC = false, bool TP = false, bool HP = false, bool IMP = false, int T = 512>
__global__ void __launch_bounds__(T, 1) k_epoch_group_hot(EpochArgs a, BinArgs b, HotArgs h) {
  constexpr int CPW = 32 / G;
  const unsigned FULL = 0xffffffffu;
  extern __shared__ float4 s_dyn[];
  float *s_pend = reinterpret_cast<float *>(s_dyn);  // [K] pending updates of the hot entries
  int32_t *s_hid = reinterpret_cast<int32_t *>(s_pend + h.K);  // [K] shared-vector index of each slot
  const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
  for (int i = threadIdx.x; i < h.K; i += blockDim.x) {
    s_pend[i] = b.dry ? -0.f : 0.f;
    s_hid[i] = __ldg(h.hot_ids + i);
  }
  __syncthreads();
  // Software pipeline: while batch i gathers, reduces and scatters, the offsets, scalars and entries
  // of batch i+1 are loading, its ticket taken one batch earlier still (ticket_async).  Only batch i
  // reads the shared vector (plus the early gathers of batch i+1, TP / HP, counted in the window
  // budget), so the prefetches add no staleness; x[c] is current because this warp is its only
  // writer (c10).  A deeper pipeline (offsets two batches ahead) measured no faster
  // (profiles/c5_shape_r2.txt).
  unsigned tk_pf = 0;  // lane 0: ticket of the next take(), obtained one batch ahead
  if (lane == 0) tk_pf = ticket_async(b, (unsigned)CPW);
  auto take = [&]() -> int64_t {  // warp-uniform: this lane's coordinate of the next batch, -2 = none
    const unsigned int t0 = __shfl_sync(FULL, tk_pf, 0);
    if (b.lo + (int64_t)t0 >= b.hi) return -2;  // slice exhausted (uniform); every later ticket is too
    if (lane == 0) tk_pf = ticket_async(b, (unsigned)CPW);
    if (HC && !b.dry) {
      const int64_t tk = (b.lo + (int64_t)t0) / CPW;
      if ((tk & (int64_t)(h.P - 1)) == 0) {  // h.P is a power of two
        const int nch = (h.K + 31) / 32;
        const int sl = (int)((tk / h.P) % nch) * 32 + lane;
        if (sl < h.K) h.hc[sl] = __ldcg(a.sv + s_hid[sl]);
      }
    }
    int64_t cl = -1;
    if (lane < CPW && b.lo + (int64_t)t0 + lane < b.hi) cl = bin_coord(b, b.lo + t0 + lane);
    return __shfl_sync(FULL, cl, sub);
  };
  struct Meta {
    int64_t c, beg, end;
    float xc, nrm, yc;
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
  auto load_meta = [&](Meta &m, int64_t c) {
    m.c = c;
    m.beg = m.end = 0;
    m.xc = m.nrm = m.yc = 0.f;
    if (c >= 0) {
      m.beg = __ldg(a.ptr + c);
      m.end = __ldg(a.ptr + c + 1);
      if (gl == 0) {
        m.xc = a.x[c];
        m.nrm = __ldg(a.norm + c);
        if (FORM == SCD_DUAL) m.yc = __ldg(a.y + c);
      }
    }
  };
  auto load_idx = [&](Batch &q, const Meta &m) {
    q.c = m.c;
    q.xc = m.xc;
    q.nrm = m.nrm;
    q.yc = m.yc;
    q.valid = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int64_t k = m.beg + (int64_t)e * G + gl;
      q.id[e] = 0;
      q.v[e] = 0.f;
      if (k < m.end) {
        q.id[e] = __ldcs(h.idx + k);
        q.v[e] = IMP ? 1.f : val_cs(a.val, k);
        q.valid |= 1u << e;
      }
    }
  };
  Batch cur, nxt;
  Meta m1;
  int64_t cn = take();
  bool more = cn != -2;  // warp-uniform: the warp holds a batch
  if (more) {
    load_meta(m1, cn);
    load_idx(cur, m1);
    if (TP) tail_prefetch(cur);
  }
  for (;;) {
    for (int it = 0; it < h.F && more; ++it) {
      // next batch: coordinates (ticket taken one batch ago) + offsets + entries (no shared-vector access)
      cn = take();
      const bool have_next = cn != -2;
      if (have_next) {
        load_meta(m1, cn);
        load_idx(nxt, m1);
      }
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
            w[e] = (HP ? cur.tw[e] : (HC ? __ldcg(h.hc + sl) : ld_sv(a.sv + s_hid[sl]))) + s_pend[sl];
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
        // tail entries: predicated REDs (no per-entry branch); hot entries: shared-memory adds
#pragma unroll
        for (int e = 0; e < E; ++e) red_if(a.sv + cur.id[e], cur.v[e] * d, (cur.valid >> e & 1) && cur.id[e] >= 0);
#pragma unroll
        for (int e = 0; e < E; ++e)
          if ((cur.valid >> e & 1) && cur.id[e] < 0) atomicAdd(s_pend + (cur.id[e] & 0x7fffffff), cur.v[e] * d);
      }
      more = have_next;
      if (have_next) {
        cur = nxt;
        if (TP) tail_prefetch(cur);  // the next batch's tail values, one step early
      }
    }
    const bool any = __syncthreads_or(more);
    for (int i = threadIdx.x; i < h.K; i += blockDim.x) {  // flush
      const float p = s_pend[i];
      const int32_t j = s_hid[i];
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

// the epoch's block permutation of a block-ordered bin, materialised once per bin and epoch (the Feistel
// evaluation was ~15% of the hot-set kernel's instructions: profiles/c5_shape_r2.txt)
__global__ void k_block_perm(Perm p, int64_t nf, int32_t *out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)perm_apply(p, (uint64_t)i);
}

// the epoch order of a bin in block order (reading c28), through bin_coord itself (identity list)
__global__ void k_block_order_export(BinArgs b, int64_t n, int64_t *out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = bin_coord(b, (uint64_t)t);
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

// ----------------------------------------------------------------------------------------------
// Heavy coordinates with their slices staged in shared memory by the bulk-copy engine (north_star
// "(c)": TMA staging of long columns; C4's cluster bin: 10 385 columns of 16k-350k entries, 44% of
// the entries).  Every CTA of the cluster owns one contiguous slice of the coordinate; its thread 0
// issues one cp.async.bulk per array (idx, val) for the first CAP entries of the slice of the NEXT
// coordinate into the other buffer of a double buffer (mbarrier with transaction count), so the
// entries arrive while the current coordinate is computed; the dot and the scatter then read shared
// memory (the rest of a slice longer than CAP streams from global as in k_epoch_cluster).  The next
// coordinate is known one iteration early: CTA 0 takes its ticket while the current one is reduced
// and publishes it with the delta.  Three cluster barriers per coordinate (previous scatter done,
// partials, delta), as in k_epoch_cluster.
struct Slice {
  int64_t beg, end;  // the CTA's entries [beg, end) of the coordinate
  int64_t st;        // entries [beg, beg + st) are staged in shared memory, from offset off of the buffer
  int off;
};

template <int CL, int CAP>
__device__ __forceinline__ Slice cluster_slice(const EpochArgs &a, int64_t c, unsigned r) {
  Slice q;
  const int64_t b0 = __ldg(a.ptr + c), e0 = __ldg(a.ptr + c + 1);
  const int64_t len = (e0 - b0 + CL - 1) / CL;
  q.beg = min(e0, b0 + (int64_t)r * len);
  q.end = min(e0, q.beg + len);
  const int64_t a0 = q.beg & ~(int64_t)3;                        // 16-byte aligned copy start
  int64_t a1 = (min(q.end, q.beg + (int64_t)CAP) + 3) & ~(int64_t)3;  // 16-byte aligned copy end
  if (a1 > (a.nnz & ~(int64_t)3)) a1 = a.nnz & ~(int64_t)3;      // never read past the arrays
  q.off = (int)(q.beg - a0);
  const int64_t st = min(min(q.end, q.beg + (int64_t)CAP), a1) - q.beg;
  q.st = st > 0 ? st : 0;
  return q;
}

template <int FORM, int CL, int T, int CAP>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(T) k_epoch_cluster_tma(EpochArgs a, BinArgs b) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int NW = T / 32;
  constexpr int BUF = CAP + 4;  // staged entries + alignment slack
  extern __shared__ float4 s_dyn[];
  int32_t *s_idx = reinterpret_cast<int32_t *>(s_dyn);  // [2][BUF]
  float *s_val = reinterpret_cast<float *>(s_idx + 2 * BUF);  // [2][BUF]
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ float s_red[NW];
  __shared__ float s_part[CL];
  __shared__ float s_delta;
  __shared__ unsigned int s_tk[2];  // CTA 0: the tickets of the current and the next coordinate
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned r = cluster.block_rank();
  float *part0 = cluster.map_shared_rank(s_part, 0);
  float *delta0 = cluster.map_shared_rank(&s_delta, 0);
  unsigned *tk0 = cluster.map_shared_rank(s_tk, 0);
  const bool implicit = a.val == nullptr;
  auto issue = [&](int buf, const Slice &q) {  // thread 0: bulk copies of the staged part of a slice
    const int64_t a0 = q.beg - q.off;
    const unsigned n = (unsigned)((q.off + q.st + 3) & ~3);
    if (q.st <= 0) {
      mbar_expect_tx(&s_bar[buf], 0);
      return;
    }
    mbar_expect_tx(&s_bar[buf], n * 4u * (implicit ? 1u : 2u));
    bulk_g2s(s_idx + buf * BUF, a.idx + a0, n * 4u, &s_bar[buf]);
    if (!implicit) bulk_g2s(s_val + buf * BUF, a.val + a0, n * 4u, &s_bar[buf]);
  };
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (r == 0) {
      s_tk[0] = atomicAdd(b.counter, 1u);
      s_tk[1] = atomicAdd(b.counter, 1u);
    }
  }
  cluster.sync();
  int64_t t_cur = b.lo + (int64_t)tk0[0], t_nxt = b.lo + (int64_t)tk0[1];
  Slice cur{}, nxt{};
  int64_t c_cur = -1, c_nxt = -1;
  if (t_cur < b.hi) {
    c_cur = bin_coord(b, t_cur);
    cur = cluster_slice<CL, CAP>(a, c_cur, r);
    if (tid == 0) issue(0, cur);
  }
  unsigned phase[2] = {0u, 0u};
  int buf = 0;
  for (;;) {
    if (t_cur >= b.hi) break;  // cluster-uniform: every CTA read the same tickets
    // every CTA of the cluster has finished scattering the previous coordinate before any gathers this
    // one (else the previous coordinate would still be in flight: one more per cluster than the bin's
    // cap; measured: C2 primal per-epoch gap 2x the sequential envelope at epoch 3 instead of 1.5x), and
    // this CTA no longer reads the other buffer
    cluster.sync();
    if (t_nxt < b.hi) {
      c_nxt = bin_coord(b, t_nxt);
      nxt = cluster_slice<CL, CAP>(a, c_nxt, r);
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(buf ^ 1, nxt);
      }
    }
    mbar_wait(&s_bar[buf], phase[buf]);
    phase[buf] ^= 1u;
    const int32_t *bi = s_idx + buf * BUF + cur.off;
    const float *bv = s_val + buf * BUF + cur.off;
    float acc = 0.f;
#pragma unroll 8
    for (int64_t k = tid; k < cur.st; k += T) acc = fmaf(ld_sv(a.svg + bi[k]), implicit ? 1.f : bv[k], acc);
    acc += dot_strided<8>(a.svg, a.idx, a.val, cur.beg + cur.st + tid, cur.end, T);
    acc = warp_sum(acc);
    if (lane == 0) s_red[wid] = acc;
    __syncthreads();
    if (wid == 0) {
      float sp = lane < NW ? s_red[lane] : 0.f;
      sp = warp_sum(sp);
      if (lane == 0) part0[r] = sp;
    }
    cluster.sync();  // partials in CTA 0
    if (r == 0 && tid == 0) {
      float sum = 0.f;
      for (int i = 0; i < CL; ++i) sum += s_part[i];
      const float xc = a.x[c_cur];
      const float d = coord_delta<FORM>(sum, xc, __ldg(a.norm + c_cur), FORM == SCD_DUAL ? __ldg(a.y + c_cur) : 0.f,
                                        a.lam, a.lamN);
      if (!b.dry) a.x[c_cur] = xc + d;
      s_delta = b.dry ? 0.f : d;
      s_tk[0] = s_tk[1];  // every CTA read both tickets before the barrier above
      s_tk[1] = t_nxt < b.hi ? atomicAdd(b.counter, 1u) : 0xFFFFFFFFu;
    }
    cluster.sync();  // delta and the next ticket published
    const float d = scatter_scale<FORM>(*delta0);
    const unsigned tk_new = tk0[1];
    if (d != 0.f || b.dry) {
#pragma unroll 8
      for (int64_t k = tid; k < cur.st; k += T) red_add(a.sv + bi[k], (implicit ? 1.f : bv[k]) * d);
      scatter_strided<8>(a.sv, a.idx, a.val, cur.beg + cur.st + tid, cur.end, T, d);
    }
    t_cur = t_nxt;
    c_cur = c_nxt;
    cur = nxt;
    t_nxt = tk_new == 0xFFFFFFFFu ? b.hi : b.lo + (int64_t)tk_new;
    buf ^= 1;
  }
  cluster.sync();  // nobody leaves while another CTA may still read CTA 0's shared memory
}

// kernel table ---------------------------------------------------------------------------------
constexpr int kCtaT = kLanesCta, kCtaE = 16;
// SM-shared head kernel (default shape): row groups per SM, threads per group, entries per staged chunk.
// 6 x 128 x 1024: 6.99 ms per C3 epoch; 4 x 256 x 2048 (SCD_SM_GRP=4): 7.7 ms, with a per-epoch rate
// ~20% better at tight gaps; 8 x 128 x 1024 (SCD_SM_GRP=8): 6.99 ms (profiles/r2/sm_groups_r2.txt)
constexpr int kSmG = 6, kSmT = 128, kSmC = 1024;
constexpr int kGrpE8 = 8, kGrpE32 = 16;
constexpr int kClE = 8;
constexpr int kCombT = 128, kCombS = 2048;  // CTA-combining kernel for 8-lane bins

// threads per CTA of the plain CTA-bin kernel: 128 (C4: 10.48 -> 10.0 ms per epoch, the per-epoch gaps
// within run-to-run noise, profiles/r2/c4_cta_threads_r2.txt); SCD_CTA_T = 256 restores the round-1 shape
int cta_threads() {
  static const int t = getenv("SCD_CTA_T") && atoi(getenv("SCD_CTA_T")) == 256 ? kCtaT : 128;
  return t;
}

template <int FORM>
void *kernel_for(int lanes, int plain) {
  switch (lanes) {
    case 8:
      // CTA-combining by default; the plain 8-lane kernel when the bin's cap is below one CTA's batch
      return plain ? (void *)k_epoch_group<FORM, 8, kGrpE8> : (void *)k_epoch_group_comb<FORM, 8, kCombT, kCombS>;
    case 32: return (void *)k_epoch_group<FORM, 32, kGrpE32>;
    case kLanesCluster: return nullptr;  // cluster_kernel()
    default: return cta_threads() == 128 ? (void *)k_epoch_cta<FORM, 128, kCtaE> : (void *)k_epoch_cta<FORM, kCtaT, kCtaE>;
  }
}

// options.wild: the plain kernel of each bin with the non-atomic scatter (PASSCoDe-Wild comparison)
template <int FORM>
void *kernel_wild(int lanes) {
  switch (lanes) {
    case 8: return (void *)k_epoch_group<FORM, 8, kGrpE8, true>;
    case 32: return (void *)k_epoch_group<FORM, 32, kGrpE32, true>;
    case kLanesCluster: return nullptr;
    default: return cta_threads() == 128 ? (void *)k_epoch_cta<FORM, 128, kCtaE, true> : (void *)k_epoch_cta<FORM, kCtaT, kCtaE, true>;
  }
}

constexpr int kClusterCap = 6144;  // staged entries per CTA slice (TMA cluster kernel): 2 x 48 KB double buffer

template <int FORM, bool WILD>
void *cluster_kernel(bool tma) {
  if (tma && !WILD) return (void *)k_epoch_cluster_tma<FORM, kClusterCtas, kClusterThreads, kClusterCap>;
  return (void *)k_epoch_cluster<FORM, kClusterCtas, kClusterThreads, kClE, WILD>;
}

// The TMA-staged cluster kernel is opt-in (SCD_CLUSTER_TMA=1): measured no faster than the register-tile
// kernel (0.52-0.57 vs 0.515 ms per C4 slice launch, profiles/c4_cluster_tma_r2.txt: the bin is bound by
// the L2 rate of gathers and REDs on the same residual lines).  It needs 16-byte aligned idx / val arrays.
bool cluster_tma_ok(const scd_ctx *c) {
  static const bool on = getenv("SCD_CLUSTER_TMA") && atoi(getenv("SCD_CLUSTER_TMA")) == 1;
  return on && ((uintptr_t)c->idx % 16) == 0 && ((uintptr_t)c->val % 16) == 0 && !c->opt.wild;
}

size_t cluster_smem(const scd_ctx *c) {
  return cluster_tma_ok(c) ? sizeof(int32_t) * 2 * 2 * (size_t)(kClusterCap + 4) : 0;
}

template <int FORM, int E, bool IMP>
void *hot_kernel_fast() {
  return (void *)k_epoch_group_hot<FORM, 8, E, true, true, true, IMP, 512>;
}

template <int FORM>
void *hot_kernel(const scd_ctx *c, const Bin &b) {
  const bool hc = c->hot_copy > 0, tp = c->hot_tp;
  if (hc && tp) {  // the default: early hot gathers from the copy; specialised on row length and values
    const bool imp = c->val == nullptr, e5 = b.maxlen <= 40;
    if (e5) return imp ? hot_kernel_fast<FORM, 5, true>() : hot_kernel_fast<FORM, 5, false>();
    return imp ? hot_kernel_fast<FORM, 8, true>() : hot_kernel_fast<FORM, 8, false>();
  }
  if (hc) return (void *)k_epoch_group_hot<FORM, 8, 8, true, false, false>;
  if (tp) return (void *)k_epoch_group_hot<FORM, 8, 8, false, true, false>;
  return (void *)k_epoch_group_hot<FORM, 8, 8, false, false, false>;
}

void *bin_kernel(const scd_ctx *c, const Bin &b) {
  if (b.hot > 0 && b.lanes == 8 && !c->opt.wild)
    return c->form == SCD_PRIMAL ? hot_kernel<SCD_PRIMAL>(c, b) : hot_kernel<SCD_DUAL>(c, b);
  if (b.lanes == kLanesCluster) {
    const bool tma = cluster_tma_ok(c);
    if (c->form == SCD_PRIMAL)
      return c->opt.wild ? cluster_kernel<SCD_PRIMAL, true>(false) : cluster_kernel<SCD_PRIMAL, false>(tma);
    return c->opt.wild ? cluster_kernel<SCD_DUAL, true>(false) : cluster_kernel<SCD_DUAL, false>(tma);
  }
  if (c->opt.wild) return c->form == SCD_PRIMAL ? kernel_wild<SCD_PRIMAL>(b.lanes) : kernel_wild<SCD_DUAL>(b.lanes);
  if (b.head > 0 && b.lanes == kLanesCta && b.sm && c->form == SCD_DUAL && c->tail_snap)
    return b.sm == 4 ? (void *)k_epoch_sm_tma<SCD_DUAL, 4, 256, 2048>
                     : (b.sm == 8 ? (void *)k_epoch_sm_tma<SCD_DUAL, 8, kSmT, kSmC> : (void *)k_epoch_sm_tma<SCD_DUAL, kSmG, kSmT, kSmC>);
  if (b.head > 0 && b.lanes == kLanesCta) {
    // the read copies exist only for the dual (setup_tail_snap); the head copy needs the rolling tail copy
    if (c->form == SCD_DUAL && c->tail_snap && c->head_copy > 0)
      return (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, 1, true>;
    if (c->form == SCD_DUAL && c->tail_snap) return (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, 1, false>;
    return c->form == SCD_PRIMAL ? (void *)k_epoch_cta_head<SCD_PRIMAL, kCtaT, kCtaE, 0, false>
                                 : (void *)k_epoch_cta_head<SCD_DUAL, kCtaT, kCtaE, 0, false>;
  }
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
  a.nnz = c->nnz;
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
// fits the budget.
void hot_launch_shape(scd_ctx *c, Bin &b) {
  // the 768-thread kernel exists only in the default (hot copy + early gathers) configuration
  // one 512-thread CTA per SM, 64 rows in flight per CTA (profiles/c5_shape_r2.txt: 768 threads are ~5%
  // faster only with a combined-update budget of 1.25 τ, 16 lanes per row at 1024 threads 30% slower)
  constexpr int T = 512;
  b.block = T;
  const size_t smem = 8 * (size_t)b.hot;
  const int64_t rows = T / 8;
  int occ = 1;
  {
    void *fn = bin_kernel(c, b);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, T, smem);
    if (occ < 1) occ = 1;
  }
  const int64_t need = (b.count + rows - 1) / rows;
  int64_t grid = std::min<int64_t>((int64_t)c->nsm * occ, std::max<int64_t>(need, 1));
  // lower the grid (whole CTAs per SM, not below one per SM) until a window of 6 batches fits
  while (combine_window(c, b, grid * rows, 1) < 6 && grid > (int64_t)c->nsm) grid -= c->nsm;
  const int64_t F = std::max<int64_t>(1, std::min<int64_t>(64, combine_window(c, b, grid * rows, 1)));
  if (F < 4) {  // too short a window to beat the CTA-combining kernel: use that instead
    b.hot = 0;
    bin_launch_shape(c, b);
    return;
  }
  b.grid = (int)std::max<int64_t>(grid, 1);
  b.block = T;
  b.flush = (int)F;
  // Hot copy: the copy's age, P · K/32 warp tickets of rows/warp rows each, joins the window budget:
  // rows in flight · (1 + F + hp) + age <= budget, hp = 1 when the hot values are also gathered one
  // step early (with the early tail gathers, hot_tp); F gives way (down to 4) until P >= 8 fits.
  c->hot_copy = 0;
  const double budget = combine_budget(c, b);
  const int64_t inflight = (int64_t)b.grid * rows, nch = (b.hot + 31) / 32, cpw = 32 / 8;
  const double hp = c->hot_tp ? 1.0 : 0.0;
  int64_t P = 0, f = F;
  for (; f >= 4; --f) {
    P = (int64_t)((budget - (double)inflight * (1.0 + hp + f)) / (double)(nch * cpw));
    if (P >= 8) break;
  }
  if (P >= 8) {
    if (!c->hot_hc && cudaMalloc((void **)&c->hot_hc, sizeof(float) * (size_t)b.hot) != cudaSuccess) {
      cudaGetLastError();
      c->hot_hc = nullptr;
      return;
    }
    int64_t p2 = 1;  // a power of two (the take() test is a mask): the copy's age only shrinks
    while (p2 * 2 <= P) p2 *= 2;
    c->hot_copy = p2;
    b.flush = (int)f;
  }
  // the early hot gathers read the copy: without it the kernel reads the hot values in their turn
  c->hot_hp = c->hot_copy > 0 && c->hot_tp;
}

// Grid/block for a bin (used by build_schedule): persistent, sized to the SM count times the
// kernel's residency, capped by max_inflight coordinates in flight.
void bin_launch_shape(scd_ctx *c, Bin &b) {
  // A cap below a kernel's minimum batch must still be honoured (staleness): the
  // combining kernel runs kCombT/8 coordinates per CTA, the 8-lane kernel >= 4 per warp, so small
  // caps fall back to the plain 8-lane kernel, and caps below 4 to one warp per coordinate.
  if (b.lanes == 8 && b.cap > 0 && b.cap < kCombT / 8) b.plain = 1;
  if (b.lanes == 8 && b.cap > 0 && b.cap < 4) b.lanes = 32;
  if (c->opt.wild) {  // plain kernels only (no head / CTA combining)
    b.plain = 1;
    b.head = 0;
  }
  if (b.lanes != kLanesCta) b.head = 0;
  if (b.lanes == kLanesCluster) b.cl = kClusterCtas;
  if (b.hot > 0 && (b.lanes != 8 || c->opt.wild)) b.hot = 0;
  if (b.hot > 0) {
    hot_launch_shape(c, b);
    return;
  }
  void *fn = bin_kernel(c, b);
  const bool group = (b.lanes <= 32);
  const bool clus = (b.lanes == kLanesCluster);
  const bool comb = (b.lanes == 8 && !b.plain);  // fixed CTA size (kernel template)
  int block = comb ? kCombT : (group ? 256 : (clus ? kClusterThreads : (b.head > 0 ? kCtaT : cta_threads())));
  // sub-warp bins with a small cap shrink the CTA so the cap can be honoured (>= one warp)
  if (group && !comb && b.cap > 0 && b.cap * b.lanes < block) {
    block = (int)(((b.cap * b.lanes) + 31) / 32 * 32);
    if (block < 32) block = 32;
  }
  const size_t smem = b.head > 0 ? sizeof(float) * (size_t)b.head : (clus ? cluster_smem(c) : 0);
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
    // of the grid coordinates in flight: grid * (1 + flush) <= combined-update budget (reading c25)
    int64_t f = std::min<int64_t>(64, combine_window(c, b, b.grid, 1));
    if (f < 2) {  // no combining possible within the budget: plain CTA kernel
      b.head = 0;
      b.flush = 0;
      bin_launch_shape(c, b);
      return;
    }
    b.flush = (int)f;
  }
}

// Dynamic shared memory of a bin's kernel.
size_t bin_smem(const scd_ctx *c, const Bin &b) {
  if (b.hot > 0) return 8 * (size_t)b.hot;
  if (b.head > 0 && b.sm == 4) return 2 * sizeof(float) * (size_t)b.head + 4 * sizeof(GroupSmem<2048, 8>);
  if (b.head > 0 && b.sm) return 2 * sizeof(float) * (size_t)b.head + b.sm * sizeof(GroupSmem<kSmC, kSmT / 32>);
  if (b.head > 0) return sizeof(float) * (size_t)b.head;
  return b.lanes == kLanesCluster ? cluster_smem(c) : 0;
}

// SM-shared head kernel (k_epoch_sm_tma) for the single head bin of a dual with the rolling tail copy
// (build_schedule): one CTA of G row groups per SM (kSmG by default, SCD_SM_GRP = 4 | 8).  Its head staleness (reading c25): rows in flight
// (nsm·G) + 2·nsm·Q (the other SMs' pending head and what they flushed since a chunk's snapshot, Q rows
// of each, Q = nh/ch·rh the rows between two refreshes of a chunk) <= the combined-update budget.  ch is
// the smallest chunk count per flushing row that fits, then rh the largest period (<= 8).  The kernel's
// head is the bin's head (the tail copy starts there).  SCD_SM_HEAD=0 keeps k_epoch_cta_head.
// Returns false when it does not fit (then k_epoch_cta_head runs).
bool sm_head_shape(scd_ctx *c, Bin &b) {
  b.sm = 0;
  const char *e = getenv("SCD_SM_HEAD");
  if ((e && atoi(e) == 0) || b.head <= 0 || b.lanes != kLanesCta || c->form != SCD_DUAL) return false;
  const int G = getenv("SCD_SM_GRP") ? atoi(getenv("SCD_SM_GRP")) : kSmG, T = G == 4 ? 256 : kSmT;
  if (G != kSmG && G != 4 && G != 8) return false;
  const int CH = 4 * T;
  if (b.head % CH != 0) return false;
  const int64_t inflight = (int64_t)c->nsm * G;
  if (b.cap > 0 && inflight > b.cap) return false;
  const double budget = combine_budget(c, b);
  const int nh = b.head / CH;
  auto fits = [&](double q) { return (double)inflight + 2.0 * (double)c->nsm * q <= budget; };
  int ch = 0, rh = 1;
  for (int k = 1; k <= nh; k *= 2)
    if (fits((double)((nh + k - 1) / k))) {
      ch = k;
      break;
    }
  if (ch == 0) return false;
  if (ch == 1)
    while (rh < 8 && fits((double)nh * (rh + 1))) ++rh;
  b.sm = G;
  b.sm_ch = ch;
  b.sm_rh = rh;
  void *fn = bin_kernel(c, b);
  const size_t smem = bin_smem(c, b);
  int occ = 0;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, G * T, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    b.sm = 0;
    return false;
  }
  b.grid = c->nsm;
  b.block = G * T;
  b.flush = 0;
  return true;
}

int sm_chunk_entries(int groups) { return groups == 4 ? 2048 : kSmC; }

// Launch one bin's kernel over the permutation positions [ba.lo, ba.hi) with `grid` CTAs.
scd_status launch_bin(scd_ctx *c, const Bin &b, EpochArgs &a, BinArgs &ba, int64_t grid, cudaStream_t s) {
  void *fn = bin_kernel(c, b);
  int H = b.head, F = b.flush;
  void *args_head[] = {&a, &ba, &H, &F};
  HotArgs ha;
  void *args_hot[] = {&a, &ba, &ha};
  SmHeadArgs sh{b.head, b.sm_ch, b.sm_rh};
  void *args_sm[] = {&a, &ba, &sh};
  void **args = b.sm ? args_sm : args_head;
  if (b.hot > 0 && b.lanes == 8 && !c->opt.wild) {
    ha.idx = c->hot_idx;
    ha.hot_ids = c->hot_ids;
    ha.K = b.hot;
    ha.F = b.flush;
    ha.hc = c->hot_hc;
    ha.P = (int)std::max<int64_t>(1, c->hot_copy);
    args = args_hot;
  }
  const size_t smem = bin_smem(c, b);
  if (smem >= 48 * 1024) SCD_CK(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
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
      ba.blk = b.blk;
      ba.blk_shift = b.blk_shift;
      ba.bperm = nullptr;
      ba.zero = 0;
      ba.perm = make_perm(c->opt.seed, epoch, b.stream_id, b.blk > 1 ? b.count / b.blk : b.count);
      if (b.blk > 1 && b.bperm && ba.perm.n > 0) {
        if (sl == 0) {  // once per epoch and bin (every slice uses the same permutation)
          k_block_perm<<<grid_for((int64_t)ba.perm.n, 256), 256, 0, s>>>(ba.perm, (int64_t)ba.perm.n, b.bperm);
          SCD_CKL(c, "k_block_perm launch");
          ++c->launches;
        }
        ba.bperm = b.bperm;
      }
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
  const int cpc = b.lanes <= 32 ? b.block / b.lanes : (b.sm ? b.sm : 1);
  const int64_t probe = std::min<int64_t>(b.count, (int64_t)b.grid * cpc * 8);  // ~0.14 ms per C3 probe launch
  SCD_CK(c, cudaMemsetAsync(c->sv_base, 0, sizeof(float) * (size_t)(c->n_shared + kMaxSvOffsetFloats), s));
  // all probe launches enqueued back to back between events (one warm-up, then kReps per candidate
  // in round-robin order so slow drifts hit every candidate alike); one synchronisation at the end
  constexpr int kReps = 2;
  const int nl = 1 + kSvCandidates * kReps;
  std::vector<cudaEvent_t> ev(nl + 1);
  for (auto &e : ev) SCD_CK(c, cudaEventCreate(&e));
  SCD_CK(c, cudaMemsetAsync(c->counters, 0, sizeof(unsigned int) * kMaxBins * kMaxSlices, s));
  SCD_CK(c, cudaEventRecord(ev[0], s));
  for (int l = 0; l < nl; ++l) {
    const int ci = l == 0 ? 0 : (l - 1) % kSvCandidates;
    c->sv = c->sv_base + kSvCandidateBytes[ci] / 4;
    EpochArgs a = make_args(c);
    BinArgs ba;
    ba.list = b.list;
    ba.lo = 0;
    ba.hi = probe;
    ba.blk = b.blk;
    ba.blk_shift = b.blk_shift;
    ba.bperm = nullptr;  // the probe's permutation differs from the epochs': evaluated inline
    ba.zero = 0;
    ba.perm = make_perm(c->opt.seed ^ 0x5052424Full, 0xFFFFFFFEu, b.stream_id, b.blk > 1 ? b.count / b.blk : b.count);
    ba.dry = 1;
    ba.counter = c->counters + l % (kMaxBins * kMaxSlices);
    if (l > 0 && l % (kMaxBins * kMaxSlices) == 0)
      SCD_CK(c, cudaMemsetAsync(c->counters, 0, sizeof(unsigned int) * kMaxBins * kMaxSlices, s));
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
  SCD_CK(c, cudaMemsetAsync(c->counters, 0, sizeof(unsigned int) * kMaxBins * kMaxSlices, s));
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

scd_status launch_block_order_export(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n, int64_t blk,
                                     int64_t *d_out, cudaStream_t s) {
  BinArgs b{};
  b.list = nullptr;
  b.lo = 0;
  b.hi = n;
  b.blk = blk;
  b.blk_shift = 0;
  while ((1ll << (b.blk_shift + 1)) <= blk) ++b.blk_shift;
  b.bperm = nullptr;
  b.perm = make_perm(seed, epoch, stream, blk > 1 ? n / blk : n);
  k_block_order_export<<<grid_for(n, 256), 256, 0, s>>>(b, n, d_out);
  return cudaGetLastError() == cudaSuccess ? SCD_OK : SCD_E_CUDA;
}

scd_status launch_partition_export(uint64_t seed, int64_t count, int32_t k, int32_t *d_owner, cudaStream_t s) {
  Perm p = make_perm(seed, 0u, kPartStream, count);
  k_partition_export<<<grid_for(count, 256), 256, 0, s>>>(p, count, k, d_owner);
  return cudaGetLastError() == cudaSuccess ? SCD_OK : SCD_E_CUDA;
}

}  // namespace scd
