// common.cuh — internal declarations of libscd (B200 TPA-SCD).  Not part of the ABI.
// P:n = PAPER.md line n.  Readings cN = DESIGN.md §4.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "scd.h"

namespace scd {

constexpr int kMaxBins = 4;
constexpr int kMaxSlices = 64;
// shared-vector placement candidates (bytes into its allocation), epoch.cu tune_shared_layout
constexpr int kSvCandidates = 18;
constexpr int64_t kSvCandidateBytes[kSvCandidates] = {0,     4096,  8192,  12288, 16384, 20480,  24576,  28672, 32768,
                                                      36864, 40960, 45056, 49152, 53248, 57344, 61440, 131072, 262144};
constexpr int64_t kMaxSvOffsetFloats = 262144 / 4;
constexpr uint32_t kPartStream = 0x50415254u;  // "PART": partition permutation stream (c15)

// ------------------------------------------------------------------------------------------
// Keyed Feistel permutation P_(seed,epoch,stream) on [0, n) (Alg. 1 "Generate random
// permutation" P:144 / Alg. 2; generator fixed by reading c8).  4-round balanced Feistel
// on [0, 4^h), h = ceil(ceil(log2 n)/2), with cycle-walking into [0, n): a bijection computed
// inline per coordinate (no permutation array is stored or read).
// ------------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

struct Perm {
  uint64_t k0, k1, k2, k3;  // round keys
  uint64_t n;
  uint64_t mask;
  int h;
};

inline Perm make_perm(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n) {
  Perm p;
  uint64_t key = mix64(seed ^ mix64(((uint64_t)epoch << 32) | (uint64_t)stream));
  p.k0 = mix64(key + 0);
  p.k1 = mix64(key + 1);
  p.k2 = mix64(key + 2);
  p.k3 = mix64(key + 3);
  p.n = (uint64_t)(n > 0 ? n : 0);
  int bits = 0;
  uint64_t v = (n >= 2) ? (uint64_t)(n - 1) : 0;
  while (v) { ++bits; v >>= 1; }
  p.h = (bits + 1) / 2;
  p.mask = (p.h >= 32) ? 0xFFFFFFFFull : ((1ull << p.h) - 1ull);
  return p;
}

__device__ __forceinline__ uint64_t feistel_round(uint64_t x, const Perm &p) {
  uint64_t L = x >> p.h, R = x & p.mask, t;
  t = L ^ (mix64(R ^ p.k0) & p.mask); L = R; R = t;
  t = L ^ (mix64(R ^ p.k1) & p.mask); L = R; R = t;
  t = L ^ (mix64(R ^ p.k2) & p.mask); L = R; R = t;
  t = L ^ (mix64(R ^ p.k3) & p.mask); L = R; R = t;
  return (L << p.h) | R;
}

__device__ __forceinline__ uint64_t perm_apply(const Perm &p, uint64_t j) {
  if (p.n <= 1) return 0;
  uint64_t x = j;
  do { x = feistel_round(x, p); } while (x >= p.n);
  return x;
}

// ------------------------------------------------------------------------------------------
// Context
// ------------------------------------------------------------------------------------------
constexpr int kLanesCta = 256;       // bin kind: one CTA of 256 threads per coordinate
constexpr int kClusterCtas = 8;      // largest cluster size used (portable); the bin's `cl` picks 2, 4 or 8
constexpr int kClusterThreads = 512;
constexpr int kLanesCluster = kClusterCtas * kClusterThreads;  // bin kind: one 8-CTA cluster per coordinate

struct Bin {
  int lanes = 0;             // lanes per coordinate: 8 / 32 (sub-warp group), 256 (CTA), 4096 (cluster)
  double tau = 0.0;          // estimated staleness bound of the bin (coordinates in flight)
  double tau_tail = 0.0;     // head bin: bound of the coupling through the tail entries alone (0 = not estimated)
  int64_t cap = 0;           // coordinates in flight allowed
  int plain = 0;             // 1 = plain sub-warp kernel (cap below the combining kernel's CTA batch)
  int head = 0;              // CTA bins: > 0 = head-combining kernel over sv[0, head) (k_epoch_cta_head)
  int flush = 0;             // head kernel: coordinates per CTA between flushes of the pending head
  int cl = kClusterCtas;     // cluster bin: CTAs per cluster (one coordinate per cluster)
  int hot = 0;               // 8-lane bin: > 0 = hot-set kernel with this many hot slots (hot.cu)
  int sm = 0;                // CTA head bin: G > 0 = SM-shared head kernel (k_epoch_sm_tma, one CTA of G row groups per SM)
  int sm_ch = 0;             // SM kernel: head chunks flushed per flushing row
  int sm_rh = 1;             // SM kernel: rows per flushing row
  int snap = 0;              // 1 = every slice launch gathers from a copy of the shared vector taken just
                             // before it (the whole slice within the bin's staleness cap)
  int64_t count = 0, nnz = 0;
  int64_t maxlen = 0;        // longest coordinate of the bin (stored entries)
  int32_t *list = nullptr;   // device, coordinate ids ascending
  int grid = 0, block = 0;
  uint32_t stream_id = 0;    // permutation stream = 1 + bin index
  int64_t blk = 0;           // > 1: the epoch visits blocks of blk consecutive coordinates (reading c28)
  int blk_shift = 0;         // log2(blk)
  int32_t *bperm = nullptr;  // device [count / blk]: the epoch's block permutation (k_block_perm)
  double ms = 0.0;           // profiling accumulator
  int64_t prof_launches = 0;
};

}  // namespace scd

struct scd_ctx {
  scd_form form;
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  int64_t n_coord = 0, n_shared = 0;
  double lam = 0, lamN = 0;
  int64_t n_global = 0;
  scd_options opt{};
  int device = 0, nsm = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // matrix (device) — borrowed or owned
  const int64_t *ptr = nullptr;
  const int32_t *idx = nullptr;
  const float *val = nullptr;
  void *own_ptr = nullptr, *own_idx = nullptr, *own_val = nullptr;
  const float *y = nullptr;  // labels [n_rows]
  void *own_y = nullptr;
  // model and shared vector (fp32) plus aggregation base point snapshots
  float *x = nullptr, *x0 = nullptr;    // β (primal) / α (dual)  [n_coord]
  float *sv = nullptr, *sv0 = nullptr;  // r = y - Aβ (primal) / w̄ = Aᵀα (dual)  [n_shared]
  float *sv_base = nullptr;             // allocation holding sv (sv may sit at an offset in it)
  int64_t sv_offset_bytes = 0;          // chosen placement of sv in sv_base
  int n_probe = 0;                      // placement probe times (ms) per candidate
  float probe_ms[32] = {0};
  float *norm = nullptr;                // ||a_m||² / ||ā_n||²  [n_coord]
  // asynchronous schedule
  int n_bins = 0;
  scd::Bin bins[scd::kMaxBins];
  int32_t *empty_list = nullptr;
  int64_t n_empty = 0, n_nonempty = 0;
  bool empty_dirty = true;
  int n_slices = 1;                  // bins are interleaved in n_slices slices per epoch
  unsigned int *counters = nullptr;  // [kMaxSlices * kMaxBins] ticket counters
  // scratch
  double *acc = nullptr;    // [32] fp64 accumulators (objective / gap / gamma)
  double *vec64 = nullptr;  // [n_shared] fp64 (u = Aβ or v = Aᵀα)
  float *comm = nullptr;    // [n_shared] fp32 aggregation buffer (Δ of the shared vector)
  ncclComm_t nccl = nullptr;
  const scd_collectives *coll = nullptr;  // host-side transport hooks (scd_options.collectives), instead of NCCL
  bool has_comm() const { return nccl != nullptr || coll != nullptr; }
  uint64_t model_version = 1;         // bumped by every change of the model (epoch, aggregation, set_model)
  uint64_t vec64_version = 0;         // model_version vec64 = A x (fp64, all-reduced) was computed for
  uint32_t rounds_done = 0;           // aggregation rounds (recompute_every with world > 1)
  int p2p_state = 0;                  // fused peer-memory aggregation: 0 = not set up, 1 = ready, -1 = unavailable
  float **p2p_ptrs = nullptr;         // device [2 * world]: every rank's sv, then every rank's sv0
  std::vector<void *> p2p_open;       // IPC mappings to close at destroy
  // profiling
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_pending;
  int64_t launches = 0;
  uint32_t epochs_done = 0;
  double tau_star = 0.0;   // smallest estimated staleness bound over the bins (layout.cu)
  int32_t *hot_idx = nullptr;         // device [nnz]: re-encoded indices for the hot-set kernel (hot.cu)
  int32_t *hot_ids = nullptr;         // device [K]: shared-vector index of each hot slot
  bool hot_hp = false;                // hot-set kernel also gathers the next batch's hot values (from the copy) early
  bool hot_tp = false;                // hot-set kernel gathers the next batch's tail values one step early
  double hot_tail_tau = 0.0;          // staleness bound of the hot bin's coupling through its non-hot entries
  int64_t hot_copy = 0;               // hot-set kernel: > 0 = hot values gathered from the rolling copy hot_hc (period)
  float *hot_hc = nullptr;            // device [K]: rolling copy of the hot values in slot order
  double hot_cover = 0.0;             // share of the bin's entries that are hot
  int64_t head_copy = 0;              // > 0: head gathers from svr[0, H), one chunk refreshed every head_copy rows
  int tail_snap = 0;                  // 1: the head kernel reads the tail [tail_lo, tail_hi) of the shared vector
                                      // from the read copy svr (rolling refresh, or before every slice)
  float *svr = nullptr;               // device [n_shared]: the read copy (only [tail_lo, tail_hi) is maintained)
  int64_t tail_lo = 0, tail_hi = 0;
  int64_t sv_active = 0;              // dual: w̄ is zero beyond [0, sv_active) on every rank (aggregation extent)
  bool sv_active_global = false;      // sv_active already reduced (max) over the ranks
  double tail_tau = 0.0;              // staleness bound of the head bin's coupling through the tail entries
  int64_t tail_roll = 0;              // > 0: the tail copy is refreshed chunk by chunk inside the epoch (every
                                      // tail_roll-th row one 1024-float chunk) instead of between slices
  std::string err;
};

namespace scd {

// error helpers -------------------------------------------------------------------------------
scd_status fail(scd_ctx *c, scd_status s, const std::string &msg);
scd_status cuda_fail(scd_ctx *c, cudaError_t e, const char *what);
void set_global_error(const std::string &msg);

#define SCD_CK(ctx, call)                                  \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return scd::cuda_fail(ctx, e_, #call); \
  } while (0)

#define SCD_CKL(ctx, what)                                 \
  do {                                                     \
    cudaError_t e_ = cudaGetLastError();                   \
    if (e_ != cudaSuccess) return scd::cuda_fail(ctx, e_, what); \
  } while (0)

// collectives over the context's communicator: NCCL, or the caller's hooks (comm.cu).  All are
// stream-ordered on c->stream; with the hooks they complete before returning.
scd_status coll_allreduce(scd_ctx *c, void *buf, size_t count, scd_dtype dt, scd_redop op);
scd_status coll_allgather(scd_ctx *c, const void *send, void *recv, size_t bytes);
scd_status coll_group_start(scd_ctx *c);
scd_status coll_group_end(scd_ctx *c);
#define SCD_COLL(call)                   \
  do {                                   \
    scd_status st_ = (call);             \
    if (st_ != SCD_OK) return st_;       \
  } while (0)

#define SCD_NCK(ctx, call)                                 \
  do {                                                     \
    ncclResult_t r_ = (call);                              \
    if (r_ != ncclSuccess) return scd::fail(ctx, SCD_E_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// layout.cu ------------------------------------------------------------------------------------
scd_status validate_matrix(scd_ctx *c, int64_t outer, int64_t inner);
scd_status compute_norms(scd_ctx *c);
scd_status build_schedule(scd_ctx *c);
scd_status estimate_bin_tau(scd_ctx *c, const int32_t *d_list, int64_t count, double *tau, int64_t lo = -1,
                            double *tau_tail = nullptr);
scd_status estimate_tail_tau(scd_ctx *c, const int32_t *d_list, int64_t count, int64_t lo, double *tau,
                             const int32_t *idx = nullptr);
scd_status renumber_device(const int64_t *ptr, const int32_t *idx, const float *val, int64_t outer, int64_t inner,
                           int64_t nnz, int64_t *optr, int32_t *oidx, float *oval, int32_t *new_of_old, cudaStream_t s,
                           std::string &err);
scd_status transpose_device(const int64_t *ptr, const int32_t *idx, const float *val, int64_t outer, int64_t inner,
                            int64_t nnz, int64_t *optr, int32_t *oidx, float *oval, cudaStream_t s, std::string &err);

// epoch.cu -------------------------------------------------------------------------------------
scd_status run_epoch(scd_ctx *c, uint32_t epoch, int part, int nparts);
scd_status profile_collect(scd_ctx *c);
scd_status tune_shared_layout(scd_ctx *c);
void bin_launch_shape(scd_ctx *c, Bin &b);
double combine_budget(const scd_ctx *c, const Bin &b);  // deferred-update budget of a bin (reading c25)
bool sm_head_shape(scd_ctx *c, Bin &b);  // SM-shared head kernel shape (false = not used)
int sm_chunk_entries(int groups);        // SM-shared head kernel: entries per staged chunk
double cap_fraction();  // in-flight cap as a fraction of a staleness bound (layout.cu)
scd_status launch_perm_export(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n, int64_t *d_out, cudaStream_t s);
scd_status launch_block_order_export(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n, int64_t blk,
                                     int64_t *d_out, cudaStream_t s);
scd_status partition_balanced_device(const int64_t *ptr, int64_t n, uint64_t seed, int32_t k, int32_t *d_owner,
                                     cudaStream_t s, std::string &err);
scd_status launch_partition_export(uint64_t seed, int64_t count, int32_t k, int32_t *d_owner, cudaStream_t s);

// hot.cu ---------------------------------------------------------------------------------------
scd_status setup_hot(scd_ctx *c);


// evaluate.cu ----------------------------------------------------------------------------------
scd_status evaluate(scd_ctx *c, double *primal, double *dual, double *gap);
scd_status evaluate_group(scd_ctx *const *cs, int32_t k, double *primal, double *dual, double *gap);
scd_status rebuild_shared(scd_ctx *c);
scd_status shared_to_w(scd_ctx *c, float *d_out);

// aggregate.cu ---------------------------------------------------------------------------------
scd_status aggregate(scd_ctx *c, scd_agg mode, double *gamma);
scd_status aggregate_group(scd_ctx *const *cs, int32_t k, scd_agg mode, double *gamma);

// shared device helpers ------------------------------------------------------------------------
// Implicit-value matrices (val == nullptr): every stored value is 1.0f — the one-hot case of the
// paper's criteo footnote ("the values ... are always 1 ... one could halve the memory usage",
// P:460).  The pointer test is uniform across the grid, so it costs no divergence.
__device__ __forceinline__ float val_cs(const float *v, int64_t k) { return v ? __ldcs(v + k) : 1.f; }
__device__ __forceinline__ float val_cg(const float *v, int64_t k) { return v ? __ldcg(v + k) : 1.f; }
__device__ __forceinline__ float val_at(const float *v, int64_t k) { return v ? v[k] : 1.f; }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide fp64 sum of `v` added atomically into *out (one atomic per block).
template <int T>
__device__ __forceinline__ void block_sum_atomic(double v, double *out) {
  __shared__ double s_part[T / 32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_part[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = (lane < T / 32) ? s_part[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) atomicAdd(out, t);
  }
  __syncthreads();
}

inline int grid_for(int64_t n, int block, int cap = 148 * 16) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace scd
