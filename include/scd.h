/* scd.h — C ABI of the B200-native TPA-SCD library (paper_1702_07005_b200/libscd.so).
 *
 * Hot path of Parnell, Dünner, Atasu, Sifalakis, Pozidis, "Large-Scale Stochastic Learning
 * using GPUs" (arXiv 1702.07005): the twice-parallel asynchronous stochastic coordinate
 * descent (TPA-SCD) epoch for L2-regularised ridge regression, in the primal form (by
 * feature, CSC columns) and the dual form (SDCA, by example, CSR rows), the fp64 objective and
 * duality-gap evaluation, and the distributed aggregation with add / average / closed-form
 * optimal gamma.  Citations: "P:n" = PAPER.md line n, with the section / equation /
 * algorithm it belongs to.  Readings of ambiguous passages are DESIGN.md §4 items (cN).
 *
 * Problem (§II): A ∈ R^{N×M} (N examples, M features), y ∈ R^N, λ > 0.
 *   primal  P(β) = 1/(2N)||Aβ - y||² + λ/2 ||β||²                 Eq. (1)
 *   dual    D(α) = -N/2 ||α||² - 1/(2λ)||Aᵀα||² + αᵀy             Eq. (3)
 *
 * Conventions for every entry point:
 *  - Every call returns scd_status; nothing throws or aborts across the ABI.  On failure a
 *    context-owned message is available from scd_last_error(ctx) (valid until the next call
 *    on that context); context-free calls report through scd_last_global_error().
 *  - Data is fp32 (values, labels, model, shared vector) with int32 inner indices and int64
 *    outer offsets ("all data is represented using 32-bit floating point").  Objective,
 *    gap and gamma are computed and returned in fp64.
 *  - "device" pointers are CUDA device pointers on the current device at scd_create time.
 *  - Calls on one context are not thread-safe; distinct contexts may be used concurrently.
 *  - scd_epoch only enqueues work on the context stream (no host sync).  scd_objective,
 *    scd_duality_gap, scd_aggregate, scd_get_* synchronise that stream.
 */
#ifndef SCD_H
#define SCD_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SCD_OK = 0,
  SCD_E_INVALID_ARG = 1,  /* λ <= 0, N < 1, M < 1, null pointer, length mismatch, form/layout mismatch */
  SCD_E_BAD_MATRIX = 2,   /* offsets/indices violate the CSR/CSC invariants; scd_last_error names the first bad outer index */
  SCD_E_OOM = 3,          /* device allocation failed */
  SCD_E_CUDA = 4,         /* a CUDA runtime call or kernel failed */
  SCD_E_NCCL = 5,         /* an NCCL call failed */
  SCD_E_STATE = 6,        /* call not valid in the context's state (e.g. world > 1 without a communicator) */
  SCD_E_UNSUPPORTED = 7   /* valid request this build does not implement */
} scd_status;

typedef enum { SCD_PRIMAL = 0 /* A must be CSC (by feature) */, SCD_DUAL = 1 /* A must be CSR (by example) */ } scd_form;

/* Aggregation of the K workers' updates each round (§IV): γ = 1 (adding), γ = 1/K
 * (averaging, Alg. 3), or the closed-form optimum (Alg. 4, Eq. 7 P:362 and the dual γ̄
 * P:369, with the corrections of DESIGN.md c3, c4, c5). */
typedef enum { SCD_AGG_ADD = 0, SCD_AGG_AVERAGE = 1, SCD_AGG_OPTIMAL = 2 } scd_agg;

typedef enum { SCD_MEM_HOST = 0, SCD_MEM_DEVICE = 1 } scd_mem;
typedef enum { SCD_CSR = 0, SCD_CSC = 1 } scd_layout;

/* Sparse matrix (the local shard of A).  outer = n_rows for CSR, n_cols for CSC.
 *   ptr[outer+1]: ptr[0] = 0, nondecreasing, ptr[outer] = nnz
 *   idx[nnz]    : inner indices in [0, inner), strictly increasing within each outer index
 *   val[nnz]    : values, or NULL = every stored value is 1.0f (one-hot data: the paper's criteo
 *                 footnote "values ... are always 1 ... could halve the memory usage")
 * Ownership: if mem == SCD_MEM_DEVICE the arrays are BORROWED for the lifetime of the context
 * (the caller keeps them alive and unmodified until scd_destroy; the paper's data "is
 * transferred into the GPU memory once ... and does not move").  If SCD_MEM_HOST the
 * library copies them to the device during scd_create and owns the copy.                    */
typedef struct {
  scd_layout layout;
  int64_t n_rows, n_cols, nnz;
  const int64_t *ptr;
  const int32_t *idx;
  const float *val;
  scd_mem mem;
} scd_matrix;

/* Collective transport for world > 1.  The default is NCCL (scd_options.nccl_comm, over NVLink /
 * NVSwitch).  Alternatively the caller may supply these two host-side hooks over its own process
 * group (e.g. torch.distributed / gloo): NCCL refuses two ranks on one GPU, so the hooks are what
 * lets the library's multi-rank logic (aggregation rounds, the active-extent exchange, the fused
 * peer-memory exchange, the collective objective/gap, the shared-vector rebuild) run with several
 * processes on a single device.  Both hooks receive DEVICE pointers of the calling context and
 * its stream; they must complete the operation in the stream's order (e.g. synchronise the
 * stream, reduce through host memory, copy back) before returning, and return 0 on success
 * (anything else makes the library call fail with SCD_E_NCCL).
 *   allreduce: in place, count elements of dtype (scd_dtype), op (scd_redop), every rank
 *   allgather: recv[r*bytes, (r+1)*bytes) = rank r's send[0, bytes)
 * The struct is BORROWED for the lifetime of the context.                                    */
typedef enum { SCD_DT_F32 = 0, SCD_DT_F64 = 1, SCD_DT_I32 = 2, SCD_DT_I64 = 3, SCD_DT_U8 = 4 } scd_dtype;
typedef enum { SCD_OP_SUM = 0, SCD_OP_MAX = 1, SCD_OP_MIN = 2 } scd_redop;
typedef struct {
  void *user;
  int32_t (*allreduce)(void *user, void *buf, int64_t count, int32_t dtype, int32_t op, void *stream);
  int32_t (*allgather)(void *user, const void *send, void *recv, int64_t bytes, void *stream);
} scd_collectives;

typedef struct {
  uint64_t seed;          /* permutation key: epoch t visits coordinates in P_t = feistel(seed, t) order (c8) */
  int64_t n_global;       /* N used in λN when the dual is sharded by example (c14); 0 = n_rows */
  int32_t rank, world;    /* world = K workers; 1 = single GPU (default) */
  void *nccl_comm;        /* ncclComm_t; world > 1 needs this or `collectives` (see scd_nccl_comm_init); not owned */
  void *stream;           /* cudaStream_t for all work; NULL = a context-owned stream */
  int32_t deterministic;  /* 1 = debug mode: ONE coordinate at a time in exact P_t order, fixed reduction
                             tree; bitwise repeatable (parity with the sequential oracle, Alg. 1) */
  int32_t max_inflight;   /* cap on coordinates in flight in the asynchronous kernels; 0 = auto */
  int32_t recompute_every;/* rebuild the shared vector from the model in fp64 (P:164 recomputation, SURVEY
                             NEXT-2): world = 1 every k epochs (in scd_epoch); world > 1 every k rounds, at
                             the end of scd_aggregate from the aggregated model (collective).  0 = off */
  int32_t validate;       /* 1 = check the matrix invariants on the device at create (default 1) */
  int32_t profile;        /* 1 = time every kernel launch of scd_epoch with CUDA events (scd_profile_read) */
  int32_t wild;           /* 1 = "wild" scatter: plain load + store instead of the atomic add, so concurrent
                             updates of one shared-vector entry can be lost (PASSCoDe-Wild, P:164, P:254;
                             SURVEY NEXT-4).  A measured comparison only: it converges to a point that
                             violates the optimality conditions.  Uses the plain kernels (no head
                             combining, no CTA combining).  0 = atomic (default, the paper's TPA-SCD). */
  const scd_collectives *collectives; /* host-side transport hooks instead of nccl_comm (NULL = NCCL) */
  int32_t block_order;    /* short coordinates (<= 64 entries, the 8-lane bins) are visited in blocks of this many
                             consecutive coordinates in a random block order (reading c28; their per-coordinate
                             offsets, model, norm and label then share sectors) when the bin's in-flight cap spans
                             >= 32 blocks; 0 = default (32), 1 = off */
} scd_options;

typedef struct scd_ctx scd_ctx;

/* Fills *opt with defaults: seed 0, n_global 0, rank 0, world 1, no comm, NULL stream,
 * deterministic 0, max_inflight 0 (auto), recompute_every 0, validate 1, profile 0. */
void scd_default_options(scd_options *opt);

/* Creates a solver context for the ridge problem (A, y, λ) in the given form.
 *   A     : local shard, CSC for SCD_PRIMAL (N × M_k: all rows, own columns), CSR for SCD_DUAL
 *           (N_k × M: own rows, all columns).
 *   y     : labels, length A->n_rows (dual: the shard's rows); copied if y_mem == SCD_MEM_HOST,
 *           borrowed if SCD_MEM_DEVICE.
 *   lambda: λ > 0.
 * Initial state: model = 0, shared vector = 0 (w = Aβ = 0; w̄ = Aᵀα = 0), as in Alg. 1/2
 * "Initialize: β = 0, w = 0".  Precomputes the squared norms ||a_m||² / ||ā_n||²
 * (c9) and the coordinate schedule.  Errors: SCD_E_INVALID_ARG, SCD_E_BAD_MATRIX, SCD_E_OOM,
 * SCD_E_CUDA, SCD_E_STATE (world > 1 without nccl_comm or collectives), SCD_E_INVALID_ARG
 * (dual with world > 1 and n_global = 0).  On error *out is NULL.                           */
scd_status scd_create(const scd_matrix *A, const float *y, scd_mem y_mem, double lambda, scd_form form,
                      const scd_options *opt, scd_ctx **out);

/* One local epoch (Alg. 2): every local coordinate is updated exactly once, in the
 * order P_epoch, by the rule Eq. (2) (primal) or Eq. (4) (dual); the shared vector
 * is updated with fp32 atomic adds.  Asynchronous: many coordinates in flight
 * (any interleaving is a valid execution, c19) unless options.deterministic.  Enqueued on the
 * context stream; returns without synchronising.                                               */
scd_status scd_epoch(scd_ctx *c, uint32_t epoch);

/* Part `part` (0 <= part < nparts <= 1024) of epoch `epoch`: the coordinates at positions
 * [n·part/nparts, n·(part+1)/nparts) of every bin's permutation (the deterministic mode: of the
 * epoch permutation).  Calling parts 0..nparts-1 in order updates every coordinate exactly once
 * (in the deterministic mode it is exactly scd_epoch's sequence of updates); calling
 * scd_aggregate between parts gives sub-epoch aggregation rounds — "communicate shared vector
 * updates more frequently".  Enqueued only, like scd_epoch.            */
scd_status scd_epoch_part(scd_ctx *c, uint32_t epoch, int32_t part, int32_t nparts);

/* Primal and dual objectives, fp64, computed from scratch (the shared vector is NOT trusted).
 *   primal form: *primal = P(β), *dual = D((y - Aβ)/N)      (Eq. 6 map)
 *   dual form  : *primal = P(Aᵀα/λ), *dual = D(α)            (Eq. 5 map)
 * Collective over the workers if world > 1.  Either output pointer may be NULL.  Syncs.     */
scd_status scd_objective(scd_ctx *c, double *primal, double *dual);

/* Duality gap G_P(β) / G_D(α) of §II.C, fp64, from scratch, evaluated through the
 * cancellation-free identity G_P = ||∇P(β)||²/(2λ), G_D = ||∇D(α)||²/(2N) (c13).  Collective
 * if world > 1.  Syncs.                                                                       */
scd_status scd_duality_gap(scd_ctx *c, double *gap);

/* One aggregation round of Alg. 3/4 over the world's workers, after each ran
 * scd_epoch from the common base point: Δ_k = (local state) - (base), Δw = Σ_k Δw_k (NCCL
 * all-reduce over NVLink when world > 1), γ per mode, then w = w_base + γΔw and
 * model_k = model_k,base + γΔmodel_k; the result becomes the next base point (c6).
 * *gamma (may be NULL) receives γ.  A zero update gives γ = 0 for SCD_AGG_OPTIMAL (c16).
 * Collective if world > 1.  Syncs.                                                            */
scd_status scd_aggregate(scd_ctx *c, scd_agg mode, double *gamma);

/* The same round for k logical workers living on ONE device (each ctx created with world = 1
 * and its own shard; all on the same device, same form and λ, n_global = the total N for the
 * dual).  Used to test the distributed algorithm without a multi-GPU box.  Syncs.            */
scd_status scd_aggregate_group(scd_ctx *const *ctxs, int32_t k, scd_agg mode, double *gamma);

/* Objectives and duality gap (as scd_objective / scd_duality_gap) of the global model held by k
 * logical workers on one device (the shards of scd_aggregate_group).  Any output may be NULL.  */
scd_status scd_evaluate_group(scd_ctx *const *ctxs, int32_t k, double *primal, double *dual, double *gap);

/* Copies β_k (primal, length n_cols) or α_k (dual, length n_rows) to host memory. Syncs. */
scd_status scd_get_model(scd_ctx *c, float *host_out, int64_t len);
/* Copies the shared vector w = Aβ (primal, length N) or w̄ = Aᵀα (dual, length M) to host.
 * (Internally the primal keeps the residual r = y - w; w is formed on the device.)  Syncs.   */
scd_status scd_get_shared(scd_ctx *c, float *host_out, int64_t len);
/* Sets the model from host memory and rebuilds the shared vector from it (fp64 accumulate;
 * collective if world > 1); resets the aggregation base point.  Syncs.                      */
scd_status scd_set_model(scd_ctx *c, const float *host_in, int64_t len);
/* Rebuilds the shared vector from the model (the recomputation scheme of A-SCD). Syncs. */
scd_status scd_recompute_shared(scd_ctx *c);

/* The cudaStream_t the context enqueues on. */
scd_status scd_get_stream(scd_ctx *c, void **stream);

typedef struct {
  int64_t n_coord;        /* local coordinates (M_k primal, N_k dual) */
  int64_t n_shared;       /* shared-vector length (N primal, M dual) */
  int64_t nnz;
  int64_t n_nonempty;     /* coordinates with at least one stored entry */
  int32_t n_bins;         /* asynchronous schedule: number of coordinate bins (one kernel launch each) */
  int32_t bin_kind[4];    /* per bin: lanes per coordinate (4..32 = sub-warp group, >= 64 = whole CTA) */
  int64_t bin_count[4];   /* coordinates per bin */
  int64_t bin_nnz[4];     /* stored entries per bin */
  int32_t bin_grid[4];    /* CTAs launched per bin */
  int32_t bin_block[4];   /* threads per CTA per bin */
  int64_t launches;       /* kernels launched by the context since create (cumulative) */
  double tau_star;        /* estimated staleness bound: coordinates in flight before the asynchronous
                             step stops being contractive */
  int64_t inflight_cap;   /* largest per-bin cap on coordinates in flight */
  int64_t bin_cap[4];     /* per bin: coordinates in flight allowed (max_inflight, else bin_tau/2) */
  double bin_tau[4];      /* per bin: estimated staleness bound */
  int32_t n_slices;       /* the bins are interleaved in this many slices per epoch (reading c24) */
  int64_t sv_offset_bytes;/* placement of the shared vector chosen at create */
  float probe_best_ms;    /* placement probe: fastest / slowest candidate (0 if not probed) */
  float probe_worst_ms;
  int32_t bin_head[4];    /* per bin: > 0 = the CTA kernel combines updates of sv[0, bin_head) in shared
                             memory (head-combining kernel); 0 = plain */
  int32_t bin_flush[4];   /* per bin: coordinates per CTA between flushes of the combined head */
  int32_t bin_hot[4];     /* per bin: > 0 = hot-set kernel with this many hot shared-vector entries (hot.cu) */
  double hot_cover;       /* share of the hot bin's stored entries that fall on a hot entry */
  int32_t tail_snap;      /* head kernel: 1 = tail gathers (ids >= bin_head) read a copy of the shared vector
                             refreshed before every slice; 0 = off */
  double tail_tau;        /* staleness bound of the coupling through the tail entries (coordinates); the
                             tail copy is used only while a slice's coordinates are <= tail_tau / 2 */
  int32_t bin_snap[4];    /* per bin: 1 = each slice launch gathers from a copy of the shared vector taken just
                             before it (the slice's coordinates are within the bin's in-flight cap) */
  int64_t tail_roll;      /* > 0: the tail copy is refreshed inside the epoch, one 1024-float chunk every tail_roll
                             rows (no slice boundaries); 0 = refreshed between slices */
  int64_t head_copy;      /* > 0: the head gathers also read a copy of w̄[0, bin_head) refreshed in rolling
                             1024-float chunks every head_copy rows; 0 = off */
  int64_t hot_copy;       /* > 0: the hot-set kernel gathers the hot values from a copy refreshed 32 slots at a
                             time every hot_copy warp tickets; 0 = off */
  int32_t hot_tp;         /* 1: the hot-set kernel gathers the next batch's non-hot values one step early */
  double hot_tail_tau;    /* staleness bound of the hot bin's coupling through its non-hot entries; the early
                             gather is used only while 2 x rows in flight <= hot_tail_tau / 2 */
  int32_t hot_hp;         /* 1: the hot values of the next batch are also gathered one step early (from the copy) */
  int32_t sm_head;        /* > 0: the head bin runs the SM-shared head kernel with this many row groups per SM
                             (one CTA per SM sharing a snapshot of w̄[0, bin_head) and its pending updates;
                             rows staged in shared memory by bulk copies); 0 = off */
  int32_t sm_chunk;       /* SM-shared head kernel: entries per bulk-copied chunk of a row */
  int32_t sm_ch;          /* SM-shared head kernel: head chunks (1024 floats) flushed and re-read per flushing row */
  int32_t sm_rh;          /* SM-shared head kernel: rows per flushing row (an SM's head chunk rotates every
                             bin_head / 1024 / sm_ch * sm_rh of its rows) */
} scd_info;
scd_status scd_get_info(scd_ctx *c, scd_info *info);

/* Per-kernel CUDA-event timing of scd_epoch launches (options.profile = 1): for each bin b,
 * ms_out[b] = summed device time of its launches since the last read, count_out[b] = launches.
 * Synchronises.  n = capacity of the arrays (>= 4 recommended); returns the bins filled.     */
scd_status scd_profile_read(scd_ctx *c, double *ms_out, int64_t *count_out, int32_t n, int32_t *filled);

const char *scd_last_error(const scd_ctx *c);   /* context-owned, valid until the next call on c */
const char *scd_last_global_error(void);         /* thread-local, for context-free calls */
const char *scd_status_string(scd_status s);
/* ABI check for bindings: sizes_out[0..3] = sizeof(scd_matrix), sizeof(scd_options), sizeof(scd_info),
 * sizeof(scd_collectives). */
void scd_struct_sizes(int64_t *sizes_out);
void scd_destroy(scd_ctx *c);                    /* NULL-safe; syncs the stream; frees owned memory */

/* ---- integer artefacts (computed on the device; bit-exact with the oracle) ---- */
/* host_out[j] = P_(seed,epoch,stream)(j) for j in [0, n): the keyed Feistel bijection of c8. */
scd_status scd_permutation(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n, int64_t *host_out);
/* Epoch visiting order in block order (reading c28: used for the short-coordinate bins): the
 * n / blk full blocks of blk consecutive positions are permuted by P_(seed,epoch,stream) over the
 * blocks, a block's coordinates are visited in turn, the last partial block comes last.  host_out[t]
 * = coordinate at position t (int64, n entries).  blk = 1 is scd_permutation.  Errors:
 * SCD_E_INVALID_ARG (n < 0, blk < 1, NULL output), SCD_E_CUDA.                                 */
scd_status scd_block_permutation(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n, int64_t blk,
                                 int64_t *host_out);
/* owner_out[c] (host) = worker owning coordinate c in [0, count) for k workers (c15). */
scd_status scd_partition(uint64_t seed, int64_t count, int32_t k, int32_t *host_owner_out);
/* Stored-entry balanced partition of the n outer coordinates of a matrix (columns of a CSC for the
 * primal, rows of a CSR for the dual) over k workers ("partition the coordinates
 * in an intelligent way"; reading c29): coordinates in decreasing length, ties in the order
 * of the partition permutation of scd_partition (same seed), dealt in snake order 0..k-1, k-1..0, ...
 * ptr[n+1] is host or device memory (ptr_mem); host_owner_out[n] receives the worker of each
 * coordinate.  Errors: SCD_E_INVALID_ARG, SCD_E_UNSUPPORTED (n > 2^31-1), SCD_E_OOM, SCD_E_CUDA.   */
scd_status scd_partition_balanced(const int64_t *ptr, int64_t n, scd_mem ptr_mem, uint64_t seed, int32_t k,
                                  int32_t *host_owner_out);
/* Stable transpose CSR <-> CSC computed on the device.  in->mem says where the input lives;
 * out_mem where ptr_out[inner+1] / idx_out[nnz] / val_out[nnz] (caller-allocated) live.
 * Within each output outer index, entries appear in increasing input-outer order.
 * If in->val is NULL (implicit values) only the pattern is transposed and val_out is ignored.  */
scd_status scd_transpose(const scd_matrix *in, int64_t *ptr_out, int32_t *idx_out, float *val_out, scd_mem out_mem);
/* Renumbering of the inner index space by frequency (the "renumber by frequency at load" of the
 * data layer, SURVEY K8'): new id of inner index j = its rank by (number of stored entries with index
 * j, descending; j ascending).  Output: the same offsets (ptr_out[outer+1]), the relabelled entries
 * re-sorted increasingly within each outer index (idx_out/val_out[nnz], values moved with their
 * entries), and new_of_old_out[inner] (caller-allocated, in out_mem) so a shared vector computed on
 * the renumbered matrix maps back as x_old[j] = x_new[new_of_old[j]].  Computed on the device; integer
 * results are exact.  The head-combining epoch kernel needs frequency-ranked indices.
 * Errors: SCD_E_INVALID_ARG (NULL / bad shape / inner > INT32_MAX), SCD_E_OOM, SCD_E_CUDA.          */
scd_status scd_renumber(const scd_matrix *in, int64_t *ptr_out, int32_t *idx_out, float *val_out,
                        int32_t *new_of_old_out, scd_mem out_mem);

/* ---- LIBSVM reader (host; the paper's datasets, P:254 webspam, P:460 criteo) ----
 * Format: one example per line, `label index:value ...`, 1-based strictly increasing indices per
 * line; text after '#' is a comment; blank lines are skipped; values parsed as double and rounded to
 * fp32; indices become 0-based.  n_cols_hint > 0 fixes the number of columns (error if an index
 * exceeds it), else n_cols = largest index.  Two passes: scd_libsvm_size reports the shape, then
 * scd_libsvm_read fills caller-allocated host CSR arrays ptr[n_rows+1], idx[nnz], val[nnz],
 * y[n_rows].  Errors: SCD_E_INVALID_ARG with the file / line in scd_last_global_error().          */
scd_status scd_libsvm_size(const char *path, int64_t n_cols_hint, int64_t *n_rows, int64_t *nnz, int64_t *n_cols);
scd_status scd_libsvm_read(const char *path, int64_t n_cols_hint, int64_t *ptr, int32_t *idx, float *val, float *y);

/* ---- NCCL bootstrap helpers (the caller broadcasts the 128-byte id, e.g. via torch.distributed) ---- */
scd_status scd_nccl_unique_id(void *id_out_128);
scd_status scd_nccl_comm_init(const void *id_128, int32_t world, int32_t rank, void **comm_out);
scd_status scd_nccl_comm_destroy(void *comm);

#ifdef __cplusplus
}
#endif
#endif /* SCD_H */
