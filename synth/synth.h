/* synth.h — seeded synthetic input generators (test/bench infrastructure).
 *
 * This module is the ONLY code shared by the oracle side and the CUDA side, and it
 * holds none of the method's arithmetic (no SCD update, objective, gap, permutation
 * or aggregation).  It produces a sparse matrix A (CSR, rows sorted, indices unique),
 * labels y, from a 64-bit seed, with the shapes the paper's workloads have
 * (§III.D l.254: webspam, 262,938 x 680,715 non-zero features;
 *  §V.B l.460: criteo, ~200M x 75M, values always 1).  The recipe is in DESIGN.md §3.
 *
 * Two twins implement the same integer-only definition:
 *   synth_host.c  — plain C, multithreaded over rows (OpenMP)
 *   synth_cuda.cu — CUDA (one CTA per row, shared-memory bitmap)
 * and the tests check them bit-exact against each other.  Every random number is a
 * counter-based hash (splitmix64 finaliser) of (seed, tag, a, b); floats are formed by
 * exact integer -> float conversion and power-of-two scaling only, so both twins agree
 * bit for bit.  The alias and row-length tables are built once on the host (fp64) and
 * passed to both twins as inputs.
 */
#ifndef SYNTH_H
#define SYNTH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define SYNTH_TAG_LEN 1ull
#define SYNTH_TAG_DRAW 2ull
#define SYNTH_TAG_VAL 3ull
#define SYNTH_TAG_SIGN 4ull
#define SYNTH_TAG_FLIP 5ull
#define SYNTH_LEN_TABLE 1024

/* Row-wise Zipf generator ("webspam-shaped"): row n has k_n = min(len_table[H(seed,LEN,n,0)>>54], n_active)
 * distinct column ids, the first k_n distinct values of the draw sequence d = 0,1,2,...
 * of an alias-table sampler over [0, n_active) (ids are frequency ranks).            */
typedef struct {
  int64_t n_rows;          /* N */
  int64_t n_cols;          /* M, column-id space (ids >= n_active are empty columns) */
  int64_t n_active;        /* F <= M, ids are drawn from [0, F) */
  uint64_t seed;
  int32_t values_one;      /* 1: every value is 1.0f (one-hot); 0: hashed codes in (0,1], row-scaled */
  int32_t flip_mask;       /* label noise: label flipped when (H(seed,FLIP,n,0) & flip_mask) == 0; 0 = never */
  const uint32_t *len_table;  /* [1024] row nnz table */
  const uint32_t *alias_thr;  /* [F] */
  const uint32_t *alias_idx;  /* [F] */
} synth_zipf_rows;

/* One-hot field generator ("criteo-shaped"): row n has exactly one id per field i,
 * id = field_off[i] + rank, rank drawn from field i's alias table (stored at
 * alias_*[field_off[i] .. field_off[i]+field_card[i]) ).  Values are 1.0f.            */
typedef struct {
  int64_t n_rows;
  int64_t n_cols;          /* = field_off[n_fields-1] + field_card[n_fields-1] */
  int32_t n_fields;
  int32_t flip_mask;
  uint64_t seed;
  const int64_t *field_off;   /* [n_fields], strictly increasing */
  const int64_t *field_card;  /* [n_fields], >= 1 */
  const uint32_t *alias_thr;  /* [n_cols] */
  const uint32_t *alias_idx;  /* [n_cols] */
} synth_fields;

/* ---- host twin (synth_host.c); all pointers host ---- */
/* Vose alias table for weights w[0..n).  thr[i] = P(keep i | bucket i) * 2^32 (saturated). */
int synth_build_alias(const double *w, int64_t n, uint32_t *thr, uint32_t *alias);
/* Row lengths for rows [row0, row0+nrows). */
void synth_zipf_row_lengths(const synth_zipf_rows *p, int64_t row0, int64_t nrows, int64_t *len_out);
/* Fill CSR rows [row0, row0+nrows): ptr_local[0..nrows] (ptr_local[0]=0) from synth_zipf_row_lengths;
 * writes idx, val (nnz entries) and y[nrows].  Returns 0 on success. */
int synth_zipf_fill(const synth_zipf_rows *p, int64_t row0, int64_t nrows, const int64_t *ptr_local,
                    int32_t *idx, float *val, float *y, int nthreads);
int synth_fields_fill(const synth_fields *p, int64_t row0, int64_t nrows,
                      int32_t *idx, float *val, float *y, int nthreads);

/* ---- device twin (synth_cuda.cu); matrix/label pointers device, tables host (uploaded) ---- */
/* Generates rows [row0, row0+nrows) into device buffers.  ptr_dev must hold nrows+1 int64,
 * idx/val must be large enough: call synth_zipf_row_lengths on host (cheap) to size them.
 * stream: cudaStream_t or NULL.  Returns 0 on success, else a CUDA error code. */
int synth_zipf_fill_device(const synth_zipf_rows *p, int64_t row0, int64_t nrows, int64_t *ptr_dev,
                           int32_t *idx_dev, float *val_dev, float *y_dev, void *stream);
int synth_fields_fill_device(const synth_fields *p, int64_t row0, int64_t nrows, int64_t *ptr_dev,
                             int32_t *idx_dev, float *val_dev, float *y_dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif
