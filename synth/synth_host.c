/* synth_host.c — host twin of the seeded synthetic input generators (see synth.h).
 * Test/bench infrastructure; holds none of the method's arithmetic. */
#include "synth.h"
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t sx_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static inline uint64_t sx_h(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b) {
  return sx_mix64(sx_mix64(sx_mix64(seed ^ (tag * 0xD6E8FEB86659FD93ull)) ^ a) ^ b);
}
static inline uint32_t sx_alias_draw(uint64_t u, uint64_t n, const uint32_t *thr, const uint32_t *alias) {
  uint32_t b = (uint32_t)(((u >> 32) * n) >> 32);
  uint32_t coin = (uint32_t)u;
  return coin < thr[b] ? b : alias[b];
}
static inline int sx_log2_floor(uint64_t k) { int e = 0; while (k > 1) { k >>= 1; ++e; } return e; }

int synth_build_alias(const double *w, int64_t n, uint32_t *thr, uint32_t *alias) {
  if (n <= 0) return 0;
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) sum += w[i];
  if (!(sum > 0.0)) return 1;
  double *p = (double *)malloc(sizeof(double) * (size_t)n);
  int64_t *small = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t *large = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  if (!p || !small || !large) { free(p); free(small); free(large); return 2; }
  int64_t ns = 0, nl = 0;
  for (int64_t i = 0; i < n; ++i) {
    p[i] = w[i] * (double)n / sum;
    alias[i] = (uint32_t)i;
    if (p[i] < 1.0) small[ns++] = i; else large[nl++] = i;
  }
  while (ns > 0 && nl > 0) {
    int64_t s = small[--ns], l = large[--nl];
    double ps = p[s];
    thr[s] = (uint32_t)(ps * 4294967296.0);
    alias[s] = (uint32_t)l;
    p[l] = (p[l] + ps) - 1.0;
    if (p[l] < 1.0) small[ns++] = l; else large[nl++] = l;
  }
  while (nl > 0) { int64_t l = large[--nl]; thr[l] = 0xFFFFFFFFu; alias[l] = (uint32_t)l; }
  while (ns > 0) { int64_t s = small[--ns]; thr[s] = 0xFFFFFFFFu; alias[s] = (uint32_t)s; }
  free(p); free(small); free(large);
  return 0;
}

static inline int64_t zipf_row_len(const synth_zipf_rows *p, int64_t n) {
  int64_t k = (int64_t)p->len_table[sx_h(p->seed, SYNTH_TAG_LEN, (uint64_t)n, 0) >> 54];
  if (k > p->n_active) k = p->n_active;
  return k;
}

void synth_zipf_row_lengths(const synth_zipf_rows *p, int64_t row0, int64_t nrows, int64_t *len_out) {
  for (int64_t r = 0; r < nrows; ++r) len_out[r] = zipf_row_len(p, row0 + r);
}

static int cmp_u32(const void *a, const void *b) {
  uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  return (x > y) - (x < y);
}

int synth_zipf_fill(const synth_zipf_rows *p, int64_t row0, int64_t nrows, const int64_t *ptr_local,
                    int32_t *idx, float *val, float *y, int nthreads) {
  const int64_t F = p->n_active;
  const size_t words = (size_t)((F + 63) / 64);
  int err = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
  {
    uint64_t *bm = (uint64_t *)calloc(words, sizeof(uint64_t));
    int64_t maxlen = 0;
    for (int64_t i = 0; i < SYNTH_LEN_TABLE; ++i)
      if ((int64_t)p->len_table[i] > maxlen) maxlen = p->len_table[i];
    if (maxlen > F) maxlen = F;
    uint32_t *list = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(maxlen > 0 ? maxlen : 1));
    if (!bm || !list) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
      err = 1;
    } else {
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
      for (int64_t r = 0; r < nrows; ++r) {
        const int64_t n = row0 + r;
        const int64_t k = ptr_local[r + 1] - ptr_local[r];
        const uint64_t rowkey = sx_mix64(sx_mix64(p->seed ^ (SYNTH_TAG_DRAW * 0xD6E8FEB86659FD93ull)) ^ (uint64_t)n);
        int64_t cnt = 0;
        for (uint64_t d = 0; cnt < k; ++d) {
          uint32_t f = sx_alias_draw(sx_mix64(rowkey ^ d), (uint64_t)F, p->alias_thr, p->alias_idx);
          uint64_t bit = 1ull << (f & 63);
          if (!(bm[f >> 6] & bit)) { bm[f >> 6] |= bit; list[cnt++] = f; }
        }
        qsort(list, (size_t)k, sizeof(uint32_t), cmp_u32);
        const int e = sx_log2_floor((uint64_t)(k > 0 ? k : 1)) / 2;
        int64_t score = 0;
        int32_t *ri = idx + ptr_local[r];
        float *rv = val + ptr_local[r];
        for (int64_t j = 0; j < k; ++j) {
          uint32_t f = list[j];
          bm[f >> 6] = 0;  /* clear (whole word; all set bits of this row are cleared by the end) */
          uint64_t code = p->values_one ? 1u : ((sx_h(p->seed, SYNTH_TAG_VAL, (uint64_t)n, f) >> 40) + 1u);
          ri[j] = (int32_t)f;
          rv[j] = p->values_one ? 1.0f : ldexpf((float)code, -24 - e);
          int64_t sgn = (sx_h(p->seed, SYNTH_TAG_SIGN, f, 0) & 1u) ? 1 : -1;
          score += sgn * (int64_t)code;
        }
        float lab = score >= 0 ? 1.0f : -1.0f;
        if (p->flip_mask && (sx_h(p->seed, SYNTH_TAG_FLIP, (uint64_t)n, 0) & (uint64_t)p->flip_mask) == 0) lab = -lab;
        y[r] = lab;
      }
    }
    free(bm);
    free(list);
  }
  return err;
}

int synth_fields_fill(const synth_fields *p, int64_t row0, int64_t nrows,
                      int32_t *idx, float *val, float *y, int nthreads) {
  const int nf = p->n_fields;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static, 4096)
#endif
  for (int64_t r = 0; r < nrows; ++r) {
    const int64_t n = row0 + r;
    const uint64_t rowkey = sx_mix64(sx_mix64(p->seed ^ (SYNTH_TAG_DRAW * 0xD6E8FEB86659FD93ull)) ^ (uint64_t)n);
    int64_t score = 0;
    for (int i = 0; i < nf; ++i) {
      const int64_t off = p->field_off[i];
      uint32_t rank = sx_alias_draw(sx_mix64(rowkey ^ (uint64_t)i), (uint64_t)p->field_card[i],
                                    p->alias_thr + off, p->alias_idx + off);
      uint64_t f = (uint64_t)off + rank;
      idx[r * nf + i] = (int32_t)f;
      val[r * nf + i] = 1.0f;
      score += (sx_h(p->seed, SYNTH_TAG_SIGN, f, 0) & 1u) ? 1 : -1;
    }
    float lab = score >= 0 ? 1.0f : -1.0f;
    if (p->flip_mask && (sx_h(p->seed, SYNTH_TAG_FLIP, (uint64_t)n, 0) & (uint64_t)p->flip_mask) == 0) lab = -lab;
    y[r] = lab;
  }
  return 0;
}
