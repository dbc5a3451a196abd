/* oracle.c — TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct sequential fp64
 * reference for the TPA-SCD hot path of Parnell et al., "Large-Scale Stochastic Learning
 * using GPUs" (arXiv 1702.07005).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code with the
 * CUDA product path (paper_1702_07005_b200/) and neither includes nor links the other.
 *
 * Citations: "P:n" = PAPER.md line n (section / equation / algorithm given alongside).
 * Readings of ambiguous passages are DESIGN.md §4 items (c1..c23).
 *
 * Data are fp32 as in the paper ("32-bit floating point"); the oracle
 * promotes every value to fp64 and computes in fp64 throughout (DESIGN.md c18).
 *
 * Pins (tests/test_oracle_pins.py): closed-form normal equations, per-update stationarity,
 * monotone objective, strong duality, SPEC hand values, brute-force permutations.
 * Permutation / partition / transpose have no paper value: "parity unpinned" beyond their
 * invariants (bijection, balance, involution) — see DESIGN.md §5.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------
 * Permutation P_epoch (Alg. 1 "Generate random permutation of features P_epoch", P:144;
 * Alg. 2).  The paper does not name a generator; DESIGN.md c8 fixes a keyed
 * 4-round balanced Feistel network on [0, 4^h) with cycle-walking into [0, n).
 * Written out here directly from that definition.
 * ---------------------------------------------------------------------------------- */
static uint64_t orc_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t orc_perm_key(uint64_t seed, uint32_t epoch, uint32_t stream) {
  return orc_mix64(seed ^ orc_mix64(((uint64_t)epoch << 32) | (uint64_t)stream));
}

/* One application of the Feistel bijection on [0, 2^(2h)). */
static uint64_t orc_feistel(uint64_t x, int h, uint64_t key) {
  uint64_t mask = (h >= 32) ? 0xFFFFFFFFull : ((1ull << h) - 1ull);
  uint64_t L = x >> h, R = x & mask;
  for (uint64_t r = 0; r < 4; ++r) {
    uint64_t F = orc_mix64(R ^ orc_mix64(key + r)) & mask;
    uint64_t t = L ^ F;
    L = R;
    R = t;
  }
  return (L << h) | R;
}

/* half-width h for domain size n >= 2: bits = ceil(log2 n), h = ceil(bits/2) */
static int orc_half_bits(int64_t n) {
  int bits = 0;
  uint64_t v = (uint64_t)(n - 1);
  while (v) { ++bits; v >>= 1; }
  return (bits + 1) / 2;
}

int64_t orc_perm_at(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n, int64_t j) {
  if (n <= 1) return 0;
  uint64_t key = orc_perm_key(seed, epoch, stream);
  int h = orc_half_bits(n);
  uint64_t x = (uint64_t)j;
  do { x = orc_feistel(x, h, key); } while (x >= (uint64_t)n);
  return (int64_t)x;
}

void orc_permutation(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n, int64_t *out) {
  for (int64_t j = 0; j < n; ++j) out[j] = orc_perm_at(seed, epoch, stream, n, j);
}

/* Block order of an epoch (reading c28, short coordinates): the n / blk full blocks of blk
 * consecutive coordinates are visited in the order of the permutation over the blocks, the coordinates
 * of a block in turn, the last partial block (n mod blk coordinates) at the end.  out[t] = coordinate
 * visited at position t. */
void orc_block_order(uint64_t seed, uint32_t epoch, uint32_t stream, int64_t n, int64_t blk, int64_t *out) {
  const int64_t nf = n / blk;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t tb = t / blk;
    out[t] = tb < nf ? orc_perm_at(seed, epoch, stream, nf, tb) * blk + (t - tb * blk) : t;
  }
}

/* Partition (Alg. 3 "Partition data by feature and distribute on the K workers", P:274;
 * random rows P:462).  DESIGN.md c15: a random permutation (stream 0x50415254, epoch 0)
 * cut into K contiguous blocks whose sizes differ by at most one (first count%K blocks
 * are one larger).  owner[c] = block holding c. */
void orc_partition(uint64_t seed, int64_t count, int32_t k, int32_t *owner) {
  int64_t base = count / k, rem = count % k;
  for (int64_t i = 0; i < count; ++i) {
    int64_t c = orc_perm_at(seed, 0u, 0x50415254u, count, i);
    int64_t b = (i < rem * (base + 1)) ? i / (base + 1) : rem + (i - rem * (base + 1)) / base;
    owner[c] = (int32_t)b;
  }
}

/* Stable transpose CSR <-> CSC (plumbing; "compressed sparse column format ... for the
 * primal and compressed sparse row format ... for the dual").  Entries of each output outer
 * index appear in increasing input-outer order (counting sort, sequential). */
void orc_transpose(int64_t n_outer, int64_t n_inner, const int64_t *ptr, const int32_t *idx, const float *val,
                   int64_t *optr, int32_t *oidx, float *oval) {
  memset(optr, 0, sizeof(int64_t) * (size_t)(n_inner + 1));
  for (int64_t o = 0; o < n_outer; ++o)
    for (int64_t e = ptr[o]; e < ptr[o + 1]; ++e) optr[idx[e] + 1] += 1;
  for (int64_t i = 0; i < n_inner; ++i) optr[i + 1] += optr[i];
  int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_inner > 0 ? n_inner : 1));
  for (int64_t i = 0; i < n_inner; ++i) cur[i] = optr[i];
  for (int64_t o = 0; o < n_outer; ++o)
    for (int64_t e = ptr[o]; e < ptr[o + 1]; ++e) {
      int64_t d = cur[idx[e]]++;
      oidx[d] = (int32_t)o;
      oval[d] = val[e];
    }
  free(cur);
}

/* Squared norms ||a_m||^2 (columns, Eq. 2 denominator) or ||ā_n||^2 (rows, Eq. 4),
 * fp64, summed in storage order.  Precomputed once (DESIGN.md c9). */
void orc_sq_norms(int64_t n_outer, const int64_t *ptr, const float *val, double *out) {
  for (int64_t o = 0; o < n_outer; ++o) {
    double s = 0.0;
    for (int64_t e = ptr[o]; e < ptr[o + 1]; ++e) s += (double)val[e] * (double)val[e];
    out[o] = s;
  }
}

/* ------------------------------------------------------------------------------------
 * Primal sequential SCD, Alg. 1, update rule Eq. (2) and shared
 * vector update.  A is CSC (columns a_m).  For each m = order[j], j = 0..n_order-1:
 *     Δβ = ( <y - w, a_m> - N λ β_m ) / ( ||a_m||^2 + N λ )
 *     β_m += Δβ ;  w += a_m Δβ
 * lamN = λ·N with N the (global) number of examples (DESIGN.md c14).
 * If stat != NULL, stat[j] = ∂P/∂β_m after the update, computed from scratch as
 * (1/N)<Aβ - y, a_m> + λ β_m using the maintained w (pinned: must vanish).
 * ---------------------------------------------------------------------------------- */
void orc_primal_epoch(int64_t n_examples, const int64_t *cptr, const int32_t *ridx, const float *val,
                      const double *y, double lam, double lamN, const double *sqnorm, double *beta, double *w,
                      const int64_t *order, int64_t n_order, double *stat) {
  for (int64_t j = 0; j < n_order; ++j) {
    int64_t m = order[j];
    double dp = 0.0;
    for (int64_t e = cptr[m]; e < cptr[m + 1]; ++e) dp += (y[ridx[e]] - w[ridx[e]]) * (double)val[e];
    double delta = (dp - lamN * beta[m]) / (sqnorm[m] + lamN);
    beta[m] += delta;
    for (int64_t e = cptr[m]; e < cptr[m + 1]; ++e) w[ridx[e]] += (double)val[e] * delta;
    if (stat) {
      double g = 0.0;
      for (int64_t e = cptr[m]; e < cptr[m + 1]; ++e) g += (w[ridx[e]] - y[ridx[e]]) * (double)val[e];
      stat[j] = g / (double)n_examples + lam * beta[m];
    }
  }
}

/* ------------------------------------------------------------------------------------
 * Dual sequential SCD (SDCA), Alg. 1 with update rule Eq. (4) (the printed
 * α_i is read as α_n, DESIGN.md c2) and shared vector update.  A is CSR (rows ā_n).
 *     Δα = ( λ y_n - <w̄, ā_n> - λ N α_n ) / ( λ N + ||ā_n||^2 )
 *     α_n += Δα ;  w̄ += ā_n Δα
 * If stat != NULL, stat[j] = ∂D/∂α_n after the update:
 *     -N α_n - (1/λ)<w̄, ā_n> + y_n        (must vanish)
 * ---------------------------------------------------------------------------------- */
void orc_dual_epoch(const int64_t *rptr, const int32_t *cidx, const float *val, const double *y, double lam,
                    int64_t n_global, const double *sqnorm, double *alpha, double *wbar, const int64_t *order,
                    int64_t n_order, double *stat) {
  const double N = (double)n_global;
  const double lamN = lam * N;
  for (int64_t j = 0; j < n_order; ++j) {
    int64_t n = order[j];
    double dp = 0.0;
    for (int64_t e = rptr[n]; e < rptr[n + 1]; ++e) dp += wbar[cidx[e]] * (double)val[e];
    double delta = (lam * y[n] - dp - lamN * alpha[n]) / (lamN + sqnorm[n]);
    alpha[n] += delta;
    for (int64_t e = rptr[n]; e < rptr[n + 1]; ++e) wbar[cidx[e]] += (double)val[e] * delta;
    if (stat) {
      double g = 0.0;
      for (int64_t e = rptr[n]; e < rptr[n + 1]; ++e) g += wbar[cidx[e]] * (double)val[e];
      stat[j] = -N * alpha[n] - g / lam + y[n];
    }
  }
}
