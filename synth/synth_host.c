/*
 * synth/synth_host.c — host side of the seeded input generator (see gen_core.h).
 * Built with: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC.
 * Contains no SsNAL-EN arithmetic; produces A (column-major), x*, b.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "gen_core.h"

/* Raw + standardised column j of a design of the given kind into col[m]. */
static int column_std(int kind, uint64_t seed, int64_t m, int64_t n, int64_t j, double* col) {
  if (kind == SX_IID_UNIT_L2 || kind == SX_IID_STD) {
    for (int64_t k = 0; k < m; ++k) col[k] = sx_iid_entry(seed, m, k, j);
  } else if (kind == SX_GENO_STD) {
    for (int64_t k = 0; k < m; ++k) col[k] = sx_geno_entry(seed, m, n, k, j);
  } else if (kind == SX_AR1_STD) {
    int64_t c0 = (j / SX_AR1_CHUNK) * SX_AR1_CHUNK;
    for (int64_t k = 0; k < m; ++k) {
      double a = sx_ar1_start(seed, m, k, c0);
      for (int64_t l = c0 + 1; l <= j; ++l) a = sx_ar1_step(a, sx_iid_entry(seed, m, k, l));
      col[k] = a;
    }
  } else {
    return -1;
  }
  return sx_standardise(col, m, kind == SX_IID_UNIT_L2) ? 0 : 1;
}

/* Fill columns [j0, j1) of A into out (column-major, (j1-j0)*m doubles).
 * Returns 0, or the number of zero-variance columns, or -1 for a bad kind. */
int synth_fill_A(int kind, uint64_t seed, int64_t m, int64_t n, int64_t j0, int64_t j1, double* out) {
  if (m < 1 || n < 1 || j0 < 0 || j1 > n || j0 > j1) return -1;
  int64_t bad = 0;
  if (kind == SX_AR1_STD) {
    int64_t cfirst = j0 / SX_AR1_CHUNK, clast = (j1 - 1) / SX_AR1_CHUNK;
    if (j1 == j0) return 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : bad)
    for (int64_t c = cfirst; c <= clast; ++c) {
      int64_t c0 = c * SX_AR1_CHUNK;
      int64_t ce = c0 + SX_AR1_CHUNK < n ? c0 + SX_AR1_CHUNK : n;
      for (int64_t k = 0; k < m; ++k) {
        double a = sx_ar1_start(seed, m, k, c0);
        for (int64_t j = c0; j < ce; ++j) {
          if (j > c0) a = sx_ar1_step(a, sx_iid_entry(seed, m, k, j));
          if (j >= j0 && j < j1) out[(j - j0) * m + k] = a;
        }
      }
      int64_t lo = c0 > j0 ? c0 : j0, hi = ce < j1 ? ce : j1;
      for (int64_t j = lo; j < hi; ++j)
        if (!sx_standardise(out + (j - j0) * m, m, 0)) bad++;
    }
    return (int)bad;
  }
  if (kind != SX_IID_UNIT_L2 && kind != SX_IID_STD && kind != SX_GENO_STD) return -1;
#pragma omp parallel for schedule(static) reduction(+ : bad)
  for (int64_t j = j0; j < j1; ++j)
    if (column_std(kind, seed, m, n, j, out + (j - j0) * m) != 0) bad++;
  return (int)bad;
}

/* Gather arbitrary columns idx[0..cnt) (each standardised) into out[cnt*m]. */
int synth_columns(int kind, uint64_t seed, int64_t m, int64_t n, const int64_t* idx, int64_t cnt, double* out) {
  int64_t bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : bad)
  for (int64_t t = 0; t < cnt; ++t)
    if (column_std(kind, seed, m, n, idx[t], out + t * m) != 0) bad++;
  return (int)bad;
}

/* x*: k distinct indices in [0,n) by counter-based rejection, sorted ascending;
 * value i = (+/-1 with prob 1/2) * U[lo, hi]. */
int synth_xstar(uint64_t seed, int64_t n, int64_t k, double lo, double hi, int64_t* idx, double* val) {
  if (k < 0 || k > n) return -1;
  uint64_t kx = sx_key(seed, SX_S_XIDX), kv = sx_key(seed, SX_S_XVAL);
  int64_t got = 0;
  for (uint64_t t = 0; got < k; ++t) {
    int64_t c = (int64_t)(sx_u01(kx, t) * (double)n);
    if (c >= n) c = n - 1;
    int dup = 0;
    for (int64_t i = 0; i < got; ++i)
      if (idx[i] == c) { dup = 1; break; }
    if (!dup) idx[got++] = c;
  }
  for (int64_t i = 1; i < k; ++i) { /* insertion sort, k is small */
    int64_t v = idx[i], p = i - 1;
    while (p >= 0 && idx[p] > v) { idx[p + 1] = idx[p]; --p; }
    idx[p + 1] = v;
  }
  for (int64_t i = 0; i < k; ++i) {
    double sgn = sx_u01(kv, 2 * (uint64_t)i) < 0.5 ? -1.0 : 1.0;
    double mag = lo + (hi - lo) * sx_u01(kv, 2 * (uint64_t)i + 1);
    val[i] = sgn * mag;
  }
  return 0;
}

/* b = A x* + eps, eps ~ N(0, s^2), s^2 = var_pop(A x*) / snr.  A x* is
 * accumulated over the support in ascending index order from regenerated
 * columns.  Also returns the realised noise sd in *s_out. */
int synth_response(int kind, uint64_t seed, int64_t m, int64_t n, int64_t k, const int64_t* idx,
                   const double* val, double snr, double* b, double* s_out) {
  double* cols = (double*)malloc(sizeof(double) * (size_t)(m * (k > 0 ? k : 1)));
  if (!cols) return -2;
  int bad = synth_columns(kind, seed, m, n, idx, k, cols);
  for (int64_t r = 0; r < m; ++r) {
    double v = 0.0;
    for (int64_t i = 0; i < k; ++i) v += val[i] * cols[i * m + r];
    b[r] = v;
  }
  free(cols);
  double s = 0.0;
  for (int64_t r = 0; r < m; ++r) s += b[r];
  double mean = s / (double)m, var = 0.0;
  for (int64_t r = 0; r < m; ++r) var += (b[r] - mean) * (b[r] - mean);
  var /= (double)m;
  double sd = snr > 0 ? sqrt(var / snr) : 0.0;
  uint64_t kn = sx_key(seed, SX_S_NOISE);
  for (int64_t r = 0; r < m; ++r) b[r] += sd * sx_normal(kn, (uint64_t)r);
  if (s_out) *s_out = sd;
  return bad;
}

/* Test vectors: count normals / uniforms from the test stream (sub-stream id). */
void synth_normals(uint64_t seed, uint64_t sub, int64_t count, double* out) {
  uint64_t key = sx_key(seed ^ (sub * 0x9E3779B97F4A7C15ULL), SX_S_TEST);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) out[i] = sx_normal(key, (uint64_t)i);
}
void synth_uniforms(uint64_t seed, uint64_t sub, int64_t count, double* out) {
  uint64_t key = sx_key(seed ^ (sub * 0x9E3779B97F4A7C15ULL), SX_S_TEST);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) out[i] = sx_u01(key, (uint64_t)i);
}

/* Packed 2-bit genotype codes of columns [j0, j1) of a SX_GENO_STD design (gen_core.h
 * sx_geno_packed): codes ((j1-j0) × stride bytes), tab ((j1-j0) × 3 doubles).
 * Returns 0, the number of zero-variance columns, or -1 for bad arguments. */
int synth_geno_codes(uint64_t seed, int64_t m, int64_t n, int64_t j0, int64_t j1, uint8_t* codes, int64_t stride,
                     double* tab) {
  if (m < 1 || n < 1 || j0 < 0 || j1 > n || j0 > j1 || stride < (m + 3) / 4) return -1;
  int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
  for (int64_t j = j0; j < j1; ++j)
    if (!sx_geno_packed(seed, m, n, j, codes + (j - j0) * stride, stride, tab + (j - j0) * 3)) bad++;
  return (int)bad;
}
