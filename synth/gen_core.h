/*
 * synth/gen_core.h — seeded, counter-based input generator shared by the
 * host library (gcc, synth_host.c) and the device library (nvcc,
 * synth_dev.cu).  It holds NONE of SsNAL-EN's arithmetic: only random numbers,
 * the design-matrix recipes of DESIGN.md §"Input recipe" and column
 * standardisation.  Both the CUDA path and the oracle consume its output.
 *
 * Bit-identity contract: every floating-point step is a single IEEE-754
 * correctly rounded operation (+, -, *, /, sqrt) applied in the same order on
 * both sides.  On the device the SX_* macros expand to the __d*_rn intrinsics,
 * which the compiler never contracts into FMAs; on the host the file is
 * compiled with -ffp-contract=off.  The logarithm and cosine used by the
 * Box–Muller transform are therefore written out here as polynomials instead
 * of calling libm / CUDA math (whose last-bit results differ).
 */
#ifndef SYNTH_GEN_CORE_H
#define SYNTH_GEN_CORE_H

#include <stdint.h>

#ifdef __CUDACC__
#define SX_HD __host__ __device__ __forceinline__
#else
#define SX_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define SX_ADD(a, b) __dadd_rn((a), (b))
#define SX_SUB(a, b) __dsub_rn((a), (b))
#define SX_MUL(a, b) __dmul_rn((a), (b))
#define SX_DIV(a, b) __ddiv_rn((a), (b))
#define SX_SQRT(a) __dsqrt_rn((a))
#define SX_AS_U64(d) ((uint64_t)__double_as_longlong(d))
#define SX_AS_F64(u) __longlong_as_double((long long)(u))
#else
#include <math.h>
#include <string.h>
#define SX_ADD(a, b) ((a) + (b))
#define SX_SUB(a, b) ((a) - (b))
#define SX_MUL(a, b) ((a) * (b))
#define SX_DIV(a, b) ((a) / (b))
#define SX_SQRT(a) sqrt((a))
SX_HD uint64_t sx_as_u64(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
SX_HD double sx_as_f64(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
#define SX_AS_U64(d) sx_as_u64(d)
#define SX_AS_F64(u) sx_as_f64(u)
#endif

/* Design-matrix kinds. */
enum {
  SX_IID_UNIT_L2 = 1, /* cfg1: iid N(0,1), centred, ||a_j||_2 = 1            */
  SX_IID_STD = 2,     /* cfg3/5: iid N(0,1), centred, ||a_j||_2^2 = m         */
  SX_AR1_STD = 3,     /* cfg2: AR(1) across columns, rho=0.5, standardised   */
  SX_GENO_STD = 4     /* cfg4: Binomial(2,p_j) genotypes with block linkage  */
};

/* Independent random streams (mixed into the key). */
enum {
  SX_S_A = 1,      /* entries of A (normal draws)                       */
  SX_S_XIDX = 2,   /* support indices of x*                             */
  SX_S_XVAL = 3,   /* signs / magnitudes of x*                          */
  SX_S_NOISE = 4,  /* response noise                                    */
  SX_S_P = 5,      /* genotype allele frequencies p_j                   */
  SX_S_LAT = 6,    /* genotype shared latent uniforms (per block)       */
  SX_S_CHO = 7,    /* genotype "use shared latent" choice               */
  SX_S_FRESH = 8,  /* genotype fresh uniforms                           */
  SX_S_TEST = 9    /* free stream for test vectors (y, x, d ...)         */
};

#define SX_AR1_CHUNK 256   /* AR(1) columns generated per independent chunk */
#define SX_AR1_BURN 64     /* burn-in steps before a chunk (0.5^64 ~ 5e-20)  */
#define SX_GENO_BLOCK 20   /* linkage block width (BASELINE.json cfg4)       */

/* splitmix64 finaliser */
SX_HD uint64_t sx_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

SX_HD uint64_t sx_key(uint64_t seed, uint64_t stream) {
  return sx_mix(sx_mix(seed) ^ (stream * 0xD1B54A32D192ED03ULL));
}

SX_HD uint64_t sx_bits(uint64_t key, uint64_t idx) { return sx_mix(key ^ sx_mix(idx)); }

/* uniform in [0,1): 53 random bits, exact conversion */
SX_HD double sx_u01(uint64_t key, uint64_t idx) {
  return SX_MUL((double)(sx_bits(key, idx) >> 11), 1.1102230246251565e-16 /* 2^-53 */);
}

/* ln(u) for u in (0, 1]; |error| ~ 1 ulp-ish, identical bits host/device. */
SX_HD double sx_log(double u) {
  uint64_t b = SX_AS_U64(u);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  double f = SX_AS_F64((b & 0x000FFFFFFFFFFFFFULL) | 0x3FF0000000000000ULL); /* [1,2) */
  if (f > 1.4142135623730951) { f = SX_MUL(f, 0.5); e += 1; }               /* exact */
  double s = SX_DIV(SX_SUB(f, 1.0), SX_ADD(f, 1.0));                           /* |s|<=0.1716 */
  double s2 = SX_MUL(s, s);
  /* ln f = 2 s (1 + s^2/3 + s^4/5 + ...), 13 terms: s2^13/27 < 1e-21 */
  double p = 1.0 / 27.0;
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 25.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 23.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 21.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 19.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 17.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 15.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 13.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 11.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 9.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 7.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 5.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0 / 3.0);
  p = SX_ADD(SX_MUL(p, s2), 1.0);
  double lnf = SX_MUL(SX_MUL(2.0, s), p);
  /* ln 2 split hi/lo so e*ln2_hi is exact for |e| < 2^11 */
  double ed = (double)e;
  return SX_ADD(SX_ADD(SX_MUL(ed, 6.93147180369123816490e-01), lnf),
                SX_MUL(ed, 1.90821492927058770002e-10));
}

/* cos and sin of phi in [0, pi/2) by Taylor series (phi^26/26! < 1e-21). */
SX_HD double sx_cos_q(double phi) {
  double x2 = SX_MUL(phi, phi);
  /* Horner in x2 on the alternating series: sum_{k=0}^{12} (-1)^k x^{2k}/(2k)! */
  double p = 1.0 / 620448401733239439360000.0;    /* + x^24/24! */
  p = SX_SUB(1.0 / 1124000727777607680000.0, SX_MUL(p, x2));  /* - x^22/22! */
  p = SX_SUB(1.0 / 2432902008176640000.0, SX_MUL(p, x2));     /* + x^20/20! */
  p = SX_SUB(1.0 / 6402373705728000.0, SX_MUL(p, x2));        /* - x^18/18! */
  p = SX_SUB(1.0 / 20922789888000.0, SX_MUL(p, x2));          /* + x^16/16! */
  p = SX_SUB(1.0 / 87178291200.0, SX_MUL(p, x2));             /* - x^14/14! */
  p = SX_SUB(1.0 / 479001600.0, SX_MUL(p, x2));               /* + x^12/12! */
  p = SX_SUB(1.0 / 3628800.0, SX_MUL(p, x2));                 /* - x^10/10! */
  p = SX_SUB(1.0 / 40320.0, SX_MUL(p, x2));                   /* + x^8/8!   */
  p = SX_SUB(1.0 / 720.0, SX_MUL(p, x2));                     /* - x^6/6!   */
  p = SX_SUB(1.0 / 24.0, SX_MUL(p, x2));                      /* + x^4/4!   */
  p = SX_SUB(0.5, SX_MUL(p, x2));                             /* - x^2/2!   */
  p = SX_SUB(1.0, SX_MUL(p, x2));                             /* + 1        */
  return p;
}

SX_HD double sx_sin_q(double phi) {
  double x2 = SX_MUL(phi, phi);
  double p = 1.0 / 15511210043330985984000000.0;              /* x^25/25! */
  p = SX_SUB(1.0 / 25852016738884976640000.0, SX_MUL(p, x2));  /* x^23/23! */
  p = SX_SUB(1.0 / 51090942171709440000.0, SX_MUL(p, x2));     /* x^21/21! */
  p = SX_SUB(1.0 / 121645100408832000.0, SX_MUL(p, x2));       /* x^19/19! */
  p = SX_SUB(1.0 / 355687428096000.0, SX_MUL(p, x2));          /* x^17/17! */
  p = SX_SUB(1.0 / 1307674368000.0, SX_MUL(p, x2));            /* x^15/15! */
  p = SX_SUB(1.0 / 6227020800.0, SX_MUL(p, x2));               /* x^13/13! */
  p = SX_SUB(1.0 / 39916800.0, SX_MUL(p, x2));                 /* x^11/11! */
  p = SX_SUB(1.0 / 362880.0, SX_MUL(p, x2));                   /* x^9/9!   */
  p = SX_SUB(1.0 / 5040.0, SX_MUL(p, x2));                     /* x^7/7!   */
  p = SX_SUB(1.0 / 120.0, SX_MUL(p, x2));                      /* x^5/5!   */
  p = SX_SUB(1.0 / 6.0, SX_MUL(p, x2));                        /* x^3/3!   */
  p = SX_SUB(1.0, SX_MUL(p, x2));                              /* x        */
  return SX_MUL(p, phi);
}

/* Standard normal by Box–Muller (cosine branch) from two counter uniforms. */
SX_HD double sx_normal(uint64_t key, uint64_t idx) {
  uint64_t h1 = sx_bits(key, 2 * idx);
  uint64_t h2 = sx_bits(key, 2 * idx + 1);
  double u1 = SX_MUL((double)((h1 >> 11) + 1), 1.1102230246251565e-16); /* (0,1] */
  double u2 = SX_MUL((double)(h2 >> 11), 1.1102230246251565e-16);       /* [0,1) */
  double rad = SX_SQRT(SX_MUL(-2.0, sx_log(u1)));
  double q4 = SX_MUL(u2, 4.0);          /* exact */
  int q = (int)q4;                      /* 0..3  */
  double v = SX_SUB(q4, (double)q);     /* exact, [0,1) */
  double phi = SX_MUL(v, 1.5707963267948966);
  double c;
  switch (q) {
    case 0: c = sx_cos_q(phi); break;
    case 1: c = -sx_sin_q(phi); break;
    case 2: c = -sx_cos_q(phi); break;
    default: c = sx_sin_q(phi); break;
  }
  return SX_MUL(rad, c);
}

/* ---- raw (pre-standardisation) entries ------------------------------------ */

/* iid N(0,1) entry (row k, column j) */
SX_HD double sx_iid_entry(uint64_t seed, int64_t m, int64_t k, int64_t j) {
  return sx_normal(sx_key(seed, SX_S_A), (uint64_t)j * (uint64_t)m + (uint64_t)k);
}

/* Genotype code g in {0,1,2}: two alleles, each 1[U < p_j]; U is the block's
 * shared latent with prob 0.8, else a fresh uniform (reading R18). */
SX_HD double sx_geno_entry(uint64_t seed, int64_t m, int64_t n, int64_t k, int64_t j) {
  double pj = SX_ADD(0.05, SX_MUL(0.45, sx_u01(sx_key(seed, SX_S_P), (uint64_t)j)));
  int64_t nb = (n + SX_GENO_BLOCK - 1) / SX_GENO_BLOCK;
  int64_t blk = j / SX_GENO_BLOCK;
  int g = 0;
  for (int a = 0; a < 2; ++a) {
    uint64_t cell = ((uint64_t)j * (uint64_t)m + (uint64_t)k) * 2u + (uint64_t)a;
    double v = sx_u01(sx_key(seed, SX_S_CHO), cell);
    double u;
    if (v < 0.8)
      u = sx_u01(sx_key(seed, SX_S_LAT), ((uint64_t)k * (uint64_t)nb + (uint64_t)blk) * 2u + (uint64_t)a);
    else
      u = sx_u01(sx_key(seed, SX_S_FRESH), cell);
    g += (u < pj) ? 1 : 0;
  }
  return (double)g;
}

/* AR(1) across columns with rho = 0.5:  a_j = 0.5 a_{j-1} + sqrt(0.75) e_j,
 * regenerated per chunk of SX_AR1_CHUNK columns after SX_AR1_BURN burn-in steps
 * (column 0 starts at e_0).  ar1_start returns the value at the chunk's first
 * column; sx_ar1_step advances one column. */
SX_HD double sx_ar1_step(double prev, double e) {
  return SX_ADD(SX_MUL(0.5, prev), SX_MUL(0.8660254037844386 /* sqrt(0.75) */, e));
}
SX_HD double sx_ar1_start(uint64_t seed, int64_t m, int64_t k, int64_t c0) {
  if (c0 == 0) return sx_iid_entry(seed, m, k, 0);
  int64_t l0 = c0 - SX_AR1_BURN;
  if (l0 < 0) l0 = 0;
  double a = sx_iid_entry(seed, m, k, l0);
  for (int64_t l = l0 + 1; l <= c0; ++l) a = sx_ar1_step(a, sx_iid_entry(seed, m, k, l));
  return a;
}

/* Column standardisation in place (col has m entries), fixed sequential order:
 * centre by the mean, then divide by sqrt(sum sq) (unit l2) or sqrt(sum sq / m)
 * (unit variance, divisor m).  Returns 0 if the column has zero variance. */
SX_HD int sx_standardise(double* col, int64_t m, int unit_l2) {
  double s = 0.0;
  for (int64_t k = 0; k < m; ++k) s = SX_ADD(s, col[k]);
  double mean = SX_DIV(s, (double)m);
  double ss = 0.0;
  for (int64_t k = 0; k < m; ++k) {
    double c = SX_SUB(col[k], mean);
    col[k] = c;
    ss = SX_ADD(ss, SX_MUL(c, c));
  }
  if (!(ss > 0.0)) return 0;
  double nrm = unit_l2 ? SX_SQRT(ss) : SX_SQRT(SX_DIV(ss, (double)m));
  for (int64_t k = 0; k < m; ++k) col[k] = SX_DIV(col[k], nrm);
  return 1;
}

/* ---- compressed genotype storage ------------------------------
 * Column j of a SX_GENO_STD design as 2-bit codes g ∈ {0,1,2}, four rows per byte
 * (row k in bits 2(k%4)..2(k%4)+1 of byte k/4), plus the 3-entry table
 * v[g] = (g − mean_j) / nrm_j computed with sx_standardise's exact operations, so that
 * v[code(k, j)] equals the standardised fp64 design entry bit for bit (zero-variance
 * column: v[g] = g − mean_j, as the generator writes it).  `codes` has `stride` bytes
 * (≥ ceil(m/4), padding zero).  Returns 1, or 0 for a zero-variance column. */
SX_HD int sx_geno_packed(uint64_t seed, int64_t m, int64_t n, int64_t j, uint8_t* codes, int64_t stride,
                         double* v) {
  for (int64_t q = 0; q < stride; ++q) codes[q] = 0;
  double s = 0.0;
  for (int64_t k = 0; k < m; ++k) {
    const double g = sx_geno_entry(seed, m, n, k, j);
    codes[k >> 2] = (uint8_t)(codes[k >> 2] | ((int)g << (2 * (int)(k & 3))));
    s = SX_ADD(s, g);
  }
  const double mean = SX_DIV(s, (double)m);
  double ss = 0.0;
  for (int64_t k = 0; k < m; ++k) {
    const double c = SX_SUB((double)((codes[k >> 2] >> (2 * (int)(k & 3))) & 3), mean);
    ss = SX_ADD(ss, SX_MUL(c, c));
  }
  const int ok = ss > 0.0;
  const double nrm = SX_SQRT(SX_DIV(ss, (double)m));
  for (int g = 0; g < 3; ++g) v[g] = ok ? SX_DIV(SX_SUB((double)g, mean), nrm) : SX_SUB((double)g, mean);
  return ok;
}

#endif /* SYNTH_GEN_CORE_H */
