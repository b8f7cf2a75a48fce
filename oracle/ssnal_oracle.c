/*
 * oracle/ssnal_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct fp64 CPU implementation of SsNAL-EN
 * (arXiv 2006.03970) used to check the CUDA path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library; the product (paper_2006_03970_b200) never does.
 *
 * It shares no code with the CUDA path.  Every function cites the passage of
 * /root/reference/PAPER.md it restates ("P:<line>", equation numbers as in the
 * paper) and, where the paper is silent or garbled, the DESIGN.md reading
 * ("R<k>", numbering of SURVEY.md Appendix A).
 *
 * Conventions: A is column-major m x n (lda = m): A[k + i*m] is row k of
 * column a_i.  All sums are sequential in ascending index order; the only
 * parallelism is `omp parallel for` over independent columns, so results are
 * bit-identical for any thread count.  Built with -O2 -ffp-contract=off.
 *
 * Pins (tests/test_oracle_*.py): Eq. (6) values and Moreau identity,
 * Prop. 1 vs a brute-force supremum, Prop. 2 vs Eq. (7) at z̄, Eq. (15) vs
 * finite differences, Eq. (18)/(19) vs a dense solve of V d = -∇ψ with Q from
 * Eq. (17), whole-solve vs coordinate descent, KKT inclusion, duality gap,
 * orthonormal / single-column / near-λmax closed forms, x = 0 above λmax.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

#define ORC_EPS 2.220446049250313e-16

/* ------------------------------------------------------------------------- */
/* Penalty, conjugate and proximal maps (Section 2)                            */
/* ------------------------------------------------------------------------- */

/* Elastic Net penalty p(x) = λ1‖x‖₁ + (λ2/2)‖x‖₂²  (Eq. (1)). */
double orc_penalty(const double* x, i64 n, double l1, double l2) {
  double a = 0.0, q = 0.0;
  for (i64 i = 0; i < n; ++i) {
    a += fabs(x[i]);
    q += x[i] * x[i];
  }
  return l1 * a + 0.5 * l2 * q;
}

/* Prop. 1: p*(z) = (1/(2λ2)) Σ ((|z_i| − λ1)_+)².
 * λ2 = 0 (Lasso, Eq. (2)): the indicator of ‖z‖∞ ≤ λ1 → 0 or +inf. */
double orc_pstar(const double* z, i64 n, double l1, double l2) {
  if (l2 == 0.0) {
    for (i64 i = 0; i < n; ++i)
      if (fabs(z[i]) > l1) return INFINITY;
    return 0.0;
  }
  double s = 0.0;
  for (i64 i = 0; i < n; ++i) {
    double zi = z[i], v = 0.0;
    if (zi >= l1) v = (zi - l1) * (zi - l1);          /* case z_i ≥ λ1  */
    else if (zi <= -l1) v = (zi + l1) * (zi + l1);    /* case z_i ≤ −λ1 */
    s += v;
  }
  return s / (2.0 * l2);
}

/* Eq. (6) left: prox_{σp}(t) = soft(t, σλ1)/(1+σλ2).
 * Ties |t| = σλ1 give 0 (P:354 uses strict ">" for the active set; R11). */
double orc_prox(double t, double sigma, double l1, double l2) {
  double thr = sigma * l1;
  double den = 1.0 + sigma * l2;
  if (t > thr) return (t - thr) / den;
  if (t < -thr) return (t + thr) / den;
  return 0.0;
}

/* Eq. (6) right: prox_{p* / σ}(t/σ), written in terms of t. */
double orc_prox_conj(double t, double sigma, double l1, double l2) {
  double thr = sigma * l1;
  double den = 1.0 + sigma * l2;
  if (t >= thr) return (t * l2 + l1) / den;
  if (t <= -thr) return (t * l2 - l1) / den;
  return t / sigma;
}

/* h*(y) = ½‖y‖² + bᵀy. */
double orc_hstar(const double* y, const double* b, i64 m) {
  double q = 0.0, l = 0.0;
  for (i64 k = 0; k < m; ++k) {
    q += y[k] * y[k];
    l += b[k] * y[k];
  }
  return 0.5 * q + l;
}

/* ------------------------------------------------------------------------- */
/* Dense products (plain loops)                                                */
/* ------------------------------------------------------------------------- */

/* w = Aᵀy: w_i = Σ_k A[k,i] y_k, k ascending. */
void orc_aty(const double* A, i64 m, i64 n, const double* y, double* w) {
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n; ++i) {
    const double* a = A + i * m;
    double s = 0.0;
    for (i64 k = 0; k < m; ++k) s += a[k] * y[k];
    w[i] = s;
  }
}

/* out = A x over the nonzeros of x (ascending i). */
void orc_ax(const double* A, i64 m, i64 n, const double* x, double* out) {
  for (i64 k = 0; k < m; ++k) out[k] = 0.0;
  for (i64 i = 0; i < n; ++i) {
    if (x[i] == 0.0) continue;
    const double* a = A + i * m;
    for (i64 k = 0; k < m; ++k) out[k] += a[k] * x[i];
  }
}

/* ------------------------------------------------------------------------- */
/* ψ, ∇ψ, z̄, active set (Section 3.1-3.2)                                      */
/* ------------------------------------------------------------------------- */

/* Prop. 2(1): ψ(y) = h*(y) + (1+σλ2)/(2σ)‖prox_{σp}(x − σAᵀy)‖² − ‖x‖²/(2σ).
 * w = Aᵀy is passed in. */
double orc_psi_w(const double* b, i64 m, i64 n, const double* x, const double* y, const double* w,
                 double sigma, double l1, double l2) {
  double pp = 0.0, xx = 0.0;
  for (i64 i = 0; i < n; ++i) {
    double P = orc_prox(x[i] - sigma * w[i], sigma, l1, l2);
    pp += P * P;
    xx += x[i] * x[i];
  }
  return orc_hstar(y, b, m) + (1.0 + sigma * l2) / (2.0 * sigma) * pp - xx / (2.0 * sigma);
}

double orc_psi(const double* A, const double* b, i64 m, i64 n, const double* x, const double* y, double sigma,
               double l1, double l2) {
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  orc_aty(A, m, n, y, w);
  double v = orc_psi_w(b, m, n, x, y, w, sigma, l1, l2);
  free(w);
  return v;
}

/* Eq. (15): ∇ψ(y) = y + b − A prox_{σp}(x − σAᵀy)  (∇h* = y + b, R1). */
void orc_grad_psi(const double* A, const double* b, i64 m, i64 n, const double* x, const double* y, double sigma,
                  double l1, double l2, double* g) {
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  orc_aty(A, m, n, y, w);
  for (i64 k = 0; k < m; ++k) g[k] = y[k] + b[k];
  for (i64 i = 0; i < n; ++i) {
    double P = orc_prox(x[i] - sigma * w[i], sigma, l1, l2);
    if (P == 0.0) continue;
    const double* a = A + i * m;
    for (i64 k = 0; k < m; ++k) g[k] -= a[k] * P;
  }
  free(w);
}

/* Prop. 2(2): z̄ = prox_{p* / σ}(x/σ − Aᵀy). */
void orc_zbar(const double* A, i64 m, i64 n, const double* x, const double* y, double sigma, double l1, double l2,
              double* z) {
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  orc_aty(A, m, n, y, w);
  for (i64 i = 0; i < n; ++i) z[i] = orc_prox_conj(x[i] - sigma * w[i], sigma, l1, l2);
  free(w);
}

/* Eq. (17): J = {i : |(x − σAᵀy)_i| > σλ1}, ascending; t = x − σAᵀy given. */
i64 orc_active_set(const double* t, i64 n, double sigma, double l1, i64* J) {
  double thr = sigma * l1;
  i64 r = 0;
  for (i64 i = 0; i < n; ++i)
    if (fabs(t[i]) > thr) J[r++] = i;
  return r;
}

/* ------------------------------------------------------------------------- */
/* Newton system (Eq. (16)-(19))                                               */
/* ------------------------------------------------------------------------- */

/* Textbook column Cholesky (lower, column-major N x N, in place).  0 = ok. */
int orc_chol(double* M, i64 N) {
  for (i64 j = 0; j < N; ++j) {
    double s = M[j + j * N];
    for (i64 p = 0; p < j; ++p) s -= M[j + p * N] * M[j + p * N];
    if (!(s > 0.0)) return -1;
    double d = sqrt(s);
    M[j + j * N] = d;
    for (i64 i = j + 1; i < N; ++i) {
      double t = M[i + j * N];
      for (i64 p = 0; p < j; ++p) t -= M[i + p * N] * M[j + p * N];
      M[i + j * N] = t / d;
    }
  }
  return 0;
}

/* Solve (L Lᵀ) v = rhs in place: forward then backward substitution. */
void orc_chol_solve(const double* L, i64 N, double* v) {
  for (i64 i = 0; i < N; ++i) {
    double s = v[i];
    for (i64 p = 0; p < i; ++p) s -= L[i + p * N] * v[p];
    v[i] = s / L[i + i * N];
  }
  for (i64 i = N - 1; i >= 0; --i) {
    double s = v[i];
    for (i64 p = i + 1; p < N; ++p) s -= L[p + i * N] * v[p];
    v[i] = s / L[i + i * N];
  }
}

/* Newton direction: V d = −g with V = I_m + κ A_J A_Jᵀ (Eq. (16), (18)),
 * κ = σ/(1+σλ2).  Branch rule (R12): r = 0 → d = −g;
 * 0 < r < m → Sherman–Morrison–Woodbury Eq. (19), factoring κ⁻¹I_r + A_JᵀA_J (R13);
 * r ≥ m → Cholesky of the m × m matrix Eq. (18).  Returns the branch (0,1,2) or −1. */
int orc_newton_direction(const double* A, i64 m, const i64* J, i64 r, const double* g, double kappa, double jitter,
                         double* d) {
  if (r == 0) {
    for (i64 k = 0; k < m; ++k) d[k] = -g[k];
    return 0;
  }
  if (r < m) {
    double* M = (double*)malloc(sizeof(double) * (size_t)(r * r));
    double* v = (double*)malloc(sizeof(double) * (size_t)r);
#pragma omp parallel for schedule(dynamic, 4)
    for (i64 b = 0; b < r; ++b) {
      const double* ab = A + J[b] * m;
      for (i64 a = b; a < r; ++a) {
        const double* aa = A + J[a] * m;
        double s = 0.0;
        for (i64 k = 0; k < m; ++k) s += aa[k] * ab[k];
        M[a + b * r] = s;
        M[b + a * r] = s;
      }
    }
    double kinv = 1.0 / kappa;
    for (i64 a = 0; a < r; ++a) M[a + a * r] += kinv;
    for (i64 a = 0; a < r; ++a) M[a + a * r] += jitter * M[a + a * r]; /* retry (R36) */
    for (i64 a = 0; a < r; ++a) {
      const double* aa = A + J[a] * m;
      double s = 0.0;
      for (i64 k = 0; k < m; ++k) s += aa[k] * g[k];
      v[a] = s;
    }
    if (orc_chol(M, r) != 0) { free(M); free(v); return -1; }
    orc_chol_solve(M, r, v);
    for (i64 k = 0; k < m; ++k) d[k] = -g[k];
    for (i64 a = 0; a < r; ++a) {
      const double* aa = A + J[a] * m;
      for (i64 k = 0; k < m; ++k) d[k] += aa[k] * v[a];
    }
    free(M);
    free(v);
    return 1;
  }
  double* M = (double*)malloc(sizeof(double) * (size_t)(m * m));
#pragma omp parallel for schedule(dynamic, 4)
  for (i64 l = 0; l < m; ++l) {
    for (i64 k = l; k < m; ++k) {
      double s = 0.0;
      for (i64 a = 0; a < r; ++a) s += A[k + J[a] * m] * A[l + J[a] * m];
      double v = kappa * s + (k == l ? 1.0 : 0.0);
      M[k + l * m] = v;
      M[l + k * m] = v;
    }
  }
  for (i64 k = 0; k < m; ++k) M[k + k * m] += jitter * M[k + k * m]; /* retry (R36) */
  if (orc_chol(M, m) != 0) { free(M); return -1; }
  for (i64 k = 0; k < m; ++k) d[k] = -g[k];
  orc_chol_solve(M, m, d);
  free(M);
  return 2;
}

/* Newton direction by the conjugate-gradient method (Algorithm 1 step (1): "solving exactly or
 * by conjugate gradient"; "approximately with the conjugate gradient method"),
 * matrix-free: V u = u + κ A_J (A_Jᵀ u).  Textbook CG from d0 = 0 (reading R32): stop when
 * ‖V d + g‖ ≤ tol·‖g‖ or after maxit iterations.  Returns the number of iterations. */
int orc_cg_direction(const double* A, i64 m, const i64* J, i64 r, const double* g, double kappa, double tol,
                     int maxit, double* d) {
  double* res = (double*)malloc(sizeof(double) * (size_t)m);
  double* p = (double*)malloc(sizeof(double) * (size_t)m);
  double* q = (double*)malloc(sizeof(double) * (size_t)m);
  double* t = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  double gg = 0.0, rr = 0.0;
  for (i64 k = 0; k < m; ++k) {
    d[k] = 0.0;
    res[k] = -g[k];
    p[k] = res[k];
    gg += g[k] * g[k];
    rr += res[k] * res[k];
  }
  const double thr = tol * tol * gg;
  int it = 0;
  while (it < maxit && rr > thr) {
    /* q = V p = p + κ A_J (A_Jᵀ p) */
    for (i64 a = 0; a < r; ++a) {
      const double* aa = A + J[a] * m;
      double s = 0.0;
      for (i64 k = 0; k < m; ++k) s += aa[k] * p[k];
      t[a] = s;
    }
    for (i64 k = 0; k < m; ++k) {
      double s = 0.0;
      for (i64 a = 0; a < r; ++a) s += A[k + J[a] * m] * t[a];
      q[k] = p[k] + kappa * s;
    }
    double pq = 0.0;
    for (i64 k = 0; k < m; ++k) pq += p[k] * q[k];
    const double alpha = rr / pq;
    double rr_new = 0.0;
    for (i64 k = 0; k < m; ++k) {
      d[k] += alpha * p[k];
      res[k] -= alpha * q[k];
      rr_new += res[k] * res[k];
    }
    const double beta = rr_new / rr;
    for (i64 k = 0; k < m; ++k) p[k] = res[k] + beta * p[k];
    rr = rr_new;
    ++it;
  }
  free(res); free(p); free(q); free(t);
  return it;
}

/* ------------------------------------------------------------------------- */
/* Objectives and certificates (used for stats and pins)                       */
/* ------------------------------------------------------------------------- */

/* F(x) = ½‖Ax − b‖² + λ1‖x‖₁ + (λ2/2)‖x‖²  (Eq. (1)). */
double orc_primal_obj(const double* A, const double* b, i64 m, i64 n, const double* x, double l1, double l2) {
  double* ax = (double*)malloc(sizeof(double) * (size_t)m);
  orc_ax(A, m, n, x, ax);
  double q = 0.0;
  for (i64 k = 0; k < m; ++k) q += (ax[k] - b[k]) * (ax[k] - b[k]);
  free(ax);
  return 0.5 * q + orc_penalty(x, n, l1, l2);
}

/* Dual objective of (D) (reading R2) at z = −Aᵀy: D(y) = −h*(y) − p*(Aᵀy),
 * w = Aᵀy given.  A lower bound on min F for every y (weak duality). */
double orc_dual_obj(const double* b, i64 m, const double* y, const double* w, i64 n, double l1, double l2) {
  return -orc_hstar(y, b, m) - orc_pstar(w, n, l1, l2);
}

/* Elastic Net KKT inclusion c := Aᵀ(b − Ax) − λ2 x ∈ λ1 ∂‖x‖₁; returns max_i v_i with
 * v_i = |c_i − λ1 sign x_i| (x_i ≠ 0) or (|c_i| − λ1)_+ (x_i = 0). */
double orc_kkt_violation(const double* A, const double* b, i64 m, i64 n, const double* x, double l1, double l2) {
  double* res = (double*)malloc(sizeof(double) * (size_t)m);
  double* c = (double*)malloc(sizeof(double) * (size_t)n);
  orc_ax(A, m, n, x, res);
  for (i64 k = 0; k < m; ++k) res[k] = b[k] - res[k];
  orc_aty(A, m, n, res, c);
  double vmax = 0.0;
  for (i64 i = 0; i < n; ++i) {
    double ci = c[i] - l2 * x[i], v;
    if (x[i] > 0) v = fabs(ci - l1);
    else if (x[i] < 0) v = fabs(ci + l1);
    else v = fabs(ci) > l1 ? fabs(ci) - l1 : 0.0;
    if (v > vmax) vmax = v;
  }
  free(res);
  free(c);
  return vmax;
}

/* ------------------------------------------------------------------------- */
/* Algorithm 1 with the readings of DESIGN.md                      */
/* ------------------------------------------------------------------------- */

typedef struct {
  double sigma_factor; /* 5                         */
  double sigma_max;    /* 1e8 (R9)                          */
  double mu;           /* 0.2                       */
  double beta;         /* 0.5 (R5)                          */
  int32_t max_outer;   /* 100 (R10)                         */
  int32_t max_inner;   /* 100 (R10)                         */
  int32_t max_bt;      /* 50 (R30)                          */
  int32_t init_mode;   /* 1: y0 = A x0 − b when x0 ≠ 0, else 0; 0: always y0 = 0 (R8) */
  double cg_ratio;     /* > 0: CG when r > cg_ratio·m (R32); 0: off                */
  double cg_threshold; /* CG when min(m, r) > cg_threshold (10⁴)          */
  double cg_tol;       /* CG relative residual (R32)                               */
  int32_t cg_maxit;
  int32_t inner_tol_mode; /* 0: tol_in = tol (R6); 1: max(tol, 0.1·res3 at the outer start) (R37) */
  double jitter;       /* factor retry: diagonal × (1 + jitter) after a non-positive pivot (R36) */
} orc_opts;

typedef struct {
  int32_t status; /* 0 converged, 1 not converged, 4 numeric */
  int32_t outer_iters, newton_iters, backtracks, aty_passes;
  int32_t branch_steps[4]; /* r = 0, SMW, m × m, CG */
  int32_t line_search_stalled;
  int32_t cg_iters;
  int32_t jitter_retries;
  int64_t active;
  double res_kkt1, res_kkt3, primal_obj, dual_obj, gap, sigma_final;
} orc_stats;

typedef struct { /* one record per Newton step (debugging parity) */
  int32_t outer, branch;
  int64_t r;
  double s, psi, res1, gd;
  int64_t jsum; /* checksum of J (Σ (i+1)·(a+1) mod 2^61) to see whether J changed */
} orc_trace;

typedef struct { /* EVAL(y, w): everything that depends on (x, σ, y) */
  double psi;    /* ψ minus the constant −‖x‖²/(2σ)  (R29) */
  double psimag; /* |½yᵀy| + |bᵀy| + |prox term|, for the Armijo guard (R29) */
  double res1;
  i64 r;
} orc_eval;

/* EVAL(y, w) of DESIGN.md §"Oracle": t = x − σw; P = prox (Eq. (6));
 * J (Eq. (17)); ψ (Prop. 2 without the constant); g = y + b − A_J P_J (Eq. (15));
 * res1 = ‖g‖/(1+‖b‖) (Eq. (20), with x := P, R6). */
static void eval_point(const double* A, const double* b, i64 m, i64 n, const double* x, const double* y,
                       const double* w, double sigma, double l1, double l2, double nb, double* P, i64* J,
                       double* g, orc_eval* ev) {
  double thr = sigma * l1;
  i64 r = 0;
  double pp = 0.0;
  for (i64 i = 0; i < n; ++i) {
    double t = x[i] - sigma * w[i];
    double Pi = orc_prox(t, sigma, l1, l2);
    P[i] = Pi;
    pp += Pi * Pi;
    if (fabs(t) > thr) J[r++] = i;
  }
  double yy = 0.0, by = 0.0;
  for (i64 k = 0; k < m; ++k) {
    yy += y[k] * y[k];
    by += b[k] * y[k];
  }
  double c = (1.0 + sigma * l2) / (2.0 * sigma);
  ev->psi = 0.5 * yy + by + c * pp;
  ev->psimag = fabs(0.5 * yy) + fabs(by) + fabs(c * pp);
  for (i64 k = 0; k < m; ++k) g[k] = y[k] + b[k];
  for (i64 a = 0; a < r; ++a) {
    const double* col = A + J[a] * m;
    double Pa = P[J[a]];
    for (i64 k = 0; k < m; ++k) g[k] -= col[k] * Pa;
  }
  double gg = 0.0;
  for (i64 k = 0; k < m; ++k) gg += g[k] * g[k];
  ev->res1 = sqrt(gg) / (1.0 + nb);
  ev->r = r;
}

/* ψ-part only at (y, w) (line-search trial, Eq. (13)); no gradient. */
static double psi_part(const double* b, i64 m, i64 n, const double* x, const double* y, const double* w,
                       double sigma, double l1, double l2) {
  double pp = 0.0;
  for (i64 i = 0; i < n; ++i) {
    double Pi = orc_prox(x[i] - sigma * w[i], sigma, l1, l2);
    pp += Pi * Pi;
  }
  double yy = 0.0, by = 0.0;
  for (i64 k = 0; k < m; ++k) {
    yy += y[k] * y[k];
    by += b[k] * y[k];
  }
  return 0.5 * yy + by + (1.0 + sigma * l2) / (2.0 * sigma) * pp;
}

void orc_default_opts(orc_opts* o) {
  o->sigma_factor = 5.0;
  o->sigma_max = 1e8;
  o->mu = 0.2;
  o->beta = 0.5;
  o->max_outer = 100;
  o->max_inner = 100;
  o->max_bt = 50;
  o->init_mode = 1;
  o->cg_ratio = 0.0;
  o->cg_threshold = 1e4;
  o->cg_tol = 1e-10;
  o->cg_maxit = 1000;
  o->inner_tol_mode = 0;
  o->jitter = 1e-10;
}

/* SsNAL-EN (Algorithm 1).  x0 may be NULL (cold start).  y0 (nullable): the dual starting point of
 * a warm-started path point — the previous point's final y (reading R39: Algorithm 1 starts "from the
 * initial values y0, z0, x0, σ0", and a path point uses "the solution at the previous
 * value for initialization"); with y0 the start is (x0, y0) and w0 = Aᵀy0 is the previous
 * point's w (recomputed here, but not counted as an aty pass: the method has it already).  x_out (n)
 * and y_out (m, nullable) receive the final iterates.  trace (nullable) receives up to trace_cap
 * Newton-step records; *trace_len their count.  Returns stats.status. */
int orc_solve(const double* A, const double* b, i64 m, i64 n, double l1, double l2, double sigma0, double tol,
              const double* x0, const double* y0, const orc_opts* opts_in, double* x_out, double* y_out,
              orc_stats* st, orc_trace* trace, i64 trace_cap, i64* trace_len) {
  orc_opts o;
  if (opts_in) o = *opts_in; else orc_default_opts(&o);
  orc_stats S;
  memset(&S, 0, sizeof(S));
  i64 ntr = 0;

  double* x = (double*)calloc((size_t)n, sizeof(double));
  double* P = (double*)malloc(sizeof(double) * (size_t)n);
  double* w = (double*)calloc((size_t)n, sizeof(double));
  double* wt = (double*)malloc(sizeof(double) * (size_t)n);
  i64* J = (i64*)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
  double* y = (double*)calloc((size_t)m, sizeof(double));
  double* yt = (double*)malloc(sizeof(double) * (size_t)m);
  double* g = (double*)malloc(sizeof(double) * (size_t)m);
  double* d = (double*)malloc(sizeof(double) * (size_t)m);

  double nb = 0.0;
  for (i64 k = 0; k < m; ++k) nb += b[k] * b[k];
  nb = sqrt(nb);

  /* Initial values (P:242 is silent; reading R8). */
  int warm = 0;
  if (x0) {
    for (i64 i = 0; i < n; ++i) {
      x[i] = x0[i];
      if (x0[i] != 0.0) warm = 1;
    }
  }
  if (y0) {  /* R39: the previous path point's final dual iterate (and its w = Aᵀy) */
    for (i64 k = 0; k < m; ++k) y[k] = y0[k];
    orc_aty(A, m, n, y, w);
  } else if (warm && o.init_mode == 1) {
    orc_ax(A, m, n, x, y);
    for (i64 k = 0; k < m; ++k) y[k] -= b[k];
    orc_aty(A, m, n, y, w);
    S.aty_passes++;
  }
  double sigma = sigma0;
  orc_eval ev;
  int converged = 0, numeric = 0;
  int k;
  for (k = 0; k < o.max_outer && !numeric; ++k) {
    eval_point(A, b, m, n, x, y, w, sigma, l1, l2, nb, P, J, g, &ev);
    /* inner tolerance: tol (R6), or SPEC's schedule max(tol, 0.1·res(kkt3)) with res(kkt3) of
     * Eq. (20) at the point this outer iteration starts from (reading R37) */
    double tol_in = tol;
    if (o.inner_tol_mode) {
      double dx2 = 0.0, zz = 0.0, yy = 0.0;
      for (i64 i = 0; i < n; ++i) {
        double dx = x[i] - P[i];
        double z = dx / sigma - w[i];
        dx2 += dx * dx;
        zz += z * z;
      }
      for (i64 q = 0; q < m; ++q) yy += y[q] * y[q];
      double res3_0 = (sqrt(dx2) / sigma) / (1.0 + sqrt(yy) + sqrt(zz));
      tol_in = fmax(tol, 0.1 * res3_0);
    }
    /* Semi-smooth Newton inner loop. */
    for (int j = 0; j < o.max_inner; ++j) {
      if (ev.res1 <= tol_in) break; /* inner stop, Eq. (20) res(kkt1) (R6) */
      double kappa = sigma / (1.0 + sigma * l2);
      /* strategy (R12, R32): CG iff r > cg_ratio·m (cg_ratio > 0) or min(m, r) > cg_threshold */
      const i64 mr_min = ev.r < m ? ev.r : m;
      const int use_cg = ev.r > 0 && ((o.cg_ratio > 0.0 && (double)ev.r > o.cg_ratio * (double)m) ||
                                      (double)mr_min > o.cg_threshold);
      int br;
      if (use_cg) {
        S.cg_iters += orc_cg_direction(A, m, J, ev.r, g, kappa, o.cg_tol, o.cg_maxit, d);
        br = 3;
      } else {
        br = orc_newton_direction(A, m, J, ev.r, g, kappa, 0.0, d);
        if (br < 0 && o.jitter > 0.0) { /* one retry with the jittered factor (R36) */
          S.jitter_retries++;
          br = orc_newton_direction(A, m, J, ev.r, g, kappa, o.jitter, d);
        }
      }
      if (br < 0) { numeric = 1; break; }
      S.branch_steps[br]++;
      double gd = 0.0;
      for (i64 q = 0; q < m; ++q) gd += g[q] * d[q];
      /* Armijo line search, Eq. (13) with μ, halving (R5), guard (R29). */
      double s = 1.0, psit;
      int nbt = 0;
      for (;;) {
        for (i64 q = 0; q < m; ++q) yt[q] = y[q] + s * d[q];
        orc_aty(A, m, n, yt, wt); /* direct recompute (R14) */
        S.aty_passes++;
        psit = psi_part(b, m, n, x, yt, wt, sigma, l1, l2);
        if (psit - ev.psi <= o.mu * s * gd + 10.0 * ORC_EPS * ev.psimag) break;
        if (nbt >= o.max_bt) { S.line_search_stalled = 1; break; } /* R30 */
        s *= o.beta;
        nbt++;
      }
      S.backtracks += nbt;
      if (trace && ntr < trace_cap) {
        trace[ntr].outer = k;
        trace[ntr].branch = br;
        trace[ntr].r = ev.r;
        trace[ntr].s = s;
        trace[ntr].psi = ev.psi;
        trace[ntr].res1 = ev.res1;
        trace[ntr].gd = gd;
        uint64_t js = 0;
        for (i64 a = 0; a < ev.r; ++a) js = (js + (uint64_t)(J[a] + 1) * (uint64_t)(a + 1)) & ((1ULL << 61) - 1);
        trace[ntr].jsum = (int64_t)js;
      }
      ntr++;
      /* y ← y + s d; z ← z̄(y) implicitly via P (Algorithm 1 steps (3)-(4)). */
      double* tmp = y; y = yt; yt = tmp;
      tmp = w; w = wt; wt = tmp;
      S.newton_iters++;
      eval_point(A, b, m, n, x, y, w, sigma, l1, l2, nb, P, J, g, &ev);
    }
    if (numeric) break;
    /* Multiplier update, Eq. (10): x ← x − σ(Aᵀy + z̄) = P (Moreau,
     * P:145); res(kkt3), Eq. (20), with z̄ = (x − P)/σ − Aᵀy. */
    double dx2 = 0.0, zz = 0.0, yy = 0.0;
    for (i64 i = 0; i < n; ++i) {
      double dx = x[i] - P[i];
      double z = dx / sigma - w[i];
      dx2 += dx * dx;
      zz += z * z;
      x[i] = P[i];
    }
    for (i64 q = 0; q < m; ++q) yy += y[q] * y[q];
    double res3 = (sqrt(dx2) / sigma) / (1.0 + sqrt(yy) + sqrt(zz));
    S.res_kkt3 = res3;
    S.res_kkt1 = ev.res1;
    if (res3 <= tol && ev.res1 <= tol) { converged = 1; k++; break; } /* R7 */
    sigma = fmin(o.sigma_factor * sigma, o.sigma_max);               /* P:497, R9 */
  }
  S.outer_iters = k;
  S.sigma_final = sigma;
  S.status = numeric ? 4 : (converged ? 0 : 1);
  i64 act = 0;
  for (i64 i = 0; i < n; ++i) act += (x[i] != 0.0);
  S.active = act;
  S.primal_obj = orc_primal_obj(A, b, m, n, x, l1, l2);
  S.dual_obj = (l2 > 0.0) ? orc_dual_obj(b, m, y, w, n, l1, l2) : NAN;
  S.gap = S.primal_obj - S.dual_obj;
  memcpy(x_out, x, sizeof(double) * (size_t)n);
  if (y_out) memcpy(y_out, y, sizeof(double) * (size_t)m);
  if (st) *st = S;
  if (trace_len) *trace_len = ntr;
  free(x); free(P); free(w); free(wt); free(J); free(y); free(yt); free(g); free(d);
  return S.status;
}

/* One fused K1-equivalent evaluation, for kernel parity tests:
 * w = Aᵀy; t = x − σw; P; J; and the four partial sums the CUDA K1 reports:
 * [0] Σ P_i², [1] Σ (x_i − P_i)², [2] Σ z_i² with z_i = (x_i − P_i)/σ − w_i,
 * [3] Σ ((|w_i| − λ1)_+)².  Also g = y + b − A_J P_J (if g != NULL). */
i64 orc_aty_fused(const double* A, const double* b, i64 m, i64 n, const double* y, const double* x, double sigma,
                  double l1, double l2, double* w, i64* J, double* PJ, double* partials, double* g) {
  orc_aty(A, m, n, y, w);
  double thr = sigma * l1;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  i64 r = 0;
  for (i64 i = 0; i < n; ++i) {
    double t = x[i] - sigma * w[i];
    double Pi = orc_prox(t, sigma, l1, l2);
    if (fabs(t) > thr) {
      J[r] = i;
      PJ[r] = Pi;
      r++;
    }
    double dx = x[i] - Pi, z = dx / sigma - w[i];
    double e = fabs(w[i]) - l1;
    s0 += Pi * Pi;
    s1 += dx * dx;
    s2 += z * z;
    if (e > 0) s3 += e * e;
  }
  partials[0] = s0; partials[1] = s1; partials[2] = s2; partials[3] = s3;
  if (g) {
    for (i64 k = 0; k < m; ++k) g[k] = y[k] + b[k];
    for (i64 a = 0; a < r; ++a) {
      const double* col = A + J[a] * m;
      for (i64 k = 0; k < m; ++k) g[k] -= col[k] * PJ[a];
    }
  }
  return r;
}

/* ------------------------------------------------------------------------- */
/* Model selection along the λ path (Section 3.3)    */
/* ------------------------------------------------------------------------- */

/* Degrees of freedom: ν = tr(A_J (A_JᵀA_J + λ2 I_r)⁻¹ A_Jᵀ) = tr((G + λ2 I)⁻¹ G),
 * G = A_JᵀA_J; computed with the textbook Cholesky of G + λ2 I and r column solves. */
double orc_dof(const double* A, i64 m, const i64* J, i64 r, double l2) {
  if (r == 0) return 0.0;
  double* G = (double*)malloc(sizeof(double) * (size_t)(r * r));
  double* L = (double*)malloc(sizeof(double) * (size_t)(r * r));
  double* c = (double*)malloc(sizeof(double) * (size_t)r);
  for (i64 b = 0; b < r; ++b)
    for (i64 a = 0; a < r; ++a) {
      double s = 0.0;
      for (i64 k = 0; k < m; ++k) s += A[k + J[a] * m] * A[k + J[b] * m];
      G[a + b * r] = s;
      L[a + b * r] = s + (a == b ? l2 : 0.0);
    }
  double nu = NAN;
  if (orc_chol(L, r) == 0) {
    nu = 0.0;
    for (i64 j = 0; j < r; ++j) { /* column j of (G + λ2 I)⁻¹ G, keep entry j */
      for (i64 a = 0; a < r; ++a) c[a] = G[a + j * r];
      orc_chol_solve(L, r, c);
      nu += c[j];
    }
  }
  free(G); free(L); free(c);
  return nu;
}

/* De-biasing by least squares on the selected features: v = argmin ‖A_J v − b‖²
 * via the normal equations (Cholesky of A_JᵀA_J); *rss = ‖b − A_J v‖².  0 ok, −1 singular. */
int orc_ols(const double* A, const double* b, i64 m, const i64* J, i64 r, double* v, double* rss) {
  double* G = (double*)malloc(sizeof(double) * (size_t)((r > 0 ? r : 1) * (r > 0 ? r : 1)));
  int rc = 0;
  for (i64 bb = 0; bb < r; ++bb)
    for (i64 a = 0; a < r; ++a) {
      double s = 0.0;
      for (i64 k = 0; k < m; ++k) s += A[k + J[a] * m] * A[k + J[bb] * m];
      G[a + bb * r] = s;
    }
  for (i64 a = 0; a < r; ++a) {
    double s = 0.0;
    for (i64 k = 0; k < m; ++k) s += A[k + J[a] * m] * b[k];
    v[a] = s;
  }
  if (r > 0) {
    if (orc_chol(G, r) != 0) rc = -1;
    else orc_chol_solve(G, r, v);
  }
  double q = 0.0;
  for (i64 k = 0; k < m; ++k) {
    double e = b[k];
    for (i64 a = 0; a < r; ++a) e -= A[k + J[a] * m] * v[a];
    q += e * e;
  }
  *rss = q;
  free(G);
  return rc;
}

/* Eq. (21): gcv = m⁻¹ rss / (1 − ν/m)²;  e-bic = log(rss/m) + (ν/m)(log m + log n). */
void orc_criteria(double rss, double nu, i64 m, i64 n, double* gcv, double* ebic) {
  const double dm = (double)m;
  const double f = 1.0 - nu / dm;
  *gcv = (rss / dm) / (f * f);
  *ebic = log(rss / dm) + (nu / dm) * (log(dm) + log((double)n));
}

/* All model-selection quantities of a solution x: out = [r, ν, rss, gcv, ebic];
 * xdb (n, nullable) = de-biased coefficients (OLS on supp x, zero elsewhere). */
int orc_model_select(const double* A, const double* b, i64 m, i64 n, const double* x, double l2, double* xdb,
                     double* out) {
  i64* J = (i64*)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
  i64 r = 0;
  for (i64 i = 0; i < n; ++i)
    if (x[i] != 0.0) J[r++] = i;
  double* v = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  double rss = 0.0;
  int rc = orc_ols(A, b, m, J, r, v, &rss);
  double nu = orc_dof(A, m, J, r, l2);
  double gcv, ebic;
  orc_criteria(rss, nu, m, n, &gcv, &ebic);
  out[0] = (double)r; out[1] = nu; out[2] = rss; out[3] = gcv; out[4] = ebic;
  if (xdb) {
    for (i64 i = 0; i < n; ++i) xdb[i] = 0.0;
    for (i64 a = 0; a < r; ++a) xdb[J[a]] = v[a];
  }
  free(J); free(v);
  return rc;
}
