/*
 * rid_oracle.c — CPU ORACLE for the randomized interpolative decomposition (arXiv 1205.3830).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library. The product path (paper_1205_3830_b200/) never
 * links, imports or executes anything under oracle/, and shares no code with it.
 *
 * Plain, slow, obviously correct complex128 arithmetic in IEEE binary64, written step by step in
 * the paper's order and notation. Compiled with -O2 -ffp-contract=off (no contraction, no
 * fast-math); every fused multiply-add is an explicit fma() call where docs/RNG.md demands one.
 * OpenMP parallelises over independent output columns (or output rows) only, so every output
 * element is accumulated in one fixed order regardless of the thread count.
 *
 * Layout: complex matrices are column-major arrays of interleaved (re, im) doubles; element
 * (i, j) of a matrix with leading dimension ld is at doubles [2*(i + j*ld)], [2*(i + j*ld) + 1].
 *
 * Functions and the passages they follow:
 *   orc_philox4x32_10   docs/RNG.md §1 ("rudimentary probabilistic functions")
 *   orc_rid_ln, orc_rid_sincos2pi, orc_normal     docs/RNG.md §3–4 (configs: parts N(0,1/2))
 *   orc_generate        docs/RNG.md §5; PAPER.md:112 (§3.3, A = BP of Gaussian factors)
 *   orc_sketch          Y = R·A, north_star Gaussian sketch; licence PAPER.md:97 (§2)
 *   orc_pivoted_cgs2    PAPER.md:82-86 (§2, Eqs. 8–9) + PAPER.md:108 (§3.2, CGS "with iteration")
 *   orc_backsolve       PAPER.md:88-93 (§2, Eqs. 10–11: R2 = R1 T, P = [I T])
 *   orc_error_estimate  PAPER.md:262-277 (Table 5, ||A − BP||_2), readings R15/R16
 *   orc_error_bound     PAPER.md:60-63 (§2, Eq. 3)
 *   orc_srft_plan, orc_srft_apply   PAPER.md:69-80 (§2, Eqs. 4–7: Y = S F D A), docs/RNG.md §7
 *
 * Parity-pinned by tests/test_oracle_*.py (curand Philox, libm, LAPACK ZGEQP3, scipy ID,
 * lstsq, dense SVD, brute force, closed forms).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define RID_OK 0
#define RID_EINVAL 1
#define RID_ERANK 2
#define RID_ESINGULAR 3
#define RID_ENOMEM 4

/* ------------------------------------------------------------------------------------------ */
/* docs/RNG.md §1 — Philox4x32-10                                                              */
/* ------------------------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    if (round < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* docs/RNG.md §3 — u = ((w >> 12) + 0.5) * 2^-52 */
static double uniform_from(uint32_t lo, uint32_t hi) {
  uint64_t w = ((uint64_t)hi << 32) | (uint64_t)lo;
  double v = (double)(w >> 12);
  v = v + 0.5;
  return v * 0x1p-52;
}

/* docs/RNG.md §4.1 — ln u for u in (0, 1), using only + - * / and fma */
double orc_rid_ln(double u) {
  int e;
  double f = frexp(u, &e); /* u = f * 2^e with f in [0.5, 1) */
  f = f * 2.0;             /* f in [1, 2), exact */
  e = e - 1;
  if (f > 0x1.6a09e667f3bcdp+0) { f = f * 0.5; e = e + 1; }
  double s = (f - 1.0) / (f + 1.0);
  double z = s * s;
  double P = 1.0 / 19.0;                 /* c9 */
  P = fma(P, z, 1.0 / 17.0);             /* c8 */
  P = fma(P, z, 1.0 / 15.0);             /* c7 */
  P = fma(P, z, 1.0 / 13.0);             /* c6 */
  P = fma(P, z, 1.0 / 11.0);             /* c5 */
  P = fma(P, z, 1.0 / 9.0);              /* c4 */
  P = fma(P, z, 1.0 / 7.0);              /* c3 */
  P = fma(P, z, 1.0 / 5.0);              /* c2 */
  P = fma(P, z, 1.0 / 3.0);              /* c1 */
  double q = z * P;
  double s2 = s + s;
  double lnf = fma(s2, q, s2);
  double de = (double)e;
  double hi = de * 0x1.62e42fee00000p-1;
  double lo = fma(de, 0x1.a39ef35793c76p-33, lnf);
  return hi + lo;
}

/* docs/RNG.md §4.3 — (cos 2πu, sin 2πu) */
void orc_rid_sincos2pi(double u, double* c_out, double* s_out) {
  double t = 4.0 * u;
  double q = nearbyint(t); /* default rounding mode: round half to even */
  double r = t - q;
  double x = r * 0x1.921fb54442d18p+0;
  double x2 = x * x;
  /* sin: S_j = (-1)^j / (2j+1)! */
  double Ps = -1.0 / 1307674368000.0;    /* S7 = -1/15! */
  Ps = fma(Ps, x2, 1.0 / 6227020800.0);  /* S6 = +1/13! */
  Ps = fma(Ps, x2, -1.0 / 39916800.0);   /* S5 = -1/11! */
  Ps = fma(Ps, x2, 1.0 / 362880.0);      /* S4 = +1/9!  */
  Ps = fma(Ps, x2, -1.0 / 5040.0);       /* S3 = -1/7!  */
  Ps = fma(Ps, x2, 1.0 / 120.0);         /* S2 = +1/5!  */
  Ps = fma(Ps, x2, -1.0 / 6.0);          /* S1 = -1/3!  */
  double xs = x * x2;
  double sinx = fma(xs, Ps, x);
  /* cos: C_j = (-1)^j / (2j)! */
  double Pc = 1.0 / 20922789888000.0;    /* C8 = +1/16! */
  Pc = fma(Pc, x2, -1.0 / 87178291200.0); /* C7 = -1/14! */
  Pc = fma(Pc, x2, 1.0 / 479001600.0);   /* C6 = +1/12! */
  Pc = fma(Pc, x2, -1.0 / 3628800.0);    /* C5 = -1/10! */
  Pc = fma(Pc, x2, 1.0 / 40320.0);       /* C4 = +1/8!  */
  Pc = fma(Pc, x2, -1.0 / 720.0);        /* C3 = -1/6!  */
  Pc = fma(Pc, x2, 1.0 / 24.0);          /* C2 = +1/4!  */
  Pc = fma(Pc, x2, -1.0 / 2.0);          /* C1 = -1/2!  */
  double cosx = fma(x2, Pc, 1.0);
  int quadrant = ((int)q) & 3;
  switch (quadrant) {
    case 0: *c_out = cosx; *s_out = sinx; break;
    case 1: *c_out = -sinx; *s_out = cosx; break;
    case 2: *c_out = -cosx; *s_out = -sinx; break;
    default: *c_out = sinx; *s_out = -cosx; break;
  }
}

/* docs/RNG.md §4 — N(seed, s, i, j) */
void orc_normal(uint64_t seed, uint32_t s, uint32_t i, uint32_t j, double out[2]) {
  uint32_t ctr[4] = {i, j, s, 0u};
  uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
  uint32_t x[4];
  orc_philox4x32_10(ctr, key, x);
  double u1 = uniform_from(x[0], x[1]);
  double u2 = uniform_from(x[2], x[3]);
  double rho = sqrt(-orc_rid_ln(u1));
  double c, sn;
  orc_rid_sincos2pi(u2, &c, &sn);
  out[0] = rho * c;
  out[1] = rho * sn;
}

/* Fill a rows x cols block (column-major, leading dim ld) with N(seed, s, row0 + i, col0 + j). */
void orc_normal_matrix(uint64_t seed, uint32_t s, int64_t rows, int64_t cols, int64_t row0,
                       int64_t col0, double* out, int64_t ld) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i)
      orc_normal(seed, s, (uint32_t)(row0 + i), (uint32_t)(col0 + j), &out[2 * (i + j * ld)]);
}

/* ------------------------------------------------------------------------------------------ */
/* docs/RNG.md §5 — A[:, col0:col0+n_loc] = X · Y0[:, shard] + noise · E[:, shard]             */
/* ------------------------------------------------------------------------------------------ */
int orc_generate(uint64_t seed, int64_t m, int64_t n, int64_t k, double noise, int64_t col0,
                 int64_t n_loc, double* A, int64_t lda) {
  if (m < 1 || n < 1 || k < 1 || k > m || k > n || col0 < 0 || n_loc < 0 || col0 + n_loc > n ||
      lda < m)
    return RID_EINVAL;
  double* X = (double*)malloc(sizeof(double) * 2 * (size_t)m * (size_t)k);
  if (!X) return RID_ENOMEM;
  orc_normal_matrix(seed, 1u, m, k, 0, 0, X, m); /* X: m x k, stream 1 */
#pragma omp parallel
  {
    double* y = (double*)malloc(sizeof(double) * 2 * (size_t)k);
#pragma omp for schedule(static)
    for (int64_t jj = 0; jj < n_loc; ++jj) {
      int64_t j = col0 + jj;
      for (int64_t t = 0; t < k; ++t) orc_normal(seed, 2u, (uint32_t)t, (uint32_t)j, &y[2 * t]);
      for (int64_t i = 0; i < m; ++i) {
        double acc_re = 0.0, acc_im = 0.0;
        for (int64_t t = 0; t < k; ++t) {
          double xr = X[2 * (i + t * m)], xi = X[2 * (i + t * m) + 1];
          double yr = y[2 * t], yi = y[2 * t + 1];
          acc_re = fma(xr, yr, acc_re);
          acc_re = fma(-xi, yi, acc_re);
          acc_im = fma(xi, yr, acc_im);
          acc_im = fma(xr, yi, acc_im);
        }
        if (noise != 0.0) {
          double e[2];
          orc_normal(seed, 3u, (uint32_t)i, (uint32_t)j, e);
          acc_re = fma(noise, e[0], acc_re);
          acc_im = fma(noise, e[1], acc_im);
        }
        A[2 * (i + jj * lda)] = acc_re;
        A[2 * (i + jj * lda) + 1] = acc_im;
      }
    }
    free(y);
  }
  free(X);
  return RID_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Gaussian sketch Y = R · A (R: l x m, R(r, i) = N(seed, stream, r, i)); ascending i,         */
/* the fma MAC form of docs/RNG.md §5/§6. North star; PAPER.md:97 licenses the substitution.  */
/* ------------------------------------------------------------------------------------------ */
int orc_sketch(uint64_t seed, uint32_t stream, int64_t l, int64_t m, int64_t n_loc,
               const double* A, int64_t lda, double* Y, int64_t ldy) {
  if (l < 1 || m < 1 || n_loc < 0 || lda < m || ldy < l) return RID_EINVAL;
  double* R = (double*)malloc(sizeof(double) * 2 * (size_t)l * (size_t)m);
  if (!R) return RID_ENOMEM;
  orc_normal_matrix(seed, stream, l, m, 0, 0, R, l); /* column-major: R(:, i) contiguous */
#pragma omp parallel
  {
    double* acc = (double*)malloc(sizeof(double) * 2 * (size_t)l);
#pragma omp for schedule(static)
    for (int64_t j = 0; j < n_loc; ++j) {
      for (int64_t r = 0; r < 2 * l; ++r) acc[r] = 0.0;
      for (int64_t i = 0; i < m; ++i) {
        double ar = A[2 * (i + j * lda)], ai = A[2 * (i + j * lda) + 1];
        const double* Rc = &R[2 * i * l];
        for (int64_t r = 0; r < l; ++r) { /* each Y(r, j) still accumulates alone, ascending i */
          double rr = Rc[2 * r], ri = Rc[2 * r + 1];
          double yr = acc[2 * r], yi = acc[2 * r + 1];
          yr = fma(rr, ar, yr);
          yr = fma(-ri, ai, yr);
          yi = fma(ri, ar, yi);
          yi = fma(rr, ai, yi);
          acc[2 * r] = yr;
          acc[2 * r + 1] = yi;
        }
      }
      for (int64_t r = 0; r < l; ++r) {
        Y[2 * (r + j * ldy)] = acc[2 * r];
        Y[2 * (r + j * ldy) + 1] = acc[2 * r + 1];
      }
    }
    free(acc);
  }
  free(R);
  return RID_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Pivoted classical Gram-Schmidt with reorthogonalisation (CGS2), PAPER.md:82-86 + :108.      */
/* Greedy max residual 2-norm pivot, ties -> lowest index (reading R8), exact norm recompute    */
/* every step (R11), rank failure below 1e-13 * max initial norm (R13). Outputs J (pivot        */
/* order), R = Q^H Y (k x n, original column order), resid_norms[j] = nu_p at step j and        */
/* tie_margins[j] = (nu_(1) - nu_(2)) / nu_(1) (R18; +inf when only one candidate).             */
/* Returns RID_OK, or RID_ERANK with *rank_achieved set.                                        */
/* ------------------------------------------------------------------------------------------ */
static double col_norm(const double* w, int64_t l) {
  double s = 0.0;
  for (int64_t r = 0; r < l; ++r) s += w[2 * r] * w[2 * r] + w[2 * r + 1] * w[2 * r + 1];
  return sqrt(s);
}

int orc_pivoted_cgs2(int64_t l, int64_t n, int64_t k, const double* Y, int64_t ldy, int64_t* J,
                     double* R, int64_t ldr, double* resid_norms, double* tie_margins,
                     int64_t* rank_achieved) {
  if (k < 1 || k > l || k > n || ldy < l || ldr < k) return RID_EINVAL;
  double* W = (double*)malloc(sizeof(double) * 2 * (size_t)l * (size_t)n);
  double* Q = (double*)malloc(sizeof(double) * 2 * (size_t)l * (size_t)k);
  double* nu = (double*)malloc(sizeof(double) * (size_t)n);
  char* chosen = (char*)calloc((size_t)n, 1);
  double* q = (double*)malloc(sizeof(double) * 2 * (size_t)l);
  double* coef = (double*)malloc(sizeof(double) * 2 * (size_t)k);
  if (!W || !Q || !nu || !chosen || !q || !coef) {
    free(W); free(Q); free(nu); free(chosen); free(q); free(coef);
    return RID_ENOMEM;
  }
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < l; ++r) {
      W[2 * (r + c * l)] = Y[2 * (r + c * ldy)];
      W[2 * (r + c * l) + 1] = Y[2 * (r + c * ldy) + 1];
    }
  double nu0max = 0.0;
  for (int64_t c = 0; c < n; ++c) {
    double v = col_norm(&Y[2 * c * ldy], l);
    if (v > nu0max) nu0max = v;
  }
  int status = RID_OK;
  if (rank_achieved) *rank_achieved = 0;
  for (int64_t j = 0; j < k; ++j) {
    /* 1. exact residual norms of every unchosen column */
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c) nu[c] = chosen[c] ? -1.0 : col_norm(&W[2 * c * l], l);
    /* 2. p = argmax, ties -> lowest index; second-best for the tie margin */
    int64_t p = -1;
    double best = -1.0, second = -1.0;
    for (int64_t c = 0; c < n; ++c) {
      if (chosen[c]) continue;
      if (nu[c] > best) { second = best; best = nu[c]; p = c; }
      else if (nu[c] > second) second = nu[c];
    }
    if (resid_norms) resid_norms[j] = best;
    if (tie_margins) tie_margins[j] = (second < 0.0) ? INFINITY : (best - second) / best;
    /* 3. rank failure */
    if (!(best >= 1e-13 * nu0max) || best == 0.0) { status = RID_ERANK; break; }
    /* 4. q = W[:, p], two classical GS passes against q_0..q_{j-1} ("twice is enough") */
    for (int64_t r = 0; r < 2 * l; ++r) q[r] = W[2 * p * l + r];
    for (int pass = 0; pass < 2; ++pass) {
      for (int64_t t = 0; t < j; ++t) { /* coef_t = q_t^H q (all from the same q: classical) */
        double cr = 0.0, ci = 0.0;
        const double* qt = &Q[2 * t * l];
        for (int64_t r = 0; r < l; ++r) {
          cr += qt[2 * r] * q[2 * r] + qt[2 * r + 1] * q[2 * r + 1];
          ci += qt[2 * r] * q[2 * r + 1] - qt[2 * r + 1] * q[2 * r];
        }
        coef[2 * t] = cr;
        coef[2 * t + 1] = ci;
      }
      for (int64_t t = 0; t < j; ++t) { /* q <- q - q_t coef_t */
        const double* qt = &Q[2 * t * l];
        double cr = coef[2 * t], ci = coef[2 * t + 1];
        for (int64_t r = 0; r < l; ++r) {
          q[2 * r] -= qt[2 * r] * cr - qt[2 * r + 1] * ci;
          q[2 * r + 1] -= qt[2 * r] * ci + qt[2 * r + 1] * cr;
        }
      }
    }
    /* 5. normalise */
    double qn = col_norm(q, l);
    for (int64_t r = 0; r < 2 * l; ++r) Q[2 * j * l + r] = q[r] / qn;
    chosen[p] = 1;
    J[j] = p;
    if (rank_achieved) *rank_achieved = j + 1;
    /* 6. project q_j out of every unchosen column */
    const double* qj = &Q[2 * j * l];
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c) {
      if (chosen[c]) continue;
      double* w = &W[2 * c * l];
      double cr = 0.0, ci = 0.0;
      for (int64_t r = 0; r < l; ++r) {
        cr += qj[2 * r] * w[2 * r] + qj[2 * r + 1] * w[2 * r + 1];
        ci += qj[2 * r] * w[2 * r + 1] - qj[2 * r + 1] * w[2 * r];
      }
      for (int64_t r = 0; r < l; ++r) {
        w[2 * r] -= qj[2 * r] * cr - qj[2 * r + 1] * ci;
        w[2 * r + 1] -= qj[2 * r] * ci + qj[2 * r + 1] * cr;
      }
    }
  }
  if (status == RID_OK && R) {
    /* R = Q^H Y, computed directly (R11 = R[:, J] is upper triangular up to rounding) */
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c) {
      const double* y = &Y[2 * c * ldy];
      for (int64_t t = 0; t < k; ++t) {
        const double* qt = &Q[2 * t * l];
        double cr = 0.0, ci = 0.0;
        for (int64_t r = 0; r < l; ++r) {
          cr += qt[2 * r] * y[2 * r] + qt[2 * r + 1] * y[2 * r + 1];
          ci += qt[2 * r] * y[2 * r + 1] - qt[2 * r + 1] * y[2 * r];
        }
        R[2 * (t + c * ldr)] = cr;
        R[2 * (t + c * ldr) + 1] = ci;
      }
    }
  }
  free(W); free(Q); free(nu); free(chosen); free(q); free(coef);
  return status;
}

/* ------------------------------------------------------------------------------------------ */
/* Back-substitution R11 T = R12 and P = [I T] in original column order (PAPER.md:88-93,       */
/* Eqs. 10–11). Only the upper triangle of R11 = R[:, J] is read.             */
/* P is k x n (ldp >= k): P[:, J_t] = e_t exactly, P[:, c] = t(c) for c not in J.               */
/* ------------------------------------------------------------------------------------------ */
int orc_backsolve(int64_t k, int64_t n, const double* R, int64_t ldr, const int64_t* J, double* P,
                  int64_t ldp, int64_t* singular_index) {
  if (k < 1 || k > n || ldr < k || ldp < k) return RID_EINVAL;
  char* isJ = (char*)calloc((size_t)n, 1);
  if (!isJ) return RID_ENOMEM;
  double dmax = 0.0;
  for (int64_t t = 0; t < k; ++t) {
    if (J[t] < 0 || J[t] >= n || isJ[J[t]]) { free(isJ); return RID_EINVAL; }
    isJ[J[t]] = 1;
    const double* d = &R[2 * (t + J[t] * ldr)];
    double a = sqrt(d[0] * d[0] + d[1] * d[1]);
    if (a > dmax) dmax = a;
  }
  for (int64_t t = 0; t < k; ++t) {
    const double* d = &R[2 * (t + J[t] * ldr)];
    double a = sqrt(d[0] * d[0] + d[1] * d[1]);
    if (a < 1e-13 * dmax) {
      if (singular_index) *singular_index = t;
      free(isJ);
      return RID_ESINGULAR;
    }
  }
  /* R11(i, s) = R(i, J[s]) */
#define R11RE(i, s) R[2 * ((i) + J[s] * ldr)]
#define R11IM(i, s) R[2 * ((i) + J[s] * ldr) + 1]
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n; ++c) {
    double* pc = &P[2 * c * ldp];
    if (isJ[c]) {
      for (int64_t t = 0; t < k; ++t) { pc[2 * t] = 0.0; pc[2 * t + 1] = 0.0; }
      continue;
    }
    const double* rc = &R[2 * c * ldr];
    for (int64_t i = k - 1; i >= 0; --i) {
      double ar = rc[2 * i], ai = rc[2 * i + 1];
      for (int64_t s = i + 1; s < k; ++s) {
        double br = R11RE(i, s), bi = R11IM(i, s);
        double tr = pc[2 * s], ti = pc[2 * s + 1];
        ar -= br * tr - bi * ti;
        ai -= br * ti + bi * tr;
      }
      double dr = R11RE(i, i), di = R11IM(i, i);
      double den = dr * dr + di * di;
      pc[2 * i] = (ar * dr + ai * di) / den;
      pc[2 * i + 1] = (ai * dr - ar * di) / den;
    }
  }
  for (int64_t t = 0; t < k; ++t) {
    double* pc = &P[2 * J[t] * ldp];
    pc[2 * t] = 1.0; /* exact identity block */
  }
#undef R11RE
#undef R11IM
  free(isJ);
  return RID_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Compensated ("doubled working precision") building blocks for the estimator: TwoSum,         */
/* TwoProd via fma, and the Dot2 accumulator of Ogita, Rump & Oishi (2005).                     */
/* ------------------------------------------------------------------------------------------ */
typedef struct { double s, c; } acc2; /* value = s + c (c collects the error terms) */

static inline void acc2_add_prod(acc2* a, double x, double y) {
  double p = x * y;
  double pe = fma(x, y, -p);  /* TwoProd: x*y = p + pe exactly */
  double s = a->s + p;        /* TwoSum(a->s, p) */
  double bv = s - a->s;
  double se = (a->s - (s - bv)) + (p - bv);
  a->s = s;
  a->c += pe + se;
}
static inline void acc2_add(acc2* a, double x) {
  double s = a->s + x;
  double bv = s - a->s;
  double se = (a->s - (s - bv)) + (x - bv);
  a->s = s;
  a->c += se;
}
static inline double acc2_val(const acc2* a) { return a->s + a->c; }

/* complex accumulator: re and im as separate acc2 */
typedef struct { acc2 re, im; } cacc2;
/* acc += x * y (complex); conj_x: use conj(x) */
static inline void cacc2_mac(cacc2* a, double xr, double xi, double yr, double yi, int conj_x) {
  if (conj_x) xi = -xi;
  acc2_add_prod(&a->re, xr, yr);
  acc2_add_prod(&a->re, -xi, yi);
  acc2_add_prod(&a->im, xr, yi);
  acc2_add_prod(&a->im, xi, yr);
}

/* ------------------------------------------------------------------------------------------ */
/* Randomised power-iteration estimate of ||A - B P||_2, B = A[:, J] (PAPER.md:262-277,          */
/* Table 5; R15/R16). x0(j) = N(seed, 5, j, 0), normalised.  */
/* q fixed iterations of  y = A x − B (P x);  z = A^H y − P^H (B^H y);  est = sqrt(||z||);       */
/* x = z / ||z||.  Every dot product is compensated; P x and B^H y are kept as (s + c) until     */
/* they are multiplied back; y and z are rounded once.  Returns est in *est.                     */
/* ------------------------------------------------------------------------------------------ */
int orc_error_estimate(int64_t m, int64_t n, const double* A, int64_t lda, const int64_t* J,
                       int64_t k, const double* P, int64_t ldp, int q, uint64_t seed,
                       double* est) {
  if (m < 1 || n < 1 || k < 1 || k > n || lda < m || ldp < k || q < 1) return RID_EINVAL;
  double* x = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  double* z = (double*)malloc(sizeof(double) * 2 * (size_t)n);
  double* y = (double*)malloc(sizeof(double) * 2 * (size_t)m);
  double* ux = (double*)malloc(sizeof(double) * 4 * (size_t)k); /* P x as (hi, lo) re, im */
  double* sb = (double*)malloc(sizeof(double) * 4 * (size_t)k); /* B^H y as (hi, lo) */
  if (!x || !z || !y || !ux || !sb) {
    free(x); free(z); free(y); free(ux); free(sb);
    return RID_ENOMEM;
  }
  for (int64_t j = 0; j < n; ++j) orc_normal(seed, 5u, (uint32_t)j, 0u, &x[2 * j]);
  {
    acc2 nn = {0.0, 0.0};
    for (int64_t j = 0; j < n; ++j) {
      acc2_add_prod(&nn, x[2 * j], x[2 * j]);
      acc2_add_prod(&nn, x[2 * j + 1], x[2 * j + 1]);
    }
    double nx = sqrt(acc2_val(&nn));
    for (int64_t j = 0; j < 2 * n; ++j) x[j] = x[j] / nx;
  }
  double s_est = 0.0;
  for (int it = 0; it < q; ++it) {
    /* u = P x (k-vector), kept as s + c */
    for (int64_t t = 0; t < k; ++t) {
      cacc2 a = {{0.0, 0.0}, {0.0, 0.0}};
      for (int64_t j = 0; j < n; ++j)
        cacc2_mac(&a, P[2 * (t + j * ldp)], P[2 * (t + j * ldp) + 1], x[2 * j], x[2 * j + 1], 0);
      ux[4 * t + 0] = a.re.s; ux[4 * t + 1] = a.re.c;
      ux[4 * t + 2] = a.im.s; ux[4 * t + 3] = a.im.c;
    }
    /* y = A x - B u, row-parallel; each y_i accumulated in one fixed order */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
      cacc2 a = {{0.0, 0.0}, {0.0, 0.0}};
      for (int64_t j = 0; j < n; ++j)
        cacc2_mac(&a, A[2 * (i + j * lda)], A[2 * (i + j * lda) + 1], x[2 * j], x[2 * j + 1], 0);
      for (int64_t t = 0; t < k; ++t) {
        const double* b = &A[2 * (i + J[t] * lda)];
        /* subtract b * (u_s + u_c): the (s) part exactly via TwoProd, the (c) part plainly */
        cacc2_mac(&a, -b[0], -b[1], ux[4 * t + 0], ux[4 * t + 2], 0);
        cacc2_mac(&a, -b[0], -b[1], ux[4 * t + 1], ux[4 * t + 3], 0);
      }
      y[2 * i] = acc2_val(&a.re);
      y[2 * i + 1] = acc2_val(&a.im);
    }
    /* s = B^H y (k-vector), kept as s + c */
    for (int64_t t = 0; t < k; ++t) {
      cacc2 a = {{0.0, 0.0}, {0.0, 0.0}};
      const double* b = &A[2 * J[t] * lda];
      for (int64_t i = 0; i < m; ++i) cacc2_mac(&a, b[2 * i], b[2 * i + 1], y[2 * i], y[2 * i + 1], 1);
      sb[4 * t + 0] = a.re.s; sb[4 * t + 1] = a.re.c;
      sb[4 * t + 2] = a.im.s; sb[4 * t + 3] = a.im.c;
    }
    /* z = A^H y - P^H s, column-parallel */
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) {
      cacc2 a = {{0.0, 0.0}, {0.0, 0.0}};
      const double* aj = &A[2 * j * lda];
      for (int64_t i = 0; i < m; ++i) cacc2_mac(&a, aj[2 * i], aj[2 * i + 1], y[2 * i], y[2 * i + 1], 1);
      for (int64_t t = 0; t < k; ++t) {
        double pr = P[2 * (t + j * ldp)], pi = P[2 * (t + j * ldp) + 1];
        /* subtract conj(p) * (s_s + s_c) */
        cacc2_mac(&a, -pr, pi, sb[4 * t + 0], sb[4 * t + 2], 0);
        cacc2_mac(&a, -pr, pi, sb[4 * t + 1], sb[4 * t + 3], 0);
      }
      z[2 * j] = acc2_val(&a.re);
      z[2 * j + 1] = acc2_val(&a.im);
    }
    acc2 nn = {0.0, 0.0};
    for (int64_t j = 0; j < n; ++j) {
      acc2_add_prod(&nn, z[2 * j], z[2 * j]);
      acc2_add_prod(&nn, z[2 * j + 1], z[2 * j + 1]);
    }
    double nz = sqrt(acc2_val(&nn));
    s_est = sqrt(nz);
    if (nz == 0.0) break;
    for (int64_t j = 0; j < 2 * n; ++j) x[j] = z[j] / nz;
  }
  *est = s_est;
  free(x); free(z); free(y); free(ux); free(sb);
  return RID_OK;
}

/* Eq. (3) right-hand side: 50 sqrt(mn) (1/eps)^(1/k) sigma_{k+1}. */
double orc_error_bound(int64_t m, int64_t n, int64_t k, double eps, double sigma_kp1) {
  return 50.0 * sqrt((double)m * (double)n) * pow(1.0 / eps, 1.0 / (double)k) * sigma_kp1;
}

/* sigma_{k+1} noise floor sqrt(2 min(m, n)) * delta (§3.3). */
double orc_noise_floor(int64_t m, int64_t n, double delta) {
  double mn = (double)(m < n ? m : n);
  return sqrt(2.0 * mn) * delta;
}

/* ------------------------------------------------------------------------------------------ */
/* SRFT randomisation Y = S F D A (§2, Eqs. 4–7; docs/RNG.md §7).             */
/* Plan: phases d_i = e^{2 pi i phi_i}, phi_i = u1 of Philox (i, 0, s_phase, 0); samples         */
/* s_k = x0 & (m-1) of Philox (k, 0, s_sample, 0). m must be a power of two.                     */
/* ------------------------------------------------------------------------------------------ */
static int is_pow2(int64_t m) { return m > 0 && (m & (m - 1)) == 0; }

int orc_srft_plan(uint64_t seed, uint32_t s_phase, uint32_t s_sample, int64_t m, int64_t l,
                  double* d, int64_t* samples) {
  if (!is_pow2(m) || l < 1 || m > ((int64_t)1 << 32)) return RID_EINVAL;
  const uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
  for (int64_t i = 0; i < m; ++i) {
    uint32_t ctr[4] = {(uint32_t)i, 0u, s_phase, 0u}, x[4];
    orc_philox4x32_10(ctr, key, x);
    double c, s;
    orc_rid_sincos2pi(uniform_from(x[0], x[1]), &c, &s);
    d[2 * i] = c;
    d[2 * i + 1] = s;
  }
  for (int64_t k = 0; k < l; ++k) {
    uint32_t ctr[4] = {(uint32_t)k, 0u, s_sample, 0u}, x[4];
    orc_philox4x32_10(ctr, key, x);
    samples[k] = (int64_t)(x[0] & (uint32_t)(m - 1));
  }
  return RID_OK;
}

/* Y(k, c) = sum_{i ascending} F[s_k, i] * (d_i * A(i, c)), F[t, i] = e^{-2 pi i (t i mod m) / m}
 * (Eq. 6, unnormalised) evaluated through the spec'd sincos on u = ((t i) mod m) / m (exact). The
 * plan (d, samples) is an input so tests can pin the transform with chosen plans. */
int orc_srft_apply(const double* d, const int64_t* samples, int64_t l, int64_t m, int64_t n_loc,
                   const double* A, int64_t lda, double* Y, int64_t ldy) {
  if (!is_pow2(m) || l < 1 || n_loc < 0 || lda < m || ldy < l) return RID_EINVAL;
  double* tw = (double*)malloc(sizeof(double) * 2 * (size_t)m); /* F entries e^{-2 pi i t / m} */
  if (!tw) return RID_ENOMEM;
  for (int64_t t = 0; t < m; ++t) {
    double c, s;
    orc_rid_sincos2pi((double)t / (double)m, &c, &s);
    tw[2 * t] = c;
    tw[2 * t + 1] = -s;
  }
#pragma omp parallel
  {
    double* b = (double*)malloc(sizeof(double) * 2 * (size_t)m);
#pragma omp for schedule(static)
    for (int64_t c = 0; c < n_loc; ++c) {
      const double* a = &A[2 * c * lda];
      for (int64_t i = 0; i < m; ++i) { /* b = D a */
        const double dr = d[2 * i], di = d[2 * i + 1], ar = a[2 * i], ai = a[2 * i + 1];
        b[2 * i] = fma(dr, ar, -(di * ai));
        b[2 * i + 1] = fma(di, ar, dr * ai);
      }
      for (int64_t k = 0; k < l; ++k) {
        const uint64_t sk = (uint64_t)samples[k];
        double yr = 0.0, yi = 0.0;
        for (int64_t i = 0; i < m; ++i) {
          const uint64_t t = (sk * (uint64_t)i) & (uint64_t)(m - 1);
          const double wr = tw[2 * t], wi = tw[2 * t + 1];
          yr = fma(wr, b[2 * i], yr);
          yr = fma(-wi, b[2 * i + 1], yr);
          yi = fma(wi, b[2 * i], yi);
          yi = fma(wr, b[2 * i + 1], yi);
        }
        Y[2 * (k + c * ldy)] = yr;
        Y[2 * (k + c * ldy) + 1] = yi;
      }
    }
    free(b);
  }
  free(tw);
  return RID_OK;
}

int orc_set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
  return omp_get_max_threads();
#else
  (void)nthreads;
  return 1;
#endif
}
