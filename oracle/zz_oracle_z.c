/*
 * oracle/zz_oracle_z.c -- TEST INFRASTRUCTURE ONLY (same rules as oracle/zz_oracle.c:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load or call it; the product path shares no code, header or constant with it).
 *
 * What it computes.  All (or the selected) right generalized eigenvectors of a COMPLEX
 * pencil (S,T) in generalized complex Schur form: S and T upper triangular, T with a real
 * diagonal (the ZTGEVC analogue named as future work in PAPER.md:333; conventions of
 * LAPACK ZTGEVC).  For the eigenvalue (alpha, beta) = (S_jj, T_jj) the eigenvector z has
 * z_i = 0 for i > j, z_j = 1 before normalisation, and solves
 * (beta S - alpha T)(0:j,0:j) z = 0 (Lemma 1, with every block 1x1).
 *
 * How.  The same plain method as zz_oracle.c, one eigenvector at a time by scalar
 * column-oriented substitution, made robust with
 * ProtectUpdate / ProtectDivision and one int32 power-of-two exponent
 * per eigenvector.  Readings for complex entries (R18-R20):
 *   R18  (alpha, beta) = (S_jj, T_jj), both negated if T_jj < 0, then scaled by the exact
 *        power of two that puts max(beta, |Re alpha| + |Im alpha|) in [1/2, 1) (R2).
 *        Im T_jj != 0 is an error (-107; ZTGEVC's "P must have a real diagonal").
 *   R19  magnitudes are max(|Re|,|Im|); a complex product's parts are bounded by
 *        2 max|.| max|.|, so the ProtectUpdate bound of one solved row k is
 *        t = 2 (beta cmS[k] + (|Re alpha| + |Im alpha|) cmT[k]), cmS[k] = max_{i<k}
 *        max(|Re S_ik|, |Im S_ik|) (R6 with complex entries).
 *   R20  the pivot d_i = beta S_ii - alpha T_ii is replaced by smin =
 *        max(u (beta |S_ii|_1 + |alpha|_1 |T_ii|), smlnum) when |d_i|_1 < smin (R8), and
 *        divided by Smith's algorithm under ProtectDivision(max|w_i|, min(1, max|d_i|)/2)
 *        (R9's complex branch).
 * Normalisation as ZTGEVC: max_i (|Re z_i| + |Im z_i|) = 1; an indefinite eigenvalue
 * (alpha = beta = 0) gives e_j (R13).
 *
 * Parity status.  Pinned by tests/test_oracle_complex.py against LAPACK ZTGEVC (black box),
 * the real oracle on real triangular pencils, the m = 1 and m = 2 closed forms, long-double
 * unprotected substitution on a stress pencil, and residual invariants.  col_scale_exp is
 * implementation-defined ("parity unpinned"; only its invariants are checked).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ZO_U 0x1p-53
#define ZO_SMLNUM 0x1p-969
#define ZO_ERR_NONFINITE (-104)
#define ZO_ERR_CPLXDIAG (-107)
#define ZO_ERR_NOMEM (-102)

int zzo_protect_update(double y, double t, double x);   /* zz_oracle.c */
int zzo_protect_division(double b, double t);

typedef struct { double re, im; } zc;

static inline double zmax2(double x, double y) { return x > y ? x : y; }
static inline double zmin2(double x, double y) { return x < y ? x : y; }
static inline zc zmk(double re, double im) { zc z = {re, im}; return z; }
static inline double zabsm(zc z) { return zmax2(fabs(z.re), fabs(z.im)); }
static inline double zabs1(zc z) { return fabs(z.re) + fabs(z.im); }
static inline zc zmul(zc x, zc y) { return zmk(x.re * y.re - x.im * y.im, x.re * y.im + x.im * y.re); }
static inline zc zdivs(zc x, zc y) { /* Smith */
  if (fabs(y.re) >= fabs(y.im)) {
    double r = y.im / y.re, den = y.re + y.im * r;
    return zmk((x.re + x.im * r) / den, (x.im - x.re * r) / den);
  } else {
    double r = y.re / y.im, den = y.im + y.re * r;
    return zmk((x.re * r + x.im) / den, (x.im * r - x.re) / den);
  }
}

#define ZS(i, j) zmk(S[2 * ((size_t)(j) * (size_t)lds + (size_t)(i))], S[2 * ((size_t)(j) * (size_t)lds + (size_t)(i)) + 1])
#define ZT(i, j) zmk(T[2 * ((size_t)(j) * (size_t)ldt + (size_t)(i))], T[2 * ((size_t)(j) * (size_t)ldt + (size_t)(i)) + 1])

/* R18: normalised eigenvalue of row j; kind 2 = indefinite. */
int zzo_zeig(int m, const double* S, int lds, const double* T, int ldt, double* a, double* b,
             double* beta, int* kind) {
  for (int j = 0; j < m; ++j) {
    zc s = ZS(j, j), t = ZT(j, j);
    if (!isfinite(s.re) || !isfinite(s.im) || !isfinite(t.re) || !isfinite(t.im)) return ZO_ERR_NONFINITE;
    if (t.im != 0.0) return ZO_ERR_CPLXDIAG;
    double ar = s.re, ai = s.im, be = t.re;
    if (be < 0.0) { ar = -ar; ai = -ai; be = -be; }
    double h = zmax2(0.5 * be, 0.5 * fabs(ar) + 0.5 * fabs(ai));
    kind[j] = 0;
    if (h == 0.0) { kind[j] = 2; a[j] = b[j] = beta[j] = 0.0; continue; }
    int k;
    frexp(h, &k);
    a[j] = ldexp(ar, -(k + 1));
    b[j] = ldexp(ai, -(k + 1));
    beta[j] = ldexp(be, -(k + 1));
  }
  return 0;
}

typedef struct { zc* w; int e; int nscal; int npert; } zv;

static void zscale(zv* v, int r, int k) {
  if (k >= 0) return;
  for (int i = 0; i <= r; ++i) { v->w[i].re = ldexp(v->w[i].re, k); v->w[i].im = ldexp(v->w[i].im, k); }
  v->e += k;
  v->nscal++;
}

/* w_i <- w_i - (S_ik (beta x_k) - T_ik (alpha x_k)), i < k,
 * protected by ProtectUpdate with the R19 bound. */
static void zupdate_above(int k, const double* S, int lds, const double* T, int ldt,
                          const double* cmS, const double* cmT, zv* v, double a, double b,
                          double beta, int protect) {
  if (k == 0) return;
  if (protect) {
    double t = 2.0 * (beta * cmS[k] + (fabs(a) + fabs(b)) * cmT[k]);
    double wmax = 0.0;
    for (int i = 0; i < k; ++i) wmax = zmax2(wmax, zabsm(v->w[i]));
    zscale(v, k, zzo_protect_update(wmax, t, zabsm(v->w[k])));
  }
  zc x = v->w[k];
  zc u = zmk(beta * x.re, beta * x.im);     /* x D */
  zc al = zmul(zmk(a, b), x);               /* x B */
  for (int i = 0; i < k; ++i) {
    zc p = zmul(ZS(i, k), u), q = zmul(ZT(i, k), al);
    v->w[i].re = v->w[i].re - (p.re - q.re);
    v->w[i].im = v->w[i].im - (p.im - q.im);
  }
}

/* Row i: (beta S_ii - alpha T_ii) x_i = w_i (R20). */
static void zsolve_row(int i, const double* S, int lds, const double* T, int ldt, zv* v, int r,
                       double a, double b, double beta, int protect) {
  zc s = ZS(i, i);
  double t = ZT(i, i).re;
  zc d = zmk(beta * s.re - a * t, beta * s.im - b * t);
  double smin = zmax2(ZO_U * (beta * zabs1(s) + (fabs(a) + fabs(b)) * fabs(t)), ZO_SMLNUM);
  if (zabs1(d) < smin) { d = zmk(smin, 0.0); v->npert++; }
  if (protect) zscale(v, r, zzo_protect_division(zabsm(v->w[i]), 0.5 * zmin2(1.0, zabsm(d))));
  v->w[i] = zdivs(v->w[i], d);
}

/* S, T, X interleaved complex (re, im), column-major, leading dimensions in complex
 * elements.  X is m x n_sel; columns in eigenvalue order.  Returns 0 or a status. */
int zzo_ztgevc(int m, const double* S, int lds, const double* T, int ldt, const int* select,
               double* X, int ldx, int* col_scale_exp, int* stats, int protect, int nthreads) {
  if (m <= 0) return 0;
  double* a = (double*)malloc(sizeof(double) * 5 * (size_t)m);
  int* kind = (int*)malloc(sizeof(int) * 2 * (size_t)m);
  if (!a || !kind) { free(a); free(kind); return ZO_ERR_NOMEM; }
  double *b = a + m, *beta = a + 2 * m, *cmS = a + 3 * m, *cmT = a + 4 * m;
  int* colof = kind + m;
  int st = zzo_zeig(m, S, lds, T, ldt, a, b, beta, kind);
  if (st) { free(a); free(kind); return st; }
  int n = 0;
  for (int j = 0; j < m; ++j) colof[j] = (!select || select[j]) ? n++ : -1;
  for (int k = 0; k < m; ++k) {
    double ms = 0.0, mt = 0.0;
    for (int i = 0; i < k; ++i) { ms = zmax2(ms, zabsm(ZS(i, k))); mt = zmax2(mt, zabsm(ZT(i, k))); }
    cmS[k] = ms;
    cmT[k] = mt;
  }
  int s0 = 0, s1 = 0, s2 = 0, bad = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel reduction(+ : s0, s1, s2, bad)
#endif
  {
    zc* w = (zc*)malloc(sizeof(zc) * (size_t)m);
    if (!w) bad++;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
    for (int j = m - 1; j >= 0; --j) {
      if (!w || colof[j] < 0) continue;
      zv v = {w, 0, 0, 0};
      for (int i = 0; i <= j; ++i) w[i] = zmk(0.0, 0.0);
      w[j] = zmk(1.0, 0.0);
      if (kind[j] != 2) {
        zupdate_above(j, S, lds, T, ldt, cmS, cmT, &v, a[j], b[j], beta[j], protect);
        for (int i = j - 1; i >= 0; --i) {
          zsolve_row(i, S, lds, T, ldt, &v, j, a[j], b[j], beta[j], protect);
          zupdate_above(i, S, lds, T, ldt, cmS, cmT, &v, a[j], b[j], beta[j], protect);
        }
      }
      /* ZTGEVC normalisation: max (|Re|+|Im|) = 1, formed as 2 max(|Re|/2 + |Im|/2) */
      double h = 0.0;
      for (int i = 0; i <= j; ++i) h = zmax2(h, 0.5 * fabs(w[i].re) + 0.5 * fabs(w[i].im));
      double rec = (h > 0.0) ? 0.5 / h : 1.0;
      double* x = X + 2 * (size_t)colof[j] * (size_t)ldx;
      for (int i = 0; i < m; ++i) {
        x[2 * i] = (i <= j) ? w[i].re * rec : 0.0;
        x[2 * i + 1] = (i <= j) ? w[i].im * rec : 0.0;
      }
      if (col_scale_exp) col_scale_exp[colof[j]] = v.e;
      s0 += v.nscal;
      s1 += v.npert;
      s2 += (kind[j] == 2);
    }
    free(w);
  }
  if (stats) { stats[0] = s0; stats[1] = s1; stats[2] = s2; }
  free(a);
  free(kind);
  return bad ? ZO_ERR_NOMEM : 0;
}
