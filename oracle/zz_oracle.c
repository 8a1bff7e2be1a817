/*
 * oracle/zz_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load, call or execute this library.  The product path
 * (paper_2003_04776_b200/) never links or imports it, and shares no code, header, table
 * or constant generator with it.
 *
 * What it computes.  All (or the selected) right generalized eigenvectors of a real
 * pencil (S,T) in generalized real Schur form, i.e. the columns of V in
 * S V D - T V B = 0 (D, B of PAPER.md:83-99).  For the eigenvalue
 * (alpha, beta), alpha = a + i b, of the diagonal block ending at row r, the eigenvector z
 * has z_i = 0 for i > r and solves (beta S - alpha T)(0:r,0:r) z = 0 (Lemma 1,
 * PAPER.md:106-111).  A complex pair is returned as two real columns [Re z, Im z] for the
 * eigenvalue with b > 0.
 *
 * How.  The plain method the paper contrasts its blocked algorithm with: a scalar
 * column-by-column substitution, one eigenvector at a time, as LAPACK xTGEVC does
 * (PAPER.md:37-39), made robust with ProtectDivision / ProtectUpdate
 * and an int32 power-of-two scaling exponent per eigenvector.
 * No blocking, no fusion, no reordering.  Every reading of an underspecified point is
 * listed in DESIGN.md section "Readings" (R1..R17) and cited below by its number.
 *
 * Parity status.  Pinned by tests/test_oracle_*.py against: SPEC worked examples for the
 * protect functions, exact-rational property tests, closed-form 1x1/2x2 eigenpairs,
 * long-double brute-force null vectors (m <= 8), LAPACK DTGEVC as a black box, long-double
 * unprotected substitution on stress pencils, and invariants.  col_scale_exp values are
 * implementation-defined: "parity unpinned" (only invariants and L_c are compared).
 * The perturbed-pivot path (smin, R8) is "parity unpinned" except for the indefinite case.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (no implicit FMA contraction;
 * every fma below is explicit).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ZZO_OMEGA 0x1p1023        /* R1: overflow threshold Omega = 2^1023 */
#define ZZO_U 0x1p-53             /* unit roundoff */
#define ZZO_SMLNUM 0x1p-969       /* smallest normal / u = 2^-1022 / 2^-53 */

/* status codes (same meaning as include/zz.h, written out independently) */
#define ZZO_OK 0
#define ZZO_ERR_NONFINITE (-104)
#define ZZO_ERR_OVERLAP (-105)
#define ZZO_ERR_NOMEM (-102)

typedef struct { double re, im; } cplx;

static inline double dmax(double x, double y) { return x > y ? x : y; }
static inline double dmin(double x, double y) { return x < y ? x : y; }
static inline double cnorm_max(cplx z) { return dmax(fabs(z.re), fabs(z.im)); } /* max(|Re|,|Im|) */
static inline double cnorm_1(cplx z) { return fabs(z.re) + fabs(z.im); }         /* |Re|+|Im| */
static inline cplx cmk(double re, double im) { cplx z = {re, im}; return z; }
static inline cplx cmul(cplx x, cplx y) {
  return cmk(x.re * y.re - x.im * y.im, x.re * y.im + x.im * y.re);
}
static inline cplx csub(cplx x, cplx y) { return cmk(x.re - y.re, x.im - y.im); }
/* Smith's complex division x / y (R9). */
static inline cplx cdiv(cplx x, cplx y) {
  if (fabs(y.re) >= fabs(y.im)) {
    double r = y.im / y.re, den = y.re + y.im * r;
    return cmk((x.re + x.im * r) / den, (x.im - x.re * r) / den);
  } else {
    double r = y.re / y.im, den = y.im + y.re * r;
    return cmk((x.re * r + x.im) / den, (x.im * r - x.re) / den);
  }
}

/* ---------------------------------------------------------------------------------
 * ProtectUpdate / ProtectDivision (definitions are reading R4/R5 of
 * DESIGN.md, the paper gives only the contracts).  Both return the exponent e <= 0 of
 * xi = 2^e.
 * ------------------------------------------------------------------------------- */

/* ProtectUpdate(y, t, x), y,t,x in [0, Omega]: xi (y + t x) <= Omega.
 * s = y/2^1023 + (t/2^512)(x/2^511) cannot overflow; s <= 1/2 => e = 0, otherwise
 * e = -ceil(log2 s) - 1, so that 2^e s <= 1/2 (the factor 2 absorbs rounding in s). */
int zzo_protect_update(double y, double t, double x) {
  double s = y * 0x1p-1023 + (t * 0x1p-512) * (x * 0x1p-511);
  if (s <= 0.5) return 0;
  int k;
  double f = frexp(s, &k); /* s = f 2^k, f in [1/2, 1) */
  int c = (f == 0.5) ? k - 1 : k; /* ceil(log2 s) */
  return -c - 1;
}

/* ProtectDivision(b, t), b in [0, Omega], t > 0: xi b <= t Omega.
 * e = 0 if t >= 1 or b <= t Omega; else e = floor(log2(t Omega / b)) - 1. */
int zzo_protect_division(double b, double t) {
  if (t >= 1.0 || b <= t * ZZO_OMEGA) return 0;
  double r = (t * ZZO_OMEGA) / b; /* in (0, 1) */
  int k;
  frexp(r, &k); /* r in [2^(k-1), 2^k) => floor(log2 r) = k - 1 */
  return (k - 1) - 1;
}

/* ---------------------------------------------------------------------------------
 * Structure: the diagonal blocks of S.  A 2x2 block starts at j when
 * S(j+1,j) != 0; two consecutive nonzero subdiagonals are an error (-105).
 * ------------------------------------------------------------------------------- */
#define S_(i, j) S[(size_t)(j) * (size_t)lds + (size_t)(i)]
#define T_(i, j) T[(size_t)(j) * (size_t)ldt + (size_t)(i)]

int zzo_blocks(int m, const double* S, int lds, int* blk_start, int* blk_size) {
  int nb = 0, j = 0;
  while (j < m) {
    int two = (j + 1 < m) && (S_(j + 1, j) != 0.0);
    if (two && j + 2 < m && S_(j + 2, j + 1) != 0.0) return ZZO_ERR_OVERLAP;
    blk_start[nb] = j;
    blk_size[nb] = two ? 2 : 1;
    nb++;
    j += two ? 2 : 1;
  }
  return nb;
}

/* ---------------------------------------------------------------------------------
 * Eigenvalue pairs (alpha, beta), alpha = a + i b, normalised by an
 * exact power of two so that max(beta, |a|+|b|) is in [1/2, 1) (reading R2 of DESIGN.md).
 * kind: 0 real, 1 complex pair (b > 0), 2 indefinite (alpha = beta = 0).
 * Returns 0, or 1 if a 2x2 block has no complex-conjugate pair (assumption 2 violated).
 * ------------------------------------------------------------------------------- */
static void normalise_pair(double* a, double* b, double* beta, int* kind) {
  double h = dmax(0.5 * *beta, 0.5 * fabs(*a) + 0.5 * fabs(*b));
  if (h == 0.0) { *kind = 2; return; }
  int k;
  frexp(h, &k); /* h in [2^(k-1), 2^k) => max(beta, |a|+|b|) * 2^-(k+1) in [1/2, 1) */
  *a = ldexp(*a, -(k + 1));
  *b = ldexp(*b, -(k + 1));
  *beta = ldexp(*beta, -(k + 1));
}

static int pair_1x1(double s, double t, double* a, double* b, double* beta, int* kind) {
  /* (alpha, beta) = (S_jj, T_jj), signs flipped together so that beta >= 0. */
  *a = s; *b = 0.0; *beta = t; *kind = 0;
  if (*beta < 0) { *a = -*a; *beta = -*beta; }
  normalise_pair(a, b, beta, kind);
  return 0;
}

/* 2x2 block: the eigenvalues lambda of (S_blk, T_blk) are those of N = T_blk^{-1} S_blk,
 * lambda = p +- i q with p = (n11+n22)/2, q = sqrt(-((n11-n22)^2/4 + n12 n21)) (reading R3).
 * The blocks are first scaled by powers of two so that their max-abs entries lie in
 * [1/2, 1); lambda = mu 2^(ks-kt) is represented as alpha = p + i q, beta = 2^(kt-ks). */
static int pair_2x2(double s11, double s21, double s12, double s22, double t11, double t12,
                    double t22, double* a, double* b, double* beta, int* kind) {
  double ms = dmax(dmax(fabs(s11), fabs(s12)), dmax(fabs(s21), fabs(s22)));
  double mt = dmax(dmax(fabs(t11), fabs(t12)), fabs(t22));
  if (!(ms > 0.0) || !(mt > 0.0)) return 1;
  int ks, kt;
  frexp(ms, &ks);
  frexp(mt, &kt);
  s11 = ldexp(s11, -ks); s21 = ldexp(s21, -ks); s12 = ldexp(s12, -ks); s22 = ldexp(s22, -ks);
  t11 = ldexp(t11, -kt); t12 = ldexp(t12, -kt); t22 = ldexp(t22, -kt);
  if (t11 == 0.0 || t22 == 0.0) return 1; /* an infinite eigenvalue: not a complex pair */
  double n21 = s21 / t22;
  double n11 = (s11 - t12 * n21) / t11;
  double n12 = (s12 - t12 * (s22 / t22)) / t11;
  double n22 = s22 / t22;
  double d = (n11 - n22) * 0.5;
  double disc = d * d + n12 * n21;
  if (!(disc < 0.0)) return 1; /* real eigenvalues: assumption 2 violated */
  *a = n22 + d;
  *b = sqrt(-disc);
  *beta = ldexp(1.0, kt - ks);
  *kind = 1;
  normalise_pair(a, b, beta, kind);
  return 0;
}

/* Per-row pairs: a[j], b[j], beta[j], kind[j]; both rows of a 2x2 block carry the same
 * values.  Returns 0, or j+1 (1-based first row) of the first 2x2 block with real
 * eigenvalues, or a negative status. */
int zzo_eig_pairs(int m, const double* S, int lds, const double* T, int ldt, double* a,
                  double* b, double* beta, int* kind) {
  int* bs = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
  int* bz = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
  if (!bs || !bz) { free(bs); free(bz); return ZZO_ERR_NOMEM; }
  int nb = zzo_blocks(m, S, lds, bs, bz);
  int info = 0;
  if (nb < 0) info = nb;
  for (int p = 0; p < nb && info == 0; ++p) {
    int j = bs[p];
    double aa, bb, be;
    int kd;
    if (bz[p] == 1) {
      if (!isfinite(S_(j, j)) || !isfinite(T_(j, j))) { info = ZZO_ERR_NONFINITE; break; }
      pair_1x1(S_(j, j), T_(j, j), &aa, &bb, &be, &kd);
      a[j] = aa; b[j] = bb; beta[j] = be; kind[j] = kd;
    } else {
      double v[7] = {S_(j, j), S_(j + 1, j), S_(j, j + 1), S_(j + 1, j + 1), T_(j, j),
                     T_(j, j + 1), T_(j + 1, j + 1)};
      for (int q = 0; q < 7; ++q)
        if (!isfinite(v[q])) info = ZZO_ERR_NONFINITE;
      if (info) break;
      if (pair_2x2(v[0], v[1], v[2], v[3], v[4], v[5], v[6], &aa, &bb, &be, &kd)) {
        info = j + 1;
        break;
      }
      a[j] = a[j + 1] = aa; b[j] = b[j + 1] = bb; beta[j] = beta[j + 1] = be;
      kind[j] = kind[j + 1] = kd;
    }
  }
  free(bs); free(bz);
  return info;
}

/* ---------------------------------------------------------------------------------
 * One eigenvector by robust substitution.
 * Running representation (Definition 1, reading R2 "true = 2^-e w"):
 * the true eigenvector (tip-normalised) is 2^-e * w; every scaling multiplies all of w by
 * 2^k (k <= 0) and adds k to e.
 * ------------------------------------------------------------------------------- */
typedef struct {
  int m, lds, ldt;
  const double* S;
  const double* T;
  const int* blkof;    /* row -> index of its diagonal block */
  const int* bstart;   /* block -> first row */
  const int* bsize;    /* block -> 1 or 2 */
  const double* cmS;   /* column j: max_{i < blockstart(j)} |S_ij| (reading R6) */
  const double* cmT;
  int protect;         /* 1 robust, 0 = naive negative control (no ProtectUpdate/Division) */
} ctx_t;

typedef struct {
  cplx* w;     /* rows 0..r */
  int r;       /* last row of the eigenvalue's block */
  int e;       /* scaling exponent */
  int nscal;   /* number of scalings applied */
  int npert;   /* number of perturbed pivots */
} vec_t;

static void vscale(vec_t* v, int k) {
  if (k >= 0) return;
  for (int i = 0; i <= v->r; ++i) {
    v->w[i].re = ldexp(v->w[i].re, k);
    v->w[i].im = ldexp(v->w[i].im, k);
  }
  v->e += k;
  v->nscal++;
}

/* max(|Re|,|Im|) over rows 0..n-1 (the pending part) */
static double pending_max(const vec_t* v, int n) {
  double mx = 0.0;
  for (int i = 0; i < n; ++i) mx = dmax(mx, cnorm_max(v->w[i]));
  return mx;
}

/* Update the pending rows 0..ks-1 with the solved block rows ks..ke (
 * protected as in PAPER.md:187-199, 235):  w_i <- w_i - (S_ik (beta x_k) - T_ik (alpha x_k)). */
static void update_above(const ctx_t* c, vec_t* v, int ks, int ke, double a, double b,
                         double beta) {
  if (ks == 0) return;
  const double* S = c->S; const double* T = c->T; int lds = c->lds, ldt = c->ldt;
  if (c->protect) {
    double xn = 0.0, t = 0.0;
    for (int k = ks; k <= ke; ++k) {
      xn = dmax(xn, cnorm_max(v->w[k]));
      t += beta * c->cmS[k] + (fabs(a) + fabs(b)) * c->cmT[k];
    }
    double wmax = pending_max(v, ks);
    vscale(v, zzo_protect_update(wmax, t, xn));
  }
  for (int k = ks; k <= ke; ++k) {
    cplx x = v->w[k];
    cplx u = cmk(beta * x.re, beta * x.im);                 /* x D  */
    cplx al = cmk(a, b);
    cplx vv = cmul(al, x);                                   /* x B  */
    if (b == 0.0) {
      /* real eigenvalue: imaginary parts are identically zero; same values as below */
      for (int i = 0; i < ks; ++i)
        v->w[i].re = v->w[i].re - (S_(i, k) * u.re - T_(i, k) * vv.re);
    } else {
      for (int i = 0; i < ks; ++i) {
        v->w[i].re = v->w[i].re - (S_(i, k) * u.re - T_(i, k) * vv.re);
        v->w[i].im = v->w[i].im - (S_(i, k) * u.im - T_(i, k) * vv.im);
      }
    }
  }
}

/* Robust scalar division x = w / d (R9): real columns use ProtectDivision(|w|, |d|);
 * complex ones ProtectDivision(max(|Re w|,|Im w|), min(1, max(|Re d|,|Im d|))/2), which
 * bounds Smith's intermediates and quotient by Omega. */
static cplx protected_div(const ctx_t* c, vec_t* v, cplx* wj, cplx d, int real) {
  if (real) {
    if (c->protect) {
      int k = zzo_protect_division(fabs(wj->re), fabs(d.re));
      if (k < 0) vscale(v, k);  /* wj points into v->w or is scaled by the caller */
    }
    return cmk(wj->re / d.re, 0.0);
  }
  if (c->protect) {
    int k = zzo_protect_division(cnorm_max(*wj), 0.5 * dmin(1.0, cnorm_max(d)));
    if (k < 0) vscale(v, k);
  }
  return cdiv(*wj, d);
}

/* Solve the 1x1 row j: (beta S_jj - alpha T_jj) x_j = w_j. */
static void solve_1x1(const ctx_t* c, vec_t* v, int j, double a, double b, double beta) {
  const double* S = c->S; const double* T = c->T; int lds = c->lds, ldt = c->ldt;
  double sjj = S_(j, j), tjj = T_(j, j);
  cplx d = cmk(fma(-a, tjj, beta * sjj), -b * tjj);
  /* R8: local, cancellation-aware perturbation threshold */
  double smin = dmax(ZZO_U * (beta * fabs(sjj) + (fabs(a) + fabs(b)) * fabs(tjj)), ZZO_SMLNUM);
  if (cnorm_1(d) < smin) { d = cmk(smin, 0.0); v->npert++; }
  v->w[j] = protected_div(c, v, &v->w[j], d, b == 0.0);
}

/* Solve the 2x2 rows (j, j+1): C x = w with C = beta S_blk - alpha T_blk, complete pivoting
 * on |Re|+|Im|, pivots below smin replaced by smin (DLALN2's role; R9). */
static void solve_2x2(const ctx_t* c, vec_t* v, int j, double a, double b, double beta) {
  const double* S = c->S; const double* T = c->T; int lds = c->lds, ldt = c->ldt;
  int real = (b == 0.0);
  double s11 = S_(j, j), s21 = S_(j + 1, j), s12 = S_(j, j + 1), s22 = S_(j + 1, j + 1);
  double t11 = T_(j, j), t12 = T_(j, j + 1), t22 = T_(j + 1, j + 1);
  cplx C[2][2];
  C[0][0] = cmk(fma(-a, t11, beta * s11), -b * t11);
  C[1][0] = cmk(beta * s21, 0.0);
  C[0][1] = cmk(fma(-a, t12, beta * s12), -b * t12);
  C[1][1] = cmk(fma(-a, t22, beta * s22), -b * t22);
  double maxs = dmax(dmax(fabs(s11), fabs(s21)), dmax(fabs(s12), fabs(s22)));
  double maxt = dmax(dmax(fabs(t11), fabs(t12)), fabs(t22));
  double smin = dmax(ZZO_U * (beta * maxs + (fabs(a) + fabs(b)) * maxt), ZZO_SMLNUM);
  /* complete pivoting: first maximal |.|_1 in the order (0,0), (1,0), (0,1), (1,1) */
  int pr = 0, pc = 0;
  double best = cnorm_1(C[0][0]);
  if (cnorm_1(C[1][0]) > best) { best = cnorm_1(C[1][0]); pr = 1; pc = 0; }
  if (cnorm_1(C[0][1]) > best) { best = cnorm_1(C[0][1]); pr = 0; pc = 1; }
  if (cnorm_1(C[1][1]) > best) { best = cnorm_1(C[1][1]); pr = 1; pc = 1; }
  cplx p = C[pr][pc];
  if (cnorm_1(p) < smin) { p = cmk(smin, 0.0); v->npert++; }
  cplx rr = C[1 - pr][pc], cc = C[pr][1 - pc], ss = C[1 - pr][1 - pc];
  cplx l = cdiv(rr, p);
  cplx u22 = csub(ss, cmul(l, cc));
  if (cnorm_1(u22) < smin) { u22 = cmk(smin, 0.0); v->npert++; }
  /* rows of the permuted system live in v->w so that whole-vector scalings reach them */
  int i1 = j + pr, i2 = j + 1 - pr;
  /* forward step y2 <- y2 - l y1 : componentwise |.| <= wn + 2 wn */
  if (c->protect) {
    double wn = dmax(cnorm_max(v->w[i1]), cnorm_max(v->w[i2]));
    vscale(v, zzo_protect_update(wn, 2.0, wn));
  }
  cplx y1 = v->w[i1];
  cplx y2 = csub(v->w[i2], cmul(l, y1));
  v->w[i2] = y2;
  /* back substitution: z2 = y2 / u22 */
  cplx z2 = protected_div(c, v, &v->w[i2], u22, real);
  v->w[i2] = z2;
  /* z1 = (y1 - cc z2) / p */
  if (c->protect) {
    vscale(v, zzo_protect_update(cnorm_max(v->w[i1]), cnorm_1(cc), cnorm_max(v->w[i2])));
  }
  z2 = v->w[i2];
  cplx n1 = csub(v->w[i1], cmul(cc, z2));
  v->w[i1] = n1;
  cplx z1 = protected_div(c, v, &v->w[i1], p, real);
  z2 = v->w[i2]; /* may have been rescaled by the last division's protection */
  /* unpermute columns: x[pc] = z1, x[1-pc] = z2 */
  v->w[j + pc] = z1;
  v->w[j + 1 - pc] = z2;
}

/* The tip (reading R10): real: x_r = 1.  Pair at rows (r-1, r):
 * p = beta S(r,r-1), q = beta S(r,r) - alpha T(r,r); if |p| >= |Re q|+|Im q|:
 * z_r = 1, z_{r-1} = -q/p; else z_{r-1} = 1, z_r = -p/q. */
static void tip(const ctx_t* c, vec_t* v, int kindc, double a, double b, double beta) {
  const double* S = c->S; const double* T = c->T; int lds = c->lds, ldt = c->ldt;
  int r = v->r;
  if (kindc != 1) { v->w[r] = cmk(1.0, 0.0); return; }
  double p = beta * S_(r, r - 1);
  cplx q = cmk(fma(-a, T_(r, r), beta * S_(r, r)), -b * T_(r, r));
  if (fabs(p) >= cnorm_1(q)) {
    v->w[r] = cmk(1.0, 0.0);
    v->w[r - 1] = cmk(-q.re / p, -q.im / p);
  } else {
    v->w[r - 1] = cmk(1.0, 0.0);
    cplx z = cdiv(cmk(p, 0.0), q);
    v->w[r] = cmk(-z.re, -z.im);
  }
}

/* One selected block p: fills X column(s) col (and col+1 for a pair). */
static void solve_one(const ctx_t* c, int p, const double* pa, const double* pb,
                      const double* pbeta, const int* pkind, cplx* work, double* X, int ldx,
                      int col, int* col_scale_exp, double* logmax, int* stats) {
  int m = c->m;
  int js = c->bstart[p], sz = c->bsize[p];
  int r = js + sz - 1;
  double a = pa[js], b = pb[js], beta = pbeta[js];
  int kindc = pkind[js];
  int ncol = (kindc == 1) ? 2 : 1;
  vec_t v;
  v.w = work; v.r = r; v.e = 0; v.nscal = 0; v.npert = 0;
  for (int i = 0; i <= r; ++i) v.w[i] = cmk(0.0, 0.0);
  if (kindc == 2) {
    /* indefinite (alpha = beta = 0): the unit vector e_r (reading R13) */
    v.w[r] = cmk(1.0, 0.0);
  } else {
    tip(c, &v, kindc, a, b, beta);
    int ks = (kindc == 1) ? r - 1 : r;
    /* a real eigenvalue inside... never: a real eigenvalue is always a 1x1 block */
    update_above(c, &v, ks, r, a, b, beta);
    /* blocks above the tip, bottom-up (PAPER.md:138-146 applied per column) */
    int q = c->blkof[ks] - 1;
    for (; q >= 0; --q) {
      int bs = c->bstart[q], bz = c->bsize[q];
      if (bz == 1) solve_1x1(c, &v, bs, a, b, beta);
      else solve_2x2(c, &v, bs, a, b, beta);
      update_above(c, &v, bs, bs + bz - 1, a, b, beta);
    }
  }
  /* LAPACK normalisation (reading R11): real max|x_i| = 1, pair max(|x_i|+|y_i|) = 1;
   * xmax is formed as 2 * max(|x|/2 + |y|/2) so that it cannot overflow. */
  double h = 0.0;
  for (int i = 0; i <= r; ++i) {
    double t = (ncol == 2) ? 0.5 * fabs(v.w[i].re) + 0.5 * fabs(v.w[i].im) : 0.5 * fabs(v.w[i].re);
    h = dmax(h, t);
  }
  double rec = (h > 0.0) ? 0.5 / h : 1.0;
  double* x0 = X + (size_t)col * (size_t)ldx;
  double* x1 = (ncol == 2) ? X + (size_t)(col + 1) * (size_t)ldx : NULL;
  for (int i = 0; i < m; ++i) {
    x0[i] = (i <= r) ? v.w[i].re * rec : 0.0;
    if (x1) x1[i] = (i <= r) ? v.w[i].im * rec : 0.0;
  }
  if (col_scale_exp) {
    col_scale_exp[col] = v.e;
    if (x1) col_scale_exp[col + 1] = v.e;
  }
  if (logmax) {
    double L = (h > 0.0) ? log2(h) + 1.0 - (double)v.e : -INFINITY;
    logmax[col] = L;
    if (x1) logmax[col + 1] = L;
  }
  if (stats) {
    stats[0] += v.nscal;
    stats[1] += v.npert;
    stats[2] += (kindc == 2);
  }
}

/* Overflow-free infinity norm (max row sum of |.|) of the upper part of a matrix
 * (rows 0..min(j+1,m-1) of column j), scaled by 2^-64. */
static double inf_norm_scaled(int m, const double* A, int lda) {
  double* rs = (double*)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
  if (!rs) return INFINITY;
  for (int j = 0; j < m; ++j) {
    int ie = (j + 1 < m) ? j + 1 : m - 1;
    for (int i = 0; i <= ie; ++i) rs[i] += fabs(A[(size_t)j * lda + i]) * 0x1p-64;
  }
  double mx = 0.0;
  for (int i = 0; i < m; ++i) mx = dmax(mx, rs[i]);
  free(rs);
  return mx;
}

/*
 * zzo_tgevc: all selected right eigenvectors.
 *   select: int[m] or NULL (all); eigenvalue j selected if select[j] != 0; a pair is
 *           computed if either of its flags is set; columns packed in block order.
 *   X (m x n_sel, ldx), col_scale_exp[n_sel], logmax[n_sel] (L_c = log2 of the
 *   tip-normalised vector's max measure, may be NULL), pairs_out (3 x m: a,b,beta per
 *   row, may be NULL), stats[3] = {#scalings, #perturbed pivots, #indefinite} (may be NULL).
 *   protect = 1 robust; 0 = naive negative control.  nthreads <= 0: OpenMP default.
 * Returns 0, j > 0 (2x2 block at 1-based row j has real eigenvalues) or a negative status.
 */
int zzo_tgevc_ex(int m, const double* S0, int lds, const double* T0, int ldt, const int* select,
                 double* X, int ldx, int* col_scale_exp, double* logmax, double* pairs_out,
                 int* stats, int protect, int nthreads) {
  if (m < 0) return -1;
  if (lds < (m > 1 ? m : 1)) return -3;
  if (ldt < (m > 1 ? m : 1)) return -5;
  if (ldx < (m > 1 ? m : 1)) return -8;
  if (stats) stats[0] = stats[1] = stats[2] = 0;
  if (m == 0) return 0;
  int status = 0;
  /* R6: pre-scale S, T by powers of two if a row sum of |.| exceeds Omega/8 */
  const double* S = S0;
  const double* T = T0;
  double* Sc = NULL;
  double* Tc = NULL;
  for (int w = 0; w < 2; ++w) {
    const double* A = w ? T0 : S0;
    int lda = w ? ldt : lds;
    double nrm = inf_norm_scaled(m, A, lda); /* true norm * 2^-64 */
    if (nrm > 0x1p1020 * 0x1p-64) {
      int k = 0;
      while (ldexp(nrm, -k) > 0x1p1020 * 0x1p-64) k++;
      double* C = (double*)malloc(sizeof(double) * (size_t)m * (size_t)m);
      if (!C) return ZZO_ERR_NOMEM;
      for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) C[(size_t)j * m + i] = ldexp(A[(size_t)j * lda + i], -k);
      if (w) { Tc = C; T = C; ldt = m; } else { Sc = C; S = C; lds = m; }
    }
  }
  int* bstart = (int*)malloc(sizeof(int) * m);
  int* bsize = (int*)malloc(sizeof(int) * m);
  int* blkof = (int*)malloc(sizeof(int) * m);
  double* pa = (double*)malloc(sizeof(double) * m);
  double* pb = (double*)malloc(sizeof(double) * m);
  double* pbeta = (double*)malloc(sizeof(double) * m);
  int* pkind = (int*)malloc(sizeof(int) * m);
  double* cmS = (double*)malloc(sizeof(double) * m);
  double* cmT = (double*)malloc(sizeof(double) * m);
  int* order = (int*)malloc(sizeof(int) * m);
  int* colof = (int*)malloc(sizeof(int) * m);
  if (!bstart || !bsize || !blkof || !pa || !pb || !pbeta || !pkind || !cmS || !cmT || !order ||
      !colof) {
    status = ZZO_ERR_NOMEM;
    goto done;
  }
  int nb = zzo_blocks(m, S, lds, bstart, bsize);
  if (nb < 0) { status = nb; goto done; }
  for (int p = 0; p < nb; ++p)
    for (int q = 0; q < bsize[p]; ++q) blkof[bstart[p] + q] = p;
  status = zzo_eig_pairs(m, S, lds, T, ldt, pa, pb, pbeta, pkind);
  if (status != 0) goto done;
  if (pairs_out)
    for (int j = 0; j < m; ++j) {
      pairs_out[3 * j] = pa[j]; pairs_out[3 * j + 1] = pb[j]; pairs_out[3 * j + 2] = pbeta[j];
    }
  /* column bounds above each diagonal block (reading R6) */
#pragma omp parallel for schedule(static)
  for (int j = 0; j < m; ++j) {
    int top = bstart[blkof[j]];
    double ms = 0.0, mt = 0.0;
    for (int i = 0; i < top; ++i) {
      ms = dmax(ms, fabs(S_(i, j)));
      mt = dmax(mt, fabs(T_(i, j)));
    }
    cmS[j] = ms; cmT[j] = mt;
  }
  /* selection and packed columns */
  int nsel = 0, ncol = 0;
  for (int p = 0; p < nb; ++p) {
    int js = bstart[p], sz = bsize[p];
    int sel = select == NULL || select[js] || (sz == 2 && select[js + 1]);
    if (!sel) continue;
    order[nsel++] = p;
    colof[p] = ncol;
    ncol += (pkind[js] == 1) ? 2 : 1;
  }
  /* longest columns first for load balance (result independent of the order) */
  for (int i = 1; i < nsel; ++i) { /* insertion sort by descending block start */
    int x = order[i], k = i - 1;
    while (k >= 0 && bstart[order[k]] < bstart[x]) { order[k + 1] = order[k]; k--; }
    order[k + 1] = x;
  }
  {
    ctx_t c;
    c.m = m; c.lds = lds; c.ldt = ldt; c.S = S; c.T = T; c.blkof = blkof; c.bstart = bstart;
    c.bsize = bsize; c.cmS = cmS; c.cmT = cmT; c.protect = protect;
    int st0 = 0, st1 = 0, st2 = 0;
    int nomem = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel reduction(+ : st0, st1, st2) reduction(| : nomem)
    {
      cplx* work = (cplx*)malloc(sizeof(cplx) * (size_t)m);
      if (!work) nomem = 1;
      int st[3] = {0, 0, 0};
#pragma omp for schedule(dynamic, 1)
      for (int i = 0; i < nsel; ++i) {
        if (!work) continue;
        int p = order[i];
        solve_one(&c, p, pa, pb, pbeta, pkind, work, X, ldx, colof[p], col_scale_exp, logmax, st);
      }
      st0 += st[0]; st1 += st[1]; st2 += st[2];
      free(work);
    }
    if (nomem) status = ZZO_ERR_NOMEM;
    if (stats) { stats[0] = st0; stats[1] = st1; stats[2] = st2; }
  }
done:
  free(bstart); free(bsize); free(blkof); free(pa); free(pb); free(pbeta); free(pkind);
  free(cmS); free(cmT); free(order); free(colof); free(Sc); free(Tc);
  return status;
}

/* Number of output columns for a selection (pairs count 2), or a negative status. */
int zzo_count_columns(int m, const double* S, int lds, const int* select) {
  int* bs = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
  int* bz = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
  if (!bs || !bz) { free(bs); free(bz); return ZZO_ERR_NOMEM; }
  int nb = zzo_blocks(m, S, lds, bs, bz);
  int n = 0;
  if (nb < 0) n = nb;
  for (int p = 0; p < nb; ++p) {
    int js = bs[p];
    int sel = select == NULL || select[js] || (bz[p] == 2 && select[js + 1]);
    if (sel) n += bz[p];
  }
  free(bs); free(bz);
  return n;
}

/* Nominal flop count F(select) = sum over selected columns c of 2 r_c (r_c - 1), r_c the
 * 1-based last row of the column's block. */
double zzo_flops(int m, const double* S, int lds, const int* select) {
  int* bs = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
  int* bz = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
  if (!bs || !bz) { free(bs); free(bz); return -1.0; }
  int nb = zzo_blocks(m, S, lds, bs, bz);
  double f = 0.0;
  for (int p = 0; p < nb; ++p) {
    int js = bs[p];
    int sel = select == NULL || select[js] || (bz[p] == 2 && select[js + 1]);
    double r = (double)(js + bz[p]);
    if (sel) f += (double)bz[p] * 2.0 * r * (r - 1.0);
  }
  free(bs); free(bz);
  return nb < 0 ? -1.0 : f;
}
