// zz_diag.cu -- the robust diagonal-block solve (Kernel 1 tips and Kernel 3 right-hand
// sides; Alg. 1 lines P:137) for tiles of at most 128
// rows, fused with the per-column scaling decision of the following update (Algs. 2/3,
// PAPER.md:216-262) and the formation of the update's B operand W.
//
// B200 design.  One THREAD per eigenvector (real column or complex pair): the shifted
// matrix beta_c S_II - alpha_c T_II differs per column but its entries S_ij, T_ij do not,
// so 32 eigenvectors of a warp read the same shared-memory word (a broadcast) and run the
// same control flow (the 1x1 / 2x2 structure is per row, not per column).  The tile is cut
// into sub-tiles of ~16 rows (a boundary never splits a 2x2 block); warp k owns sub-tile
// k of a group of 32 eigenvectors and keeps those rows in registers:
//
//   for k2 = nsub-1 .. k+1:  wait for x(k2) (named barrier k2), then apply the block update
//                            y_k <- y_k - S(k,k2) (beta x_k2) + T(k,k2) (alpha x_k2)
//                            after the Alg. 3 decision (own exponent vs. x_k2's exponent,
//                            ProtectUpdate with the block's infinity norms);
//   solve sub-tile k bottom-up (1x1 / 2x2 micro-solves with ProtectDivision and the
//   in-sub-tile ProtectUpdate), publish x_k with its exponent and norm, arrive on barrier k.
//
// Each sub-tile carries its own power-of-two exponent (an augmented matrix at sub-tile
// granularity, Definition 1); at the end the segment is brought to the
// smallest exponent (exact), stored to X, and W = [-2^sX X D ; 2^sX X B] is written.
// Powers of two are exact, so with no scaling the result is the plain substitution.
#include <math.h>
#include <stdint.h>

#include "zz_internal.cuh"
#include "zz_device.cuh"

namespace zz {

namespace {

constexpr int kSR = 17;       // max rows of a sub-tile (16, +1 when a 2x2 block straddles)
constexpr int kNSub = 8;      // max sub-tiles per tile (nt <= 128)
constexpr int kDW = 8;        // warps per CTA (one per sub-tile)
constexpr int kXP = 33;       // padded lane dimension of the exchange buffer

__device__ __forceinline__ int poff2(int j) { return j * (j + 3) / 2; }

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// x * 2^k for k <= 0 (exact while the result is normal; powers of two below 2^-1022 are
// applied in steps).  Much shorter code than ldexp in the unrolled register loops.
__device__ __forceinline__ double pow2i(int k) { return __hiloint2double((k + 1023) << 20, 0); }
__device__ __noinline__ double scale2_slow(double x, int k) {
  while (k < -1022) { x *= 0x1p-1022; k += 1022; }
  return x * pow2i(k);
}
__device__ __forceinline__ double scale2(double x, int k) { return k >= -1022 ? x * pow2i(k) : scale2_slow(x, k); }

struct Sm {
  double2* ST;       // packed upper tile (+ subdiagonal): (S_ij, T_ij) at poff2(j) + i
  double2* cm;       // per row j: max |S|, |T| over the sub-tile rows above j's block
  double2* nb;       // [kNSub][kNSub] block infinity norms (S, T), block (k, k2), k < k2
  double2* xs;       // [kNSub][kSR][kXP] exchange of solved sub-tiles (re, im)
  double* xn;        // [kNSub][32] max(|Re|,|Im|) of a published sub-tile
  int* xe;           // [kNSub][32] its exponent
  double* rn;        // [kNSub][32] final segment norms per sub-tile
  double* rh;        // [kNSub][32]
  int* wsx;          // [32] exponent shift of W per lane
  int* cols;         // [32] column of each lane (-1 invalid)
  int* sb;           // [kNSub + 1] sub-tile boundaries
  signed char* fl;   // [nt] row flags
};

// smem carve-up (all offsets 16-byte aligned)
__host__ __device__ __forceinline__ size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ __forceinline__ size_t smem_need(int nt) {
  size_t o = 0;
  o += al16(sizeof(double2) * (size_t)(nt * (nt + 3) / 2 + 2));
  o += al16(sizeof(double2) * (size_t)nt);
  o += al16(sizeof(double2) * kNSub * kNSub);
  o += al16(sizeof(double2) * kNSub * kSR * kXP);
  o += al16(sizeof(double) * kNSub * 32) * 3;
  o += al16(sizeof(int) * kNSub * 32);
  o += al16(sizeof(int) * 32) * 2;
  o += al16(sizeof(int) * (kNSub + 1));
  o += al16((size_t)nt);
  return o;
}

__device__ __forceinline__ Sm carve(unsigned char* base, int nt) {
  Sm s;
  size_t o = 0;
  s.ST = reinterpret_cast<double2*>(base + o); o += al16(sizeof(double2) * (size_t)(nt * (nt + 3) / 2 + 2));
  s.cm = reinterpret_cast<double2*>(base + o); o += al16(sizeof(double2) * (size_t)nt);
  s.nb = reinterpret_cast<double2*>(base + o); o += al16(sizeof(double2) * kNSub * kNSub);
  s.xs = reinterpret_cast<double2*>(base + o); o += al16(sizeof(double2) * kNSub * kSR * kXP);
  s.xn = reinterpret_cast<double*>(base + o); o += al16(sizeof(double) * kNSub * 32);
  s.rn = reinterpret_cast<double*>(base + o); o += al16(sizeof(double) * kNSub * 32);
  s.rh = reinterpret_cast<double*>(base + o); o += al16(sizeof(double) * kNSub * 32);
  s.xe = reinterpret_cast<int*>(base + o); o += al16(sizeof(int) * kNSub * 32);
  s.wsx = reinterpret_cast<int*>(base + o); o += al16(sizeof(int) * 32);
  s.cols = reinterpret_cast<int*>(base + o); o += al16(sizeof(int) * 32);
  s.sb = reinterpret_cast<int*>(base + o); o += al16(sizeof(int) * (kNSub + 1));
  s.fl = reinterpret_cast<signed char*>(base + o);
  return s;
}

// ------------------------------------------------------------------------------------
// Micro-solves (reading R9).  They take the current right-hand side values of the block,
// return the solution and the exponent k <= 0 of the power of two that the caller must
// apply to every OTHER value of the sub-tile (the returned values are already scaled).
// Arithmetic, operation order and protection are those of the warp-per-column kernel
// (zz_kernels.cu) and of the oracle's O7, so pivots are bit-identical (reading R17).
// ------------------------------------------------------------------------------------
template <bool PAIR>
__device__ __forceinline__ cpx pdiv_v(cpx z, cpx d, int& k) {
  if (!PAIR) {
    int e = protect_division(fabs(z.re), fabs(d.re));
    if (e < 0) { z.re = ldexp(z.re, e); k += e; }
    return mkc(__ddiv_rn(z.re, d.re), 0.0);
  }
  int e = protect_division(nmax(z), __dmul_rn(0.5, dmind(1.0, nmax(d))));
  if (e < 0) { z.re = ldexp(z.re, e); z.im = ldexp(z.im, e); k += e; }
  return cdivx(z, d);
}

// 1x1 row: (beta S_jj - alpha T_jj) x = w
template <bool PAIR>
__device__ __forceinline__ cpx micro1(cpx w, double sjj, double tjj, double a, double b, double beta, double ab,
                                   int& k) {
  cpx d = mkc(__fma_rn(-a, tjj, __dmul_rn(beta, sjj)), __dmul_rn(-b, tjj));
  double smin = dmaxd(__dmul_rn(kU, __dadd_rn(__dmul_rn(beta, fabs(sjj)), __dmul_rn(ab, fabs(tjj)))), kSmlnum);
  if (n1(d) < smin) d = mkc(smin, 0.0);
  k = 0;
  return pdiv_v<PAIR>(w, d, k);
}

// 2x2 rows (top, bot): complete pivoting on |Re|+|Im|, pivots below smin -> smin.
template <bool PAIR>
__device__ __forceinline__ void micro2(cpx& wt, cpx& wb, double s11, double s21, double s12, double s22, double t11,
                                    double t12, double t22, double a, double b, double beta, double ab, int& k) {
  cpx C[2][2];
  C[0][0] = mkc(__fma_rn(-a, t11, __dmul_rn(beta, s11)), __dmul_rn(-b, t11));
  C[1][0] = mkc(__dmul_rn(beta, s21), 0.0);
  C[0][1] = mkc(__fma_rn(-a, t12, __dmul_rn(beta, s12)), __dmul_rn(-b, t12));
  C[1][1] = mkc(__fma_rn(-a, t22, __dmul_rn(beta, s22)), __dmul_rn(-b, t22));
  double maxs = dmaxd(dmaxd(fabs(s11), fabs(s21)), dmaxd(fabs(s12), fabs(s22)));
  double maxt = dmaxd(dmaxd(fabs(t11), fabs(t12)), fabs(t22));
  double smin = dmaxd(__dmul_rn(kU, __dadd_rn(__dmul_rn(beta, maxs), __dmul_rn(ab, maxt))), kSmlnum);
  int pr = 0, pc = 0;
  double best = n1(C[0][0]);
  if (n1(C[1][0]) > best) { best = n1(C[1][0]); pr = 1; pc = 0; }
  if (n1(C[0][1]) > best) { best = n1(C[0][1]); pr = 0; pc = 1; }
  if (n1(C[1][1]) > best) { best = n1(C[1][1]); pr = 1; pc = 1; }
  cpx p = C[pr][pc];
  if (n1(p) < smin) p = mkc(smin, 0.0);
  cpx rr = C[1 - pr][pc], cc = C[pr][1 - pc], ss = C[1 - pr][1 - pc];
  cpx l = cdivx(rr, p);
  cpx u22 = csubx(ss, cmulx(l, cc));
  if (n1(u22) < smin) u22 = mkc(smin, 0.0);
  cpx w1 = pr ? wb : wt, w2 = pr ? wt : wb;
  k = 0;
  {
    double wn = dmaxd(nmax(w1), nmax(w2));
    int e = protect_update(wn, 2.0, wn);
    if (e < 0) {
      k += e;
      w1 = mkc(ldexp(w1.re, e), ldexp(w1.im, e));
      w2 = mkc(ldexp(w2.re, e), ldexp(w2.im, e));
    }
  }
  w2 = csubx(w2, cmulx(l, w1));
  int k0 = k;
  cpx z2 = pdiv_v<PAIR>(w2, u22, k);
  if (k != k0) w1 = mkc(ldexp(w1.re, k - k0), ldexp(w1.im, k - k0));
  {
    int e = protect_update(nmax(w1), n1(cc), nmax(z2));
    if (e < 0) {
      k += e;
      w1 = mkc(ldexp(w1.re, e), ldexp(w1.im, e));
      z2 = mkc(ldexp(z2.re, e), ldexp(z2.im, e));
    }
  }
  cpx nn = csubx(w1, cmulx(cc, z2));
  k0 = k;
  cpx z1 = pdiv_v<PAIR>(nn, p, k);
  if (k != k0) z2 = mkc(ldexp(z2.re, k - k0), ldexp(z2.im, k - k0));
  // z1 belongs to row top + pc, z2 to row top + 1 - pc
  if (pc == 0) { wt = z1; wb = z2; }
  else { wb = z1; wt = z2; }
}

template <bool PAIR>
__device__ __forceinline__ void scale_regs(double (&yr)[kSR], double (&yi)[kSR], int k) {
  while (k < -1022) {
#pragma unroll
    for (int i = 0; i < kSR; ++i) {
      yr[i] *= 0x1p-1022;
      if (PAIR) yi[i] *= 0x1p-1022;
    }
    k += 1022;
  }
  const double f = pow2i(k);
#pragma unroll
  for (int i = 0; i < kSR; ++i) {
    yr[i] *= f;
    if (PAIR) yi[i] *= f;
  }
}

// the same on the lane's column of a published sub-tile in shared memory (rows < n)
__device__ __forceinline__ void scale_smem(double2* x, int n, int k) {
  for (int i = 0; i < n; ++i) {
    double2 v = x[i * kXP];
    v.x = scale2(v.x, k);
    v.y = scale2(v.y, k);
    x[i * kXP] = v;
  }
}

template <bool PAIR>
__device__ __forceinline__ double max_rows(const double (&yr)[kSR], const double (&yi)[kSR], int n) {
  double m = 0.0;
#pragma unroll
  for (int i = 0; i < kSR; ++i)
    if (i < n) m = fmax(m, PAIR ? fmax(fabs(yr[i]), fabs(yi[i])) : fabs(yr[i]));
  return m;
}


// ------------------------------------------------------------------------------------
// One group of (up to) 32 eigenvectors of one kind.
// ------------------------------------------------------------------------------------
template <bool PAIR>
__device__ void run_group(const Diag2Params& p, const Sm& sm, int nsub, const int* items, int n_items,
                          int gbase, int warp, int lane) {
  const DevPlan& P = p.P;
  const int idx = gbase + lane;
  const bool valid = idx < n_items;
  const int c = valid ? items[idx] : -1;
  double a = 0.0, b = 0.0, beta = 0.0;
  bool tip = false;
  int tipr = -1;
  if (valid) {
    a = P.col_a[c];
    b = PAIR ? P.col_b[c] : 0.0;
    beta = P.col_beta[c];
    tip = c < p.tip_col_end;
    if (tip) tipr = P.col_r[c] - p.t0;
  }
  const double ab = __dadd_rn(fabs(a), fabs(b));
  if (warp == 0) sm.cols[lane] = c;

  double yr[kSR], yi[kSR];
  int ex = 0;
  const bool active = warp < nsub;
  const int r0 = active ? sm.sb[warp] : 0;
  const int len = active ? sm.sb[warp + 1] - r0 : 0;

  if (active) {
    // ---- right-hand side of this sub-tile (tips start from zero) ----
    const double* xc = p.X + (long long)(valid ? c : 0) * p.ldx + p.t0 + r0;
#pragma unroll
    for (int i = 0; i < kSR; ++i) {
      const bool ld = valid && !tip && i < len;
      yr[i] = ld ? xc[i] : 0.0;
      yi[i] = (PAIR && ld) ? xc[i + p.ldx] : 0.0;
    }
    // ---- block updates from the sub-tiles below (Alg. 3 per block) ----
    for (int k2 = nsub - 1; k2 > warp; --k2) {
      named_sync(1 + k2, 32 * (k2 + 1));
      const int c0 = sm.sb[k2], len2 = sm.sb[k2 + 1] - c0;
      const double xnv = sm.xn[k2 * 32 + lane];
      const int ek = sm.xe[k2 * 32 + lane];
      const double ymax = max_rows<PAIR>(yr, yi, len);
      const int g = min(ex, ek);
      const double yh = (g != ex) ? scale2(ymax, g - ex) : ymax;
      const double xh = (g != ek) ? scale2(xnv, g - ek) : xnv;
      const double2 nbv = sm.nb[warp * kNSub + k2];
      const double tau = __dadd_rn(__dmul_rn(beta, nbv.x), __dmul_rn(ab, nbv.y));
      const int en = g + protect_update(yh, tau, xh);
      if (en != ex) scale_regs<PAIR>(yr, yi, en - ex);
      ex = en;
      const int sx = en - ek;
      const double2* xsk = sm.xs + (k2 * kSR) * kXP + lane;
      for (int l = len2 - 1; l >= 0; --l) {
        const double2 xv = xsk[l * kXP];
        double xr = xv.x, xi = xv.y;
        if (sx != 0) { xr = scale2(xr, sx); xi = scale2(xi, sx); }
        // u = x D (beta x), w = x B (alpha x)
        const double ur = beta * xr, ui = beta * xi;
        const double wr = PAIR ? (a * xr - b * xi) : a * xr;
        const double wi = PAIR ? (a * xi + b * xr) : 0.0;
        const double2* col = sm.ST + poff2(c0 + l) + r0;
#pragma unroll
        for (int i = 0; i < kSR; ++i) {
          if (i < len) {
            const double2 st = col[i];
            yr[i] = fma(st.y, wr, fma(-st.x, ur, yr[i]));
            if (PAIR) yi[i] = fma(st.y, wi, fma(-st.x, ui, yi[i]));
          }
        }
      }
    }
    // ---- bottom-up substitution inside the sub-tile ----
    // The lane's column of the sub-tile moves to its slot of the exchange buffer, where the
    // row loop can index it at run time (short code; the structure is per row, so the
    // control flow stays uniform across the warp).
    double2* xw = sm.xs + (warp * kSR) * kXP + lane;
#pragma unroll
    for (int i = 0; i < kSR; ++i)
      if (i < len) xw[i * kXP] = make_double2(yr[i], PAIR ? yi[i] : 0.0);
    int j = len - 1;
    while (j >= 0) {
      const int gj = r0 + j;
      const bool two = sm.fl[gj] == kRowBot2;
      const int js = two ? j - 1 : j;
      int k = 0;
      cpx xt, xb;   // solution of rows js (top) and j (bottom)
      if (two) {
        const double2 d11 = sm.ST[poff2(gj - 1) + gj - 1], d21 = sm.ST[poff2(gj - 1) + gj];
        const double2 d12 = sm.ST[poff2(gj) + gj - 1], d22 = sm.ST[poff2(gj) + gj];
        const double2 vt = xw[(j - 1) * kXP], vb = xw[j * kXP];
        xt = mkc(vt.x, vt.y);
        xb = mkc(vb.x, vb.y);
        micro2<PAIR>(xt, xb, d11.x, d21.x, d12.x, d22.x, d11.y, d12.y, d22.y, a, b, beta, ab, k);
        if (PAIR && tip && tipr == gj) {
          // tip of a complex pair (reading R10): rows (r-1, r) of the eigenvalue block
          const double pp = __dmul_rn(beta, d21.x);
          const cpx q = mkc(__fma_rn(-a, d22.y, __dmul_rn(beta, d22.x)), __dmul_rn(-b, d22.y));
          if (fabs(pp) >= n1(q)) {
            xb = mkc(1.0, 0.0);
            xt = mkc(__ddiv_rn(-q.re, pp), __ddiv_rn(-q.im, pp));
          } else {
            xt = mkc(1.0, 0.0);
            const cpx z = cdivx(mkc(pp, 0.0), q);
            xb = mkc(-z.re, -z.im);
          }
          k = 0;
        }
      } else {
        const double2 d = sm.ST[poff2(gj) + gj];
        const double2 v = xw[j * kXP];
        xb = micro1<PAIR>(mkc(v.x, v.y), d.x, d.y, a, b, beta, ab, k);
        if (!PAIR && tip && tipr == gj) { xb = mkc(1.0, 0.0); k = 0; }
        xt = xb;
      }
      if (k < 0) { scale_smem(xw, len, k); ex += k; }
      // in-sub-tile update of the rows above the block (ProtectUpdate)
      if (js > 0) {
        double t = 0.0;
        for (int kk = js; kk <= j; ++kk) {
          const double2 cmv = sm.cm[r0 + kk];
          t = __dadd_rn(t, __dadd_rn(__dmul_rn(beta, cmv.x), __dmul_rn(ab, cmv.y)));
        }
        double xnb = PAIR ? nmax(xb) : fabs(xb.re);
        if (two) xnb = dmaxd(PAIR ? nmax(xt) : fabs(xt.re), xnb);
        double ym = 0.0;
        for (int i = 0; i < js; ++i) {
          const double2 v = xw[i * kXP];
          ym = fmax(ym, PAIR ? fmax(fabs(v.x), fabs(v.y)) : fabs(v.x));
        }
        const int eu = protect_update(ym, t, xnb);
        if (eu < 0) {
          scale_smem(xw, len, eu);   // the whole sub-tile: solved rows too
          ex += eu;
          xt = mkc(scale2(xt.re, eu), scale2(xt.im, eu));
          xb = mkc(scale2(xb.re, eu), scale2(xb.im, eu));
        }
        // sources in ascending row order, as the oracle's O6
        for (int s2 = two ? 0 : 1; s2 < 2; ++s2) {
          const cpx x = s2 ? xb : xt;
          const double ur = beta * x.re, ui = beta * x.im;
          const double wr = PAIR ? (a * x.re - b * x.im) : a * x.re;
          const double wi = PAIR ? (a * x.im + b * x.re) : 0.0;
          const double2* col = sm.ST + poff2(r0 + (s2 ? j : js)) + r0;
#pragma unroll 4
          for (int i = 0; i < js; ++i) {
            const double2 st = col[i];
            double2 v = xw[i * kXP];
            v.x = fma(st.y, wr, fma(-st.x, ur, v.x));
            if (PAIR) v.y = fma(st.y, wi, fma(-st.x, ui, v.y));
            xw[i * kXP] = v;
          }
        }
      }
      if (two) xw[(j - 1) * kXP] = make_double2(xt.re, PAIR ? xt.im : 0.0);
      xw[j * kXP] = make_double2(xb.re, PAIR ? xb.im : 0.0);
      j = js - 1;
    }
    // ---- publish the solved sub-tile (already in place in the exchange buffer) ----
    double xm = 0.0;
#pragma unroll
    for (int i = 0; i < kSR; ++i) {
      if (i < len) {
        const double2 v = xw[i * kXP];
        yr[i] = v.x;
        yi[i] = v.y;
        xm = fmax(xm, PAIR ? fmax(fabs(v.x), fabs(v.y)) : fabs(v.x));
      }
    }
    sm.xn[warp * 32 + lane] = xm;
    sm.xe[warp * 32 + lane] = ex;
    if (warp > 0) {
      __threadfence_block();
      named_arrive(1 + warp, 32 * (warp + 1));
    }
  }
  __syncthreads();
  // ---- consistency inside the segment: one exponent per (tile, column) ----
  int emin = 0;
  for (int k = 0; k < nsub; ++k) emin = min(emin, sm.xe[k * 32 + lane]);
  if (active) {
    if (emin != ex) scale_regs<PAIR>(yr, yi, emin - ex);
    double lm = 0.0, lh = 0.0;
    double2* xo = sm.xs + (warp * kSR) * kXP + lane;
#pragma unroll
    for (int i = 0; i < kSR; ++i) {
      if (i < len) {
        xo[i * kXP] = make_double2(yr[i], PAIR ? yi[i] : 0.0);
        lm = fmax(lm, PAIR ? fmax(fabs(yr[i]), fabs(yi[i])) : fabs(yr[i]));
        lh = fmax(lh, PAIR ? __dadd_rn(__dmul_rn(0.5, fabs(yr[i])), __dmul_rn(0.5, fabs(yi[i])))
                           : __dmul_rn(0.5, fabs(yr[i])));
      }
    }
    sm.rn[warp * 32 + lane] = lm;
    sm.rh[warp * 32 + lane] = lh;
  }
  __syncthreads();
  // ---- coalesced store of the segment: warp k writes sub-tile k column by column ----
  if (active) {
    for (int q = 0; q < 32; ++q) {
      const int cq = sm.cols[q];
      if (cq < 0) break;
      if (lane < len) {
        const double2 v = sm.xs[(warp * kSR + lane) * kXP + q];
        double* dst = p.X + (long long)cq * p.ldx + p.t0 + r0 + lane;
        dst[0] = v.x;
        if (PAIR) dst[p.ldx] = v.y;
      }
    }
  }
  // ---- segment exponent, norms and the scaling decision of the next update (a5) ----
  if (warp == 0 && valid) {
    double nrm = 0.0, nrmh = 0.0;
    for (int k = 0; k < nsub; ++k) {
      nrm = fmax(nrm, sm.rn[k * 32 + lane]);
      nrmh = fmax(nrmh, sm.rh[k * 32 + lane]);
    }
    const int ep = tip ? 0 : P.e_pend[c];
    const int es = ep + emin;
    const long long so = (long long)p.I * p.n_sel + c;
    P.e_seg[so] = es;
    P.nrm_seg[so] = nrm;
    P.nrmh_seg[so] = nrmh;
    if (PAIR) { P.e_seg[so + 1] = es; P.nrm_seg[so + 1] = nrm; P.nrmh_seg[so + 1] = nrmh; }
    if (p.do_update) {
      // Alg. 3 with Alg. 2, reading R5
      const double nyv = tip ? 0.0 : __longlong_as_double((long long)P.nY[(long long)p.nY_in * p.n_sel + c]);
      const int g = min(ep, es);
      const double yh = scale2(nyv, g - ep), xh = scale2(nrm, g - es);
      const double tau = __dadd_rn(__dmul_rn(beta, P.cS[p.I]), __dmul_rn(ab, P.cT[p.I]));
      const int en = g + protect_update(yh, tau, xh);
      sm.wsx[lane] = en - es;
      P.sY[c] = en - ep;
      P.e_pend[c] = en;
      P.nY[(long long)(1 - p.nY_in) * p.n_sel + c] = 0ull;
      if (PAIR) {
        P.sY[c + 1] = en - ep;
        P.e_pend[c + 1] = en;
        P.nY[(long long)(1 - p.nY_in) * p.n_sel + c + 1] = 0ull;
      }
    }
  }
  if (p.do_update) {
    __syncthreads();
    // ---- B operand of the update: W = [-2^sx X_I D ; 2^sx X_I B], in the
    // update kernel's stage layout [ntile][kc][BK/4][BN][4] ----
    if (valid && active) {
      const int sx = sm.wsx[lane];
      const double fx = (sx >= -1022) ? pow2i(sx) : 0.0;
      const long long tstride = (long long)(2 * p.nks) * (kBN * kBK);
      double* Wc = P.W + (long long)(c / kBN) * tstride + (c % kBN) * 4;
      double* Wc1 = P.W + (long long)((c + 1) / kBN) * tstride + ((c + 1) % kBN) * 4;
      const long long half = (long long)p.nks * (kBN * kBK);
#pragma unroll
      for (int i = 0; i < kSR; ++i) {
        if (i < len) {
          const int kr = r0 + i;
          const long long o = (long long)(kr / kBK) * (kBN * kBK) + (long long)((kr % kBK) >> 2) * (kBN * 4) + (kr & 3);
          const double xr = (sx >= -1022) ? yr[i] * fx : scale2_slow(yr[i], sx);
          if (!PAIR) {
            Wc[o] = -(beta * xr);
            Wc[o + half] = a * xr;
          } else {
            const double xi = (sx >= -1022) ? yi[i] * fx : scale2_slow(yi[i], sx);
            Wc[o] = -(beta * xr);
            Wc1[o] = -(beta * xi);
            Wc[o + half] = a * xr - b * xi;
            Wc1[o + half] = b * xr + a * xi;
          }
        }
      }
      // zero rows nt .. nks*BK-1 (the K padding of the last chunk)
      if (warp == nsub - 1) {
        for (int kr = p.nt; kr < p.nks * kBK; ++kr) {
          const long long o = (long long)(kr / kBK) * (kBN * kBK) + (long long)((kr % kBK) >> 2) * (kBN * 4) + (kr & 3);
          Wc[o] = 0.0;
          Wc[o + half] = 0.0;
          if (PAIR) { Wc1[o] = 0.0; Wc1[o + half] = 0.0; }
        }
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kDW * 32, 1) k_diag2(Diag2Params p) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int nt = p.nt;
  Sm sm = carve(smraw, nt);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // ---- stage the diagonal tile: (S_ij, T_ij) for i <= j, (S_{j+1,j}, 0) below ----
  for (int j = warp; j < nt; j += kDW) {
    const int len = min(j + 2, nt);
    const double* sc = p.S + (long long)(p.t0 + j) * p.lds + p.t0;
    const double* tc = p.T + (long long)(p.t0 + j) * p.ldt + p.t0;
    for (int i = lane; i < len; i += 32) sm.ST[poff2(j) + i] = make_double2(sc[i], i <= j ? tc[i] : 0.0);
  }
  for (int i = threadIdx.x; i < nt; i += blockDim.x) sm.fl[i] = p.P.row_flag[p.t0 + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    int k = 0;
    sm.sb[0] = 0;
    while (sm.sb[k] < nt) {
      int nx = 16 * (k + 1);
      if (nx >= nt) nx = nt;
      else if (sm.fl[nx] == kRowBot2) nx += 1;
      sm.sb[++k] = nx;
    }
    for (int q = k + 1; q <= kNSub; ++q) sm.sb[q] = nt;
  }
  __syncthreads();
  int nsub = 0;
  while (nsub < kNSub && sm.sb[nsub] < nt) ++nsub;
  // in-sub-tile column bounds: rows of j's sub-tile above j's block (reading R6)
  for (int j = threadIdx.x; j < nt; j += blockDim.x) {
    int k = 0;
    while (sm.sb[k + 1] <= j) ++k;
    const int top = (sm.fl[j] == kRowBot2) ? j - 1 : j;
    double ms = 0.0, mt = 0.0;
    for (int i = sm.sb[k]; i < top; ++i) {
      const double2 v = sm.ST[poff2(j) + i];
      ms = fmax(ms, fabs(v.x));
      mt = fmax(mt, fabs(v.y));
    }
    sm.cm[j] = make_double2(ms, mt);
  }
  // block infinity norms: max over rows of sub-tile k of the row sums over sub-tile k2
  for (int pr = warp; pr < kNSub * kNSub; pr += kDW) {
    const int k = pr / kNSub, k2 = pr % kNSub;
    if (k >= k2 || k2 >= nsub) continue;
    const int i = sm.sb[k] + lane;
    double s = 0.0, t = 0.0;
    if (i < sm.sb[k + 1]) {
      for (int l = sm.sb[k2]; l < sm.sb[k2 + 1]; ++l) {
        const double2 v = sm.ST[poff2(l) + i];
        s += fabs(v.x);
        t += fabs(v.y);
      }
    }
    for (int o = 16; o; o >>= 1) {
      s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
      t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    }
    if (lane == 0) sm.nb[k * kNSub + k2] = make_double2(s, t);
  }
  __syncthreads();
  // ---- groups of 32 eigenvectors: complex pairs first, then real columns ----
  const int npg = (p.n_pair + 31) / 32, nrg = (p.n_real + 31) / 32;
  for (int g = blockIdx.x; g < npg + nrg; g += gridDim.x) {
    if (g < npg) run_group<true>(p, sm, nsub, p.pair_items, p.n_pair, g * 32, warp, lane);
    else run_group<false>(p, sm, nsub, p.real_items, p.n_real, (g - npg) * 32, warp, lane);
  }
}

int g_sms = 0;

}  // namespace

size_t diag2_smem_bytes(int nt) { return smem_need(nt); }

cudaError_t launch_diag2(const Diag2Params& p, cudaStream_t st) {
  const int groups = (p.n_pair + 31) / 32 + (p.n_real + 31) / 32;
  if (groups == 0) return cudaSuccess;
  if (p.nt > kDiag2MaxNT) return cudaErrorInvalidValue;
  if (!g_sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = smem_need(p.nt);
  cudaError_t e = cudaFuncSetAttribute(k_diag2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = groups < g_sms ? groups : g_sms;
  k_diag2<<<grid, kDW * 32, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace zz
