// zz_diag3.cu -- the robust diagonal-block solve (Kernel 1 tips and Kernel 3 right-hand
// sides; Alg. 1 lines P:137) for tiles of at most 128
// rows, fused with the per-column scaling decision of the following update (Algs. 2/3,
// PAPER.md:216-262) and the formation of the update's B operand W.
//
// B200 design.  A warp solves 8 columns at once (8 real eigenvector columns, or 4 complex
// pairs as (Re, Im) column couples), 4 lanes per column.  The tile's rows live in
// registers in the accumulator layout of the FP64 tensor instruction
// mma.m8n8k4.f64 (DMMA.8x8x4): for 8-row group g, lane (team = column, t) holds rows
// 8g + 2t and 8g + 2t + 1.  The solve walks the tile bottom-up in blocks of 8 rows
// (block boundaries never split a 2x2 block):
//   * inside a block, rows are solved one 1x1 / 2x2 block at a time; the 4 lanes of a
//     column compute the division redundantly (the pivot beta S_jj - alpha T_jj is per
//     column, S_jj and T_jj are shared-memory broadcasts) and update the block's rows;
//   * the block's solution then updates every row above it inside the tile with DMMA:
//     Y(8 cols x 8 rows) += [-beta x | alpha x]^T (8 cols x 4) . [S | T]^T (4 x 8 rows),
//     two (real) or two per component (pairs) DMMAs per 4 source rows and 8 target rows.
// The shifted matrix differs per column, but the update is linear in the columns: only
// the 1x1 / 2x2 divisions are per column.
//
// Robustness: one power-of-two exponent per (tile, column) (Definition 1);
// every division is protected by ProtectDivision, every update by ProtectUpdate against a
// running upper bound of the pending rows (exact maximum recomputed whenever the bound
// would trigger a scaling, so decisions equal those of the exact maximum); a scaling
// multiplies the whole segment by a power of two (exact).
#include <math.h>
#include <stdint.h>

#include "zz_internal.cuh"
#include "zz_device.cuh"

namespace zz {

namespace {

// warps per CTA: G = 16 (tiles of 65..128 rows) needs ~170 registers per lane
template <int G> struct W3 { static constexpr int n = (G > 8) ? 12 : 16; };
constexpr int kPad3 = 32;      // zero double2 padding after the packed tile

__device__ __forceinline__ int poff3(int j) { return j * (j + 3) / 2; }

__device__ __forceinline__ double pow2k(int k) { return __hiloint2double((k + 1023) << 20, 0); }
__device__ __forceinline__ double scale2_slow3(double x, int k) {
  while (k < -1022) { x *= 0x1p-1022; k += 1022; }
  return x * pow2k(k);
}
__device__ __forceinline__ double scale2k(double x, int k) { return k >= -1022 ? x * pow2k(k) : scale2_slow3(x, k); }

__device__ __forceinline__ void dmma3(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct Sm3 {
  double2* ST;     // packed tile: (S_ij, T_ij) at poff3(j) + i, rows i <= j + 1
  double2* cm;     // per row j: max |S_ij|, |T_ij| over the tile rows above j's block (R6)
  double2* tau;    // per block b: max over rows i < s_b of the sums over the block's rows
  int* bs;         // block b = rows [bs[b], bs[b+1]); bs[b] = 8b - (row 8b is a 2x2 bottom)
  double* slab;    // per warp: the current block's rows, [9 slots][8 columns]
  double* pslab;   // per warp: prepared pivots of the block's 1x1 rows, [9][8][8]
  signed char* fl; // row flags
};

__host__ __device__ __forceinline__ size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ __forceinline__ size_t smem3(int nt) {
  return a16(sizeof(double2) * (size_t)(nt * (nt + 3) / 2 + kPad3)) + a16(sizeof(double2) * (size_t)nt) +
         a16(sizeof(double2) * 17) + a16(sizeof(int) * 18) + a16(sizeof(double) * 16 * 72) + a16(sizeof(double) * 16 * 576) + a16((size_t)nt);
}
__device__ __forceinline__ Sm3 carve3(unsigned char* base, int nt) {
  Sm3 s;
  size_t o = 0;
  s.ST = reinterpret_cast<double2*>(base + o); o += a16(sizeof(double2) * (size_t)(nt * (nt + 3) / 2 + kPad3));
  s.cm = reinterpret_cast<double2*>(base + o); o += a16(sizeof(double2) * (size_t)nt);
  s.tau = reinterpret_cast<double2*>(base + o); o += a16(sizeof(double2) * 17);
  s.bs = reinterpret_cast<int*>(base + o); o += a16(sizeof(int) * 18);
  s.slab = reinterpret_cast<double*>(base + o); o += a16(sizeof(double) * 16 * 72);
  s.pslab = reinterpret_cast<double*>(base + o); o += a16(sizeof(double) * 16 * 576);
  s.fl = reinterpret_cast<signed char*>(base + o);
  return s;
}

// ------------------------------------------------------------------------------------
// Micro-solves (reading R9): same arithmetic, order and protection as the oracle's O7 and
// the warp-per-column kernel, so the pivots are bit-identical (reading R17).  They return
// the solution (already scaled) and the exponent k <= 0 to apply to all other values.
// ------------------------------------------------------------------------------------
template <bool PAIR>
__device__ __forceinline__ cpx pdiv3(cpx z, cpx d, int& k) {
  if (!PAIR) {
    int e = protect_division(fabs(z.re), fabs(d.re));
    if (e < 0) { z.re = scale2k(z.re, e); k += e; }
    return mkc(__ddiv_rn(z.re, d.re), 0.0);
  }
  int e = protect_division(nmax(z), __dmul_rn(0.5, dmind(1.0, nmax(d))));
  if (e < 0) { z.re = scale2k(z.re, e); z.im = scale2k(z.im, e); k += e; }
  return cdivx(z, d);
}

template <bool PAIR>
__device__ __forceinline__ cpx solve1x1(cpx w, double sjj, double tjj, double a, double b, double beta,
                                        double ab, int& k) {
  cpx d = mkc(__fma_rn(-a, tjj, __dmul_rn(beta, sjj)), __dmul_rn(-b, tjj));
  double smin = dmaxd(__dmul_rn(kU, __dadd_rn(__dmul_rn(beta, fabs(sjj)), __dmul_rn(ab, fabs(tjj)))), kSmlnum);
  if (n1(d) < smin) d = mkc(smin, 0.0);
  k = 0;
  return pdiv3<PAIR>(w, d, k);
}

template <bool PAIR>
__device__ __forceinline__ void solve2x2(cpx& wt, cpx& wb, double s11, double s21, double s12, double s22,
                                         double t11, double t12, double t22, double a, double b, double beta,
                                         double ab, int& k) {
  // C = beta S_blk - alpha T_blk, complete pivoting on |Re| + |Im| (no indexed arrays: the
  // entries stay in registers)
  const cpx c00 = mkc(__fma_rn(-a, t11, __dmul_rn(beta, s11)), __dmul_rn(-b, t11));
  const cpx c10 = mkc(__dmul_rn(beta, s21), 0.0);
  const cpx c01 = mkc(__fma_rn(-a, t12, __dmul_rn(beta, s12)), __dmul_rn(-b, t12));
  const cpx c11 = mkc(__fma_rn(-a, t22, __dmul_rn(beta, s22)), __dmul_rn(-b, t22));
  double maxs = dmaxd(dmaxd(fabs(s11), fabs(s21)), dmaxd(fabs(s12), fabs(s22)));
  double maxt = dmaxd(dmaxd(fabs(t11), fabs(t12)), fabs(t22));
  double smin = dmaxd(__dmul_rn(kU, __dadd_rn(__dmul_rn(beta, maxs), __dmul_rn(ab, maxt))), kSmlnum);
  int pr = 0, pc = 0;
  double best = n1(c00);
  if (n1(c10) > best) { best = n1(c10); pr = 1; pc = 0; }
  if (n1(c01) > best) { best = n1(c01); pr = 0; pc = 1; }
  if (n1(c11) > best) { best = n1(c11); pr = 1; pc = 1; }
  auto pick = [&](int r, int q) -> cpx { return r ? (q ? c11 : c10) : (q ? c01 : c00); };
  cpx p = pick(pr, pc);
  if (n1(p) < smin) p = mkc(smin, 0.0);
  const cpx rr = pick(1 - pr, pc), cc = pick(pr, 1 - pc), ss = pick(1 - pr, 1 - pc);
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
      w1 = mkc(scale2k(w1.re, e), scale2k(w1.im, e));
      w2 = mkc(scale2k(w2.re, e), scale2k(w2.im, e));
    }
  }
  w2 = csubx(w2, cmulx(l, w1));
  int k0 = k;
  cpx z2 = pdiv3<PAIR>(w2, u22, k);
  if (k != k0) w1 = mkc(scale2k(w1.re, k - k0), scale2k(w1.im, k - k0));
  {
    int e = protect_update(nmax(w1), n1(cc), nmax(z2));
    if (e < 0) {
      k += e;
      w1 = mkc(scale2k(w1.re, e), scale2k(w1.im, e));
      z2 = mkc(scale2k(z2.re, e), scale2k(z2.im, e));
    }
  }
  cpx nn = csubx(w1, cmulx(cc, z2));
  k0 = k;
  cpx z1 = pdiv3<PAIR>(nn, p, k);
  if (k != k0) z2 = mkc(scale2k(z2.re, k - k0), scale2k(z2.im, k - k0));
  if (pc == 0) { wt = z1; wb = z2; }
  else { wb = z1; wt = z2; }
}

// ------------------------------------------------------------------------------------
// Per-lane register file of one column segment, rotated so that the block being solved
// always sits at position G-1 (static register indices; a select over a run-time group
// index would push the array to local memory).  Position p holds group (p - rot) mod G.
// ------------------------------------------------------------------------------------
template <int G>
struct Seg {
  double y[G][2];   // lane t: rows 8g + 2t, 8g + 2t + 1 of group g
  __device__ __forceinline__ void rotate() {   // group at position p moves to p + 1 (mod G)
    const double l0 = y[G - 1][0], l1 = y[G - 1][1];
#pragma unroll
    for (int q = G - 1; q > 0; --q) { y[q][0] = y[q - 1][0]; y[q][1] = y[q - 1][1]; }
    y[0][0] = l0;
    y[0][1] = l1;
  }
  __device__ __forceinline__ void scale(int k) {
    while (k < -1022) {
#pragma unroll
      for (int q = 0; q < G; ++q) { y[q][0] *= 0x1p-1022; y[q][1] *= 0x1p-1022; }
      k += 1022;
    }
    const double f = pow2k(k);
#pragma unroll
    for (int q = 0; q < G; ++q) { y[q][0] *= f; y[q][1] *= f; }
  }
};

// max |value| over the pending rows (< lim) of the column, given that position p holds
// group (p - rot) mod G (pairs: over both components)
template <int G, bool PAIR>
__device__ __forceinline__ double pending_max(const Seg<G>& s, int rot, int t, int lim) {
  double m = 0.0;
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int g = (q - rot + G) % G;
    const int r = 8 * g + 2 * t;
    if (r < lim) m = fmax(m, fabs(s.y[q][0]));
    if (r + 1 < lim) m = fmax(m, fabs(s.y[q][1]));
  }
  m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 1));
  m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 2));
  if (PAIR) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 4));
  return m;
}

// ------------------------------------------------------------------------------------
// One task: 8 real columns (PAIR = false) or 4 complex pairs (PAIR = true) of tile I.
// ------------------------------------------------------------------------------------
template <int G, bool PAIR>
__device__ void solve_task(const Diag2Params& p, const Sm3& sm, int nblk, int task, int lane, double* wslab,
                           double* pslab) {
  const DevPlan& P = p.P;
  const int team = lane >> 2, t = lane & 3;
  const int comp = PAIR ? (team & 1) : 0;
  // cpt columns per task (8, 4 or 2: fewer when the step has few columns, so that more
  // warps run; a column's arithmetic does not depend on the other columns of its warp)
  const int cpt = p.cpt;
  const int slot = PAIR ? (team >> 1) : team;
  const int item = PAIR ? task * (cpt / 2) + slot : task * cpt + slot;
  const int n_items = PAIR ? p.n_pair : p.n_real;
  const bool valid = item < n_items && slot < (PAIR ? cpt / 2 : cpt);
  const int c0 = valid ? (PAIR ? p.pair_items[item] : p.real_items[item]) : -1;
  const int c = c0 + comp;                       // this lane's output column
  double a = 0.0, b = 0.0, beta = 0.0;
  bool tip = false;
  int tipr = -1;
  if (valid) {
    a = P.col_a[c0];
    b = PAIR ? P.col_b[c0] : 0.0;
    beta = P.col_beta[c0];
    tip = c0 < p.tip_col_end;
    if (tip) tipr = P.col_r[c0] - p.t0;
  }
  const double ab = __dadd_rn(fabs(a), fabs(b));
  const int nt = p.nt;
  const int pbase = lane & ~3;           // first lane of this column's team
  constexpr int CUR = G - 1, PRV = G - 2;

  // ---- right-hand side (tips start from zero) ----
  Seg<G> s;
  {
    const double* xc = p.X + (long long)(valid ? c : 0) * p.ldx + p.t0;
    const bool ld = valid && !tip;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int r = 8 * g + 2 * t;
      s.y[g][0] = (ld && r < nt) ? xc[r] : 0.0;
      s.y[g][1] = (ld && r + 1 < nt) ? xc[r + 1] : 0.0;
    }
  }
  int rot = 0;
  while (rot < G - nblk) { s.rotate(); ++rot; }   // group nblk-1 -> position G-1
  int ex = 0;   // exponent of the segment relative to e_pend (stored = 2^ex true)
  double bound = pending_max<G, PAIR>(s, rot, t, nt);   // running bound of max |pending|

  for (int blk = nblk - 1; blk >= 0; --blk) {
    const int s0 = sm.bs[blk], e0 = sm.bs[blk + 1];
    const int g8 = 8 * blk;
    const bool st = s0 < g8;             // row 8 blk - 1 (a 2x2 top) belongs to this block
    double xnb = 0.0;                    // max |x| over the block's solved rows
    // ---- bottom-up substitution inside the block ----
    // The block's rows go to a per-warp shared-memory slab (slot q = row 8 blk - 1 + q; slot
    // 0 is the top of a straddling 2x2 block; entry [q][team] = this column's value) where
    // the row loop indexes them at run time.  All 4 lanes of a column (and both columns of
    // a pair) compute identical values, hence identical decisions, and store identical
    // values.
    __syncwarp();
    wslab[(1 + 2 * t) * 8 + team] = s.y[CUR][0];
    wslab[(2 + 2 * t) * 8 + team] = s.y[CUR][1];
    if (t == 3) wslab[team] = s.y[PRV][1];
    const int q0 = s0 - (g8 - 1);
    // pivots of the block's 1x1 rows, off the dependency chain: lane t prepares slots t,
    // t+4, t+8 of its column -- the perturbed pivot d (R8), its reciprocal (real) or Smith's
    // ratio and denominator (pair), and the ProtectDivision threshold (|w| <= thr: no scaling)
    for (int q = t; q < 9; q += 4) {
      const int j = g8 - 1 + q;
      if (q < q0 || j >= e0 || sm.fl[j] != kRow1x1) continue;
      const double2 dd = sm.ST[poff3(j) + j];
      cpx d = mkc(__fma_rn(-a, dd.y, __dmul_rn(beta, dd.x)), __dmul_rn(-b, dd.y));
      const double smin =
          dmaxd(__dmul_rn(kU, __dadd_rn(__dmul_rn(beta, fabs(dd.x)), __dmul_rn(ab, fabs(dd.y)))), kSmlnum);
      if (n1(d) < smin) d = mkc(smin, 0.0);
      double* pd = pslab + (q * 8 + team) * 8;
      pd[0] = d.re;
      pd[1] = d.im;
      if (!PAIR) {
        const double td = fabs(d.re);
        pd[2] = __drcp_rn(d.re);
        pd[3] = (td >= 1.0) ? INFINITY : __dmul_rn(td, kOmega);
      } else {
        const double td = __dmul_rn(0.5, dmind(1.0, nmax(d)));
        const bool re_dom = fabs(d.re) >= fabs(d.im);
        const double sr = re_dom ? __ddiv_rn(d.im, d.re) : __ddiv_rn(d.re, d.im);
        const double den = re_dom ? __dadd_rn(d.re, __dmul_rn(d.im, sr)) : __dadd_rn(d.im, __dmul_rn(d.re, sr));
        pd[2] = sr;
        pd[3] = den;
        pd[4] = __drcp_rn(den);
        pd[5] = re_dom ? 1.0 : 0.0;
        pd[6] = (td >= 1.0) ? INFINITY : __dmul_rn(td, kOmega);
      }
    }
    __syncwarp();
    int j = e0 - 1;
    int kseg = 0;
    while (j >= s0) {
      const int q = j - (g8 - 1);
      const bool two = sm.fl[j] == kRowBot2;
      const int qs = two ? q - 1 : q;
      const int pt = PAIR ? (team & ~1) : team;     // (Re, Im) entries of the pair
      int k = 0;
      cpx xt, xb;
      {
        cpx wb = mkc(wslab[q * 8 + pt], PAIR ? wslab[q * 8 + pt + 1] : 0.0);
        if (two) {
          cpx wt = mkc(wslab[(q - 1) * 8 + pt], PAIR ? wslab[(q - 1) * 8 + pt + 1] : 0.0);
          const double2 d11 = sm.ST[poff3(j - 1) + j - 1], d21 = sm.ST[poff3(j - 1) + j];
          const double2 d12 = sm.ST[poff3(j) + j - 1], d22 = sm.ST[poff3(j) + j];
          solve2x2<PAIR>(wt, wb, d11.x, d21.x, d12.x, d22.x, d11.y, d12.y, d22.y, a, b, beta, ab, k);
          if (PAIR && tip && tipr == j) {
            // tip of a complex pair (reading R10): rows (r-1, r) of the eigenvalue block
            const double pp = __dmul_rn(beta, d21.x);
            const cpx qq = mkc(__fma_rn(-a, d22.y, __dmul_rn(beta, d22.x)), __dmul_rn(-b, d22.y));
            if (fabs(pp) >= n1(qq)) {
              wb = mkc(1.0, 0.0);
              wt = mkc(__ddiv_rn(-qq.re, pp), __ddiv_rn(-qq.im, pp));
            } else {
              wt = mkc(1.0, 0.0);
              const cpx z = cdivx(mkc(pp, 0.0), qq);
              wb = mkc(-z.re, -z.im);
            }
            k = 0;
          }
          xt = wt;
          xb = wb;
        } else {
          // (beta S_jj - alpha T_jj) x = w with the prepared pivot: q = w r corrected once by
          // the residual (the quotient of __ddiv_rn); scaling only past the threshold
          const double* pd = pslab + (q * 8 + team) * 8;
          const cpx d = mkc(pd[0], pd[1]);
          if (!PAIR) {
            const double r = pd[2];
            if (fabs(wb.re) <= pd[3]) {
              const double x0 = wb.re * r;
              xb = mkc(fma(r, fma(-d.re, x0, wb.re), x0), 0.0);
            } else {
              xb = pdiv3<false>(wb, d, k);
            }
          } else {
            if (nmax(wb) <= pd[6]) {
              const double sr = pd[2], den = pd[3], rd = pd[4];
              const double n1v = (pd[5] != 0.0) ? __dadd_rn(wb.re, __dmul_rn(wb.im, sr))
                                                : __dadd_rn(__dmul_rn(wb.re, sr), wb.im);
              const double n2v = (pd[5] != 0.0) ? __dsub_rn(wb.im, __dmul_rn(wb.re, sr))
                                                : __dsub_rn(__dmul_rn(wb.im, sr), wb.re);
              const double y1 = n1v * rd, y2 = n2v * rd;
              xb = mkc(fma(rd, fma(-den, y1, n1v), y1), fma(rd, fma(-den, y2, n2v), y2));
            } else {
              xb = pdiv3<true>(wb, d, k);
            }
          }
          if (!PAIR && tip && tipr == j) { xb = mkc(1.0, 0.0); k = 0; }
          xt = xb;
        }
      }
      // scalars follow the solve's scaling at once; the stored values once (below)
      if (k < 0) {
        bound = scale2k(bound, k);
        xnb = scale2k(xnb, k);
      }
      double xn = two ? dmaxd(nmax(xt), nmax(xb)) : nmax(xb);
      int eu = 0;
      double tt = 0.0;
      const bool upd = qs > q0;
      if (upd) {
        // in-block update of the block rows above (ProtectUpdate) against a running
        // upper bound of the pending rows; lane-local (every lane holds the same values)
        const double2 cmv = sm.cm[j];
        tt = __dadd_rn(__dmul_rn(beta, cmv.x), __dmul_rn(ab, cmv.y));
        double nb = fma(tt, xn, bound);
        if (!(nb <= 0x1p1020)) {
          eu = protect_update(bound, tt, xn);
          nb = __dadd_rn(scale2k(bound, eu), __dmul_rn(tt, scale2k(xn, eu)));
        }
        bound = nb;
      }
      if (k + eu < 0) {
        // the whole segment by 2^(k+eu): the block's rows in the slab now, the rows in
        // registers once after the row loop (kseg) -- s.y is then not modified inside the
        // loop, so it keeps its registers (no copies around the loop; powers of two)
        const int kk = k + eu;
        kseg += kk;
        // slot r of the slab is always written by lane r & 3 of its column (here and in the
        // update below), so no warp barrier is needed in this column-divergent branch
        for (int r = t; r < 9; r += 4) wslab[r * 8 + team] = scale2k(wslab[r * 8 + team], kk);
        ex += kk;
        if (eu < 0) {
          xnb = scale2k(xnb, eu);
          xn = scale2k(xn, eu);
          xt = mkc(scale2k(xt.re, eu), scale2k(xt.im, eu));
          xb = mkc(scale2k(xb.re, eu), scale2k(xb.im, eu));
        }
      }
      xnb = dmaxd(xnb, xn);
      if (upd) {
        // sources in ascending row order, as the oracle's O6; each lane updates the rows of
        // its column (4 lanes split the rows)
#pragma unroll
        for (int sidx = 0; sidx < 2; ++sidx) {
          if (sidx == 0 && !two) continue;
          const cpx x = sidx ? xb : xt;
          const double xo = PAIR ? (comp ? x.im : x.re) : x.re;
          const double ur = beta * xo;
          const double wr = PAIR ? (comp ? (a * x.im + b * x.re) : (a * x.re - b * x.im)) : a * x.re;
          const double2* col = sm.ST + poff3(sidx ? j : j - 1) + (g8 - 1);
          for (int r = q0 + ((t - q0) & 3); r < qs; r += 4) {
            const double2 v = col[r];
            wslab[r * 8 + team] = fma(v.y, wr, fma(-v.x, ur, wslab[r * 8 + team]));
          }
        }
      }
      // the solution into the slab (own component; slot r by lane r & 3)
      if (t == (q & 3)) wslab[q * 8 + team] = PAIR ? (comp ? xb.im : xb.re) : xb.re;
      if (two && t == ((q - 1) & 3)) wslab[(q - 1) * 8 + team] = PAIR ? (comp ? xt.im : xt.re) : xt.re;
      __syncwarp();
      j = qs - 1 + (g8 - 1);
    }
    // ---- the block's rows back to their owner lanes ----
    if (kseg < 0) s.scale(kseg);
    s.y[CUR][0] = wslab[(1 + 2 * t) * 8 + team];
    s.y[CUR][1] = wslab[(2 + 2 * t) * 8 + team];
    if (st && t == 3) s.y[PRV][1] = wslab[team];
    __syncwarp();
    if (blk > 0) {
      // ---- update of all rows above the block by DMMA (Alg. 3 on the in-tile panel) ----
      const double2 tv = sm.tau[blk];
      const double tt = __dadd_rn(__dmul_rn(beta, tv.x), __dmul_rn(ab, tv.y));
      double nb = fma(tt, xnb, bound);
      if (__any_sync(0xffffffffu, !(nb <= 0x1p1020))) {
        bound = pending_max<G, PAIR>(s, rot, t, s0);
        const int eu = protect_update(bound, tt, xnb);
        if (eu < 0) {
          s.scale(eu);
          ex += eu;
          bound = scale2k(bound, eu);
          xnb = scale2k(xnb, eu);
        }
        nb = __dadd_rn(bound, __dmul_rn(tt, xnb));
      }
      bound = nb;
      // A fragments: lane (team, t) holds its column's coefficient for source row src0 + t;
      // the value of row 8 blk + r lives on lane r >> 1 of the team (register r & 1).
      double aS[3], aT[3];
#pragma unroll
      for (int kk = 0; kk < 3; ++kk) {
        double v;
        if (kk < 2) {
          // rows 8 blk + 4 kk + t
          const int r = g8 + 4 * kk + t;
          const double q0 = __shfl_sync(0xffffffffu, s.y[CUR][0], pbase + 2 * kk + (t >> 1));
          const double q1 = __shfl_sync(0xffffffffu, s.y[CUR][1], pbase + 2 * kk + (t >> 1));
          v = (t & 1) ? q1 : q0;
          if (!(r < e0)) v = 0.0;   // row 8 blk + 7 may belong to the block below; rows >= nt
        } else {
          // row 8 blk - 1 (top of a straddling 2x2 block) as source row src0 + 3
          v = __shfl_sync(0xffffffffu, s.y[PRV][1], pbase + 3);
          if (!(st && t == 3)) v = 0.0;
        }
        const double o = PAIR ? __shfl_xor_sync(0xffffffffu, v, 4) : 0.0;
        const double xr = PAIR ? (comp ? o : v) : v, xi = PAIR ? (comp ? v : o) : 0.0;
        aS[kk] = -(beta * v);
        aT[kk] = PAIR ? (comp ? (a * xi + b * xr) : (a * xr - b * xi)) : a * xr;
      }
      const double keep = s.y[PRV][1];   // solved straddling row: kept out of the update
#pragma unroll
      for (int q = 0; q < G - 1; ++q) {
        const int g = blk - (CUR - q);     // group at position q (pending iff g >= 0)
        if (g >= 0) {
#pragma unroll
          for (int kk = 0; kk < 3; ++kk) {
            if (kk == 2 && !st) continue;
            const int src0 = (kk < 2) ? g8 + 4 * kk : g8 - 4;
            const double2 v = sm.ST[poff3(min(src0 + t, nt - 1)) + 8 * g + team];
            dmma3(s.y[q][0], s.y[q][1], aS[kk], v.x);
            dmma3(s.y[q][0], s.y[q][1], aT[kk], v.y);
          }
        }
      }
      if (st && t == 3) s.y[PRV][1] = keep;
    }
    s.rotate();
    ++rot;
  }
  // ---- segment norms, exponent and the scaling decision of the next update (a5) ----
  double lm = 0.0, lh = 0.0;
#pragma unroll
  for (int q = 0; q < G; ++q) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double v = s.y[q][i];
      const double o = PAIR ? __shfl_xor_sync(0xffffffffu, v, 4) : 0.0;
      lm = fmax(lm, fabs(v));
      lh = fmax(lh, PAIR ? __dadd_rn(__dmul_rn(0.5, fabs(v)), __dmul_rn(0.5, fabs(o))) : __dmul_rn(0.5, fabs(v)));
    }
  }
  lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, 1));
  lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, 2));
  lh = fmax(lh, __shfl_xor_sync(0xffffffffu, lh, 1));
  lh = fmax(lh, __shfl_xor_sync(0xffffffffu, lh, 2));
  if (PAIR) lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, 4));
  const int ep = (valid && !tip) ? P.e_pend[c] : 0;
  const int es = ep + ex;
  int sx = 0;
  if (valid) {
    const long long so = (long long)p.I * p.n_sel + c;
    if (t == 0) {
      P.e_seg[so] = es;
      P.nrm_seg[so] = lm;
      P.nrmh_seg[so] = lh;
    }
    if (p.do_update && p.fused == 3) {
      // last step L of a step group (I, I-1, ..., L): one update of the rows above tile L
      // (region R, still at the exponent e_p it had before step I) with all the group's
      // tiles, K = [tile L | tile L+1 | ... | tile I].  The W of an earlier step X is at the
      // exponent e_X of its decision (e_grp), W_L at es; the band rows of tile L are at
      // ep = the last middle decision's exponent.  The decision bounds every term at once
      // (Alg. 3 with the sum of the panels' norms and the largest aligned segment norm, R5):
      //   2^(ef-e_p) y^_R + sum_X tau_X 2^(ef-e_X) x^_X <= 2^(ef-g)(y^ + (sum tau) max_X x^_X 2^(g-e_X)) <= Omega
      // A column not active at an earlier step has no term (and zero W) for it; a column
      // active only at L gets exactly the single-step decision.
      const bool act_first = p.n_prev > 0 && c0 >= p.prev_cs[0];
      const int e_p = act_first ? P.e_prev[c] : 0;            // written by the group's first step
      const unsigned long long* nyi = P.nY + (long long)p.nY_in * p.n_sel;
      double nyv = 0.0;
      if (c0 >= p.zero_pend_end) {                            // not a tip of the group
        nyv = __longlong_as_double((long long)nyi[c0]);
        if (PAIR) nyv = dmaxd(nyv, __longlong_as_double((long long)nyi[c0 + 1]));
      }
      const int g0 = min(ep, es);
      double xh = scale2k(lm, g0 - es);
      double tau = __dadd_rn(__dmul_rn(beta, P.cS[p.I]), __dmul_rn(ab, P.cT[p.I]));
      // earlier steps nearest first (tile L+1, ..., tile I): the order of the terms
#pragma unroll
      for (int k = kMaxGroup - 2; k >= 0; --k) {
        if (k < p.n_prev && c0 >= p.prev_cs[k]) {
          const long long sp = (long long)p.prev_I[k] * p.n_sel + c;
          xh = dmaxd(xh, scale2k(P.nrm_seg[sp], g0 - P.e_seg[sp]));
          tau = __dadd_rn(tau, __dadd_rn(__dmul_rn(beta, P.cS[p.prev_I[k]]), __dmul_rn(ab, P.cT[p.prev_I[k]])));
        }
      }
      const double yh = scale2k(nyv, g0 - e_p);
      const int ef = g0 + protect_update(yh, tau, xh);
      sx = ef - es;
      if (t == 0) {
        P.sY[c] = ef - e_p;
        P.e_pend[c] = ef;
        P.nY[(long long)(1 - p.nY_in) * p.n_sel + c] = 0ull;
        // lookahead: an upper bound of |pending| after this group's update, at exponent ef
        // (2^(ef-g) (y^ + tau x^), with a margin for the rounding of the sum and the update)
        if (p.record_bound)
          P.nYb[c] = scale2k(__dmul_rn(__dadd_rn(yh, __dmul_rn(tau, xh)), 1.0 + 0x1p-40), ef - g0);
      }
      // each earlier W of this column brought to ef (rare), or zero where the column was not
      // active at that step (stale entries)
#pragma unroll
      for (int k = 0; k < kMaxGroup - 1; ++k) {
        if (k < p.n_prev) {
          const bool act = c0 >= p.prev_cs[k];
          const int ek = act ? P.e_grp[(long long)k * p.n_sel + c] : 0;
          if (!act || ef != ek) {
            const long long tstr = (long long)(2 * p.prev_nks[k]) * (kBN * kBK);
            const long long hf = (long long)p.prev_nks[k] * (kBN * kBK);
            double* Wp = p.prev_W[k] + (long long)(c / kBN) * tstr + (c % kBN) * 4;
            for (int r = t; r < p.prev_nks[k] * kBK; r += 4) {
              const long long off = (long long)(r / kBK) * (kBN * kBK) + (long long)((r % kBK) >> 2) * (kBN * 4) + (r & 3);
              Wp[off] = act ? scale2k(Wp[off], ef - ek) : 0.0;
              Wp[off + hf] = act ? scale2k(Wp[off + hf], ef - ek) : 0.0;
            }
          }
        }
      }
    } else if (p.do_update) {
      // Alg. 3 with Alg. 2, reading R5; pending max of the column
      // (pairs: of both columns)
      // (fused == 2: a middle step of a group -- the decision covers the group's rows below
      // it only, whose maximum the previous thin update left in band buffer nY_in; the
      // exponent e_p of the rows above the group stays in e_prev for the last step)
      const unsigned long long* nyi = P.nY + (long long)p.nY_in * p.n_sel;
      double nyv = 0.0;
      if (!tip) {
        // (lookahead: the first step of a group takes the previous group's recorded bound)
        nyv = p.use_bound ? P.nYb[c0] : __longlong_as_double((long long)nyi[c0]);
        if (PAIR) nyv = dmaxd(nyv, p.use_bound ? P.nYb[c0 + 1] : __longlong_as_double((long long)nyi[c0 + 1]));
      }
      const int g0 = min(ep, es);
      const double yh = scale2k(nyv, g0 - ep), xh = scale2k(lm, g0 - es);
      const double tau = __dadd_rn(__dmul_rn(beta, P.cS[p.I]), __dmul_rn(ab, P.cT[p.I]));
      const int en = g0 + protect_update(yh, tau, xh);
      sx = en - es;
      if (t == 0) {
        // lookahead: a shift taken on the recorded bound rather than the measured maximum may
        // over-scale; flag it, and the call is recomputed without lookahead (zz_api.cu)
        if (p.use_bound && en < g0) atomicOr(&P.status[6], 1);
        P.sY[c] = en - ep;
        if (p.fused != 2) P.e_prev[c] = ep;   // the pending exponent before this step (read by a fused J/K)
        P.e_pend[c] = en;
        if (p.fused != 2) P.nY[(long long)(1 - p.nY_in) * p.n_sel + c] = 0ull;
        if (p.grp_slot >= 0) P.e_grp[(long long)p.grp_slot * p.n_sel + c] = en;   // exponent of this W
        for (int k = 0; k < p.n_band_reset; ++k) P.nY[(2LL + k) * p.n_sel + c] = 0ull;   // band maxima
      }
    }
  }
  // ---- store the segment and W = [-2^sx X D ; 2^sx X B] ----
  const double fx = (sx >= -1022) ? pow2k(sx) : 0.0;
  double* xo = p.X + (long long)(valid ? c : 0) * p.ldx + p.t0;
  const long long tstride = (long long)(2 * p.nks) * (kBN * kBK);
  const long long half = (long long)p.nks * (kBN * kBK);
  double* Wc = p.Wout + (long long)((valid ? c : 0) / kBN) * tstride + ((valid ? c : 0) % kBN) * 4;
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int g = (q - rot % G + G) % G;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = 8 * g + 2 * t + i;
      const double v = s.y[q][i];
      const double o = PAIR ? __shfl_xor_sync(0xffffffffu, v, 4) : 0.0;
      if (valid && r < nt) {
        xo[r] = v;
        if (p.do_update) {
          const double xs = (sx >= -1022) ? v * fx : scale2_slow3(v, sx);
          const double os = PAIR ? ((sx >= -1022) ? o * fx : scale2_slow3(o, sx)) : 0.0;
          const long long off = (long long)(r / kBK) * (kBN * kBK) + (long long)((r % kBK) >> 2) * (kBN * 4) + (r & 3);
          Wc[off] = -(beta * xs);
          Wc[off + half] = PAIR ? (comp ? (b * os + a * xs) : (a * xs - b * os)) : a * xs;
        }
      }
    }
  }
  // zero rows nt .. nks*BK-1 (the K padding of the last chunk)
  if (valid && p.do_update) {
    for (int r = nt + t; r < p.nks * kBK; r += 4) {
      const long long off = (long long)(r / kBK) * (kBN * kBK) + (long long)((r % kBK) >> 2) * (kBN * 4) + (r & 3);
      Wc[off] = 0.0;
      Wc[off + half] = 0.0;
    }
  }
  // W is read next by bulk copies (the async proxy): order the generic writes before them
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int G>
__global__ void __launch_bounds__(W3<G>::n * 32, 1) k_diag3(Diag2Params p) {
  constexpr int kW3 = W3<G>::n;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int nt = p.nt;
  Sm3 sm = carve3(smraw, nt);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // ---- stage the diagonal tile: (S_ij, T_ij) for i <= j, (S_{j+1,j}, 0) below ----
  const int plen = nt * (nt + 3) / 2;
  // asynchronous 8-byte global->shared copies (cp.async): every element of the tile is in
  // flight at once instead of one column per warp at a time (the staging was a third of the
  // kernel's time on latency-bound steps)
  for (int j = warp; j < nt; j += kW3) {
    const int len = min(j + 2, nt);
    const double* sc = p.S + (long long)(p.t0 + j) * p.lds + p.t0;
    const double* tc = p.T + (long long)(p.t0 + j) * p.ldt + p.t0;
    double2* col = sm.ST + poff3(j);
    for (int i = lane; i < len; i += 32) {
      const unsigned ds = (unsigned)__cvta_generic_to_shared(&col[i]);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(ds), "l"(sc + i) : "memory");
      if (i <= j)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(ds + 8u), "l"(tc + i) : "memory");
      else
        col[i].y = 0.0;
    }
  }
  for (int i = threadIdx.x; i < kPad3; i += blockDim.x) sm.ST[plen + i] = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < nt; i += blockDim.x) sm.fl[i] = p.P.row_flag[p.t0 + i];
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int nblk = (nt + 7) / 8;
  if (threadIdx.x <= nblk) {
    const int b = threadIdx.x;
    int v = 8 * b;
    if (v >= nt) v = nt;
    else if (b > 0 && sm.fl[v] == kRowBot2) v -= 1;
    sm.bs[b] = v;
  }
  // in-tile column bounds above each block (reading R6)
  for (int j = threadIdx.x; j < nt; j += blockDim.x) {
    const int top = (sm.fl[j] == kRowBot2) ? j - 1 : j;
    double ms = 0.0, mt = 0.0;
#pragma unroll 8
    for (int i = 0; i < top; ++i) {
      const double2 v = sm.ST[poff3(j) + i];
      ms = fmax(ms, fabs(v.x));
      mt = fmax(mt, fabs(v.y));
    }
    sm.cm[j] = make_double2(ms, mt);
  }
  __syncthreads();
  // a 2x2 block's bottom row carries the bound of both of its source columns (one row per
  // thread: blockDim >= kDiag2MaxNT >= nt)
  double2 cm2 = make_double2(0.0, 0.0);
  for (int j = threadIdx.x; j < nt; j += blockDim.x)
    if (sm.fl[j] == kRowBot2) cm2 = make_double2(sm.cm[j - 1].x + sm.cm[j].x, sm.cm[j - 1].y + sm.cm[j].y);
  __syncthreads();
  for (int j = threadIdx.x; j < nt; j += blockDim.x)
    if (sm.fl[j] == kRowBot2) sm.cm[j] = cm2;
  __syncthreads();
  // block panel norms: max over rows above the block of the row sums over its rows
  for (int b = warp; b < nblk; b += kW3) {
    const int s0 = sm.bs[b], e0 = sm.bs[b + 1];
    double ms = 0.0, mt = 0.0;
    for (int i = lane; i < s0; i += 32) {
      double rs = 0.0, rt = 0.0;
      for (int l = s0; l < e0; ++l) {
        const double2 v = sm.ST[poff3(l) + i];
        rs += fabs(v.x);
        rt += fabs(v.y);
      }
      ms = fmax(ms, rs);
      mt = fmax(mt, rt);
    }
    for (int o = 16; o; o >>= 1) {
      ms = fmax(ms, __shfl_xor_sync(0xffffffffu, ms, o));
      mt = fmax(mt, __shfl_xor_sync(0xffffffffu, mt, o));
    }
    if (lane == 0) sm.tau[b] = make_double2(ms, mt);
  }
  __syncthreads();
  // ---- tasks: 4 complex pairs or 8 real columns per warp ----
  const int npt = (p.n_pair + p.cpt / 2 - 1) / (p.cpt / 2), nrt = (p.n_real + p.cpt - 1) / p.cpt;
  // CTA-fastest assignment: with few tasks every SM gets one before any SM gets two
  // (measured: contiguous per-CTA task ranges were slower, pair tasks being heavier)
  for (int task = warp * gridDim.x + blockIdx.x; task < npt + nrt; task += gridDim.x * kW3) {
    if (task < npt) solve_task<G, true>(p, sm, nblk, task, lane, sm.slab + warp * 72, sm.pslab + warp * 576);
    else solve_task<G, false>(p, sm, nblk, task - npt, lane, sm.slab + warp * 72, sm.pslab + warp * 576);
  }
}

int g_sms3 = 0;

}  // namespace

size_t diag3_smem_bytes(int nt) { return smem3(nt); }

cudaError_t launch_diag3(const Diag2Params& pin, cudaStream_t st) {
  Diag2Params p = pin;
  if (!g_sms3) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms3, cudaDevAttrMultiProcessorCount, dev);
  }
  // 8 columns per task (measured: 4 or 2 columns per task on steps with few columns were
  // slower -- more tasks, more instruction-cache pressure, no shorter chain per task)
  p.cpt = 8;
  const int tasks = (p.n_pair + 3) / 4 + (p.n_real + 7) / 8;
  if (tasks == 0) return cudaSuccess;
  if (p.nt > kDiag2MaxNT) return cudaErrorInvalidValue;
  const size_t smem = smem3(p.nt);
  cudaError_t e;
  // pack: as few CTAs as the tasks need (one task per warp), leaving the other SMs to a
  // concurrent update (lookahead); otherwise one task per CTA first (lowest latency alone)
  if (p.nt <= 64) {
    constexpr int nw = W3<8>::n;
    const int grid = p.pack ? std::min(g_sms3, (tasks + nw - 1) / nw) : (tasks < g_sms3 ? tasks : g_sms3);
    e = cudaFuncSetAttribute(k_diag3<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_diag3<8><<<grid, nw * 32, smem, st>>>(p);
  } else {
    constexpr int nw = W3<16>::n;
    const int grid = p.pack ? std::min(g_sms3, (tasks + nw - 1) / nw) : (tasks < g_sms3 ? tasks : g_sms3);
    e = cudaFuncSetAttribute(k_diag3<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_diag3<16><<<grid, nw * 32, smem, st>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace zz
