// zz_complex.cu -- right eigenvectors of a COMPLEX pencil (S,T) in generalized complex Schur
// form (the ZTGEVC analogue; PAPER.md:333 names complex pencils as the next step, SURVEY.md
// s.8(f) NEXT-4).  Every diagonal block is 1x1, so the method is Algorithm 1
// with complex entries: a wavefront over tiles I = M-1 .. 0 of
//   (2) a robust diagonal-tile solve per active eigenvector (k_zdiag, two or four columns per warp,
//       the tile of S and T in shared memory, ProtectDivision / ProtectUpdate per row,
//       PAPER.md:175-200), which also takes the per-column scaling decision of Algorithm 3
//        and stages the scaled B operand [beta x ; -alpha x];
//   (3) the update of every pending row above the tile as ONE complex contraction
//       Y <- 2^sy Y + [S_panel | T_panel] [-sigma beta X_I ; sigma alpha X_I]   (K = 2 nb),
//       k_zupdate: Gauss's three-multiplication form (R23) as three DMMA.8x8x4 contractions
//       sharing one TMA-staged panel, with the scaling sigma_Y in its prologue;
//   (4) consistency and normalisation (max |Re|+|Im| = 1, ZTGEVC's convention).
// Readings R18-R21 of DESIGN.md; the pending-row maximum is carried as an upper bound
// (R21) instead of being measured, so the update needs no epilogue.
#include <cuda.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <utility>
#include <vector>

#include "../../include/zz.h"
#include "zz_internal.cuh"
#include "zz_pipe.cuh"

int ctx_acquire(cudaStream_t* st, int* mb, int* lookahead, zz_info_t** info);
int ctx_fusion();
int ctx_fusion_explicit();
void* ctx_zwork(size_t bytes);

namespace zz {
namespace {

constexpr int kZMaxNB = 64;        // rows per tile: two rows per lane
// k_zupdate tiling (below)
constexpr int kZBM = 64;        // complex rows per CTA tile
constexpr int kZBN = 32;        // columns per CTA tile
constexpr int kZBK = 16;        // complex panel columns per chunk (8 with 5 stages: 82 -> 78 ms at
                                // m = 10000, the barrier wait amortised over 96 instead of 48 DMMAs)
constexpr int kZKS = kZBK / 4;  // DMMA k-steps per chunk
constexpr int kZWPlane = kZBK * kZBN;   // doubles per plane of a W chunk
constexpr int kZStages = 3;
constexpr int kZABytes = 3 * kZBM * kZBK * 8;      // 24 KB: [8 row groups][3 planes][kZKS][32]
constexpr int kZBBytes = 3 * kZBK * kZBN * 8;      // 12 KB: [3][kZKS][32][4]
constexpr int kZUThreads = 5 * 32;
constexpr int kZUSmem = kZStages * (kZABytes + kZBBytes) + 2 * kZStages * 8;
constexpr int kZNGroup = 64;    // N tiles per group of the CTA order
constexpr int kZMaxG = 4;       // steps per step group (K segments of one update)

constexpr int kZWarps = 16;        // warps per CTA of k_zdiag (2 or 4 columns per warp)
constexpr int kZErrNonfinite = 0;  // status key = 2*row + kind
constexpr int kZErrCplxDiag = 1;

struct ZDiagParams {
  int I, r0, nt, cs, n_act, n_sel;
  const double2* S; long long lds;
  const double2* T; long long ldt;
  double2* X; long long ldx;
  const int* jcol;
  const double2* alpha;
  const double* beta;
  const double* cmS;
  const double* cmT;
  int* e_pend;
  double* nYb;
  int* e_seg;        // row I of the M x n_sel array
  double* nrmh_seg;  // row I
  double* W;         // update operand, k_zupdate's layout [n-tile][chunk][3 planes][2][32][4]
  int nkS;           // chunks of kZBK panel columns per part (S, then T)
  int* sy;           // per column: exponent shift of the pending rows (<= 0), this step's set
  int zero_begin;    // step groups: columns [zero_begin, cs) are not active at this step but
                     // are in the group's fused update -- their W and sy are written as zero
  int wact;          // warps of a CTA that solve (all kZWarps stage the tile)
};

__device__ __forceinline__ double zabsm(double2 z) { return fmax(fabs(z.x), fabs(z.y)); }
__device__ __forceinline__ double zabs1(double2 z) { return fabs(z.x) + fabs(z.y); }
__device__ __forceinline__ double2 zmul(double2 x, double2 y) {
  return make_double2(__dsub_rn(__dmul_rn(x.x, y.x), __dmul_rn(x.y, y.y)),
                      __dadd_rn(__dmul_rn(x.x, y.y), __dmul_rn(x.y, y.x)));
}
// y - s*u + t*v with fused multiply-adds
__device__ __forceinline__ double2 zaxpy2(double2 y, double2 s, double2 u, double2 t, double2 v) {
  double re = fma(-s.x, u.x, y.x);
  re = fma(s.y, u.y, re);
  re = fma(t.x, v.x, re);
  re = fma(-t.y, v.y, re);
  double im = fma(-s.x, u.y, y.y);
  im = fma(-s.y, u.x, im);
  im = fma(t.x, v.y, im);
  im = fma(t.y, v.x, im);
  return make_double2(re, im);
}
__device__ __forceinline__ double2 zldexp(double2 z, int k) { return make_double2(ldexp(z.x, k), ldexp(z.y, k)); }
// Smith's division (R20)
__device__ __forceinline__ double2 zdiv(double2 x, double2 y) {
  if (fabs(y.x) >= fabs(y.y)) {
    double r = y.y / y.x, den = y.x + y.y * r;
    return make_double2((x.x + x.y * r) / den, (x.y - x.x * r) / den);
  }
  double r = y.x / y.y, den = y.y + y.x * r;
  return make_double2((x.x * r + x.y) / den, (x.y * r - x.x) / den);
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// f(R-1), ..., f(0) with the index as a compile-time constant
template <class F, int... I>
__device__ __forceinline__ void zfor_rev(std::integer_sequence<int, I...>, F&& f) {
  (f(std::integral_constant<int, (int)sizeof...(I) - 1 - I>{}), ...);
}

// Per output column: normalised eigenvalue (R18) and zeroed state; per diagonal entry: the
// first invalid row (status key 2*row + kind, atomicMin).
__global__ void k_zprep(const double2* __restrict__ S, long long lds, const double2* __restrict__ T, long long ldt,
                        int m, const int* __restrict__ jcol, int n_sel, double2* alpha, double* beta, int* e_pend,
                        double* nYb, int* status) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < m) {
    double2 s = S[(long long)g * lds + g], t = T[(long long)g * ldt + g];
    if (!isfinite(s.x) || !isfinite(s.y) || !isfinite(t.x) || !isfinite(t.y)) atomicMin(status, 2 * g + kZErrNonfinite);
    else if (t.y != 0.0) atomicMin(status, 2 * g + kZErrCplxDiag);
  }
  if (g < n_sel) {
    const int j = jcol[g];
    double2 s = S[(long long)j * lds + j];
    double be = T[(long long)j * ldt + j].x;
    if (be < 0.0) { s.x = -s.x; s.y = -s.y; be = -be; }
    const double h = fmax(0.5 * be, 0.5 * fabs(s.x) + 0.5 * fabs(s.y));
    if (h == 0.0 || !isfinite(h)) {
      alpha[g] = make_double2(0.0, 0.0);
      beta[g] = 0.0;
    } else {
      int k;
      frexp(h, &k);
      alpha[g] = make_double2(ldexp(s.x, -(k + 1)), ldexp(s.y, -(k + 1)));
      beta[g] = ldexp(be, -(k + 1));
    }
    e_pend[g] = 0;
    nYb[g] = 0.0;
  }
}

// cmS[k] = max_{i<k} max(|Re S_ik|, |Im S_ik|), likewise cmT (R19): one warp per column.
__global__ void k_zcolmax(const double2* __restrict__ S, long long lds, const double2* __restrict__ T, long long ldt,
                          int m, double* cmS, double* cmT) {
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (k >= m) return;
  double ms = 0.0, mt = 0.0;
  const double2* s = S + (long long)k * lds;
  const double2* t = T + (long long)k * ldt;
  for (int i = lane; i < k; i += 32) {
    ms = fmax(ms, zabsm(s[i]));
    mt = fmax(mt, zabsm(t[i]));
  }
  ms = warp_max(ms);
  mt = warp_max(mt);
  if (lane == 0) { cmS[k] = ms; cmT[k] = mt; }
}

// Robust diagonal-tile solve + Algorithm 3's decision
// + the B operand of the update.  A warp solves C active columns: the
// L = 32 / C lanes of a column own the tile rows sub + L h (h < R = 64 / L).  The tile is
// walked bottom-up one row at a time for all C columns together, so the per-row instructions
// that are the same for every lane of a column (broadcasts, the update bound, Algorithm 2/3's
// tests, x D and x B) are issued once for C columns; the rows of a column are in registers
// with static indices (the row loop is unrolled over h, so row i = h L + s updates the
// register rows h' < h of every lane and row h of the lanes sub < s).  Every column sees
// exactly the operations of the one-column-per-warp form (bitwise the same results).
template <int C>
__global__ void __launch_bounds__(kZWarps * 32) k_zdiag(ZDiagParams p) {
  constexpr int L = 32 / C, R = kZMaxNB / L;
  extern __shared__ double2 sm[];
  double2* Ss = sm;                       // nt x nt, column-major
  double2* Ts = sm + p.nt * p.nt;
  double* cS = reinterpret_cast<double*>(Ts + p.nt * p.nt);
  double* cT = cS + kZMaxNB;
  const int nt = p.nt, r0 = p.r0;
  for (int idx = threadIdx.x; idx < nt * nt; idx += blockDim.x) {
    const int c = idx / nt, r = idx - c * nt;
    Ss[idx] = r <= c ? p.S[(long long)(r0 + c) * p.lds + r0 + r] : make_double2(0.0, 0.0);
    Ts[idx] = r <= c ? p.T[(long long)(r0 + c) * p.ldt + r0 + r] : make_double2(0.0, 0.0);
  }
  for (int r = threadIdx.x; r < nt; r += blockDim.x) { cS[r] = p.cmS[r0 + r]; cT[r] = p.cmT[r0 + r]; }
  if (p.zero_begin < p.cs) {
    const int per = 2 * kZBK * p.nkS;   // W rows (S part, then T part) of a column
    const long long nz = (long long)(p.cs - p.zero_begin) * per;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nz; q += (long long)gridDim.x * blockDim.x) {
      const int c = p.zero_begin + (int)(q / per), kk = (int)(q % per);
      double* o = p.W + (long long)(c / kZBN) * (2 * p.nkS) * (kZBBytes / 8) + (c % kZBN) * 4 +
                  (long long)(kk / kZBK) * (kZBBytes / 8) + ((kk % kZBK) >> 2) * (kZBN * 4) + (kk & 3);
      o[0] = 0.0;
      o[kZWPlane] = 0.0;
      o[2 * kZWPlane] = 0.0;
      if (kk == 0) p.sy[c] = 0;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int sub = lane % L, grp = lane / L;
  const unsigned gmask = (L == 32 ? 0xffffffffu : ((1u << L) - 1u)) << (grp * L);   // the column's lanes
  auto gmax = [&](double v) {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(gmask, v, o));
    return v;
  };
  auto gsum = [&](double v) {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o);
    return v;
  };
  const int ntask = (p.n_act + C - 1) / C;
  const int nw = gridDim.x * p.wact;
  if ((threadIdx.x >> 5) >= p.wact) {   // (no CTA-wide barrier follows)
    asm volatile("fence.proxy.async.global;" ::: "memory");   // its zeros of W above
    return;
  }
  for (int w = blockIdx.x * p.wact + (threadIdx.x >> 5); w < ntask; w += nw) {
    const bool cv = w * C + grp < p.n_act;       // this group has a column
    const int c = p.cs + (cv ? w * C + grp : 0);
    const int jl = p.jcol[c] - r0;               // >= nt: not a tip
    const bool tipc = jl < nt;
    const int top = cv ? (tipc ? jl : nt - 1) : -1;
    const double2 al = p.alpha[c];
    const double be = p.beta[c];
    const double aa = fabs(al.x) + fabs(al.y);
    double2* xc = p.X + (long long)c * p.ldx + r0;
    double2 y[R];
#pragma unroll
    for (int h = 0; h < R; ++h) {
      y[h] = make_double2(0.0, 0.0);
      if (!tipc && sub + L * h <= top) y[h] = xc[sub + L * h];
    }
    int e = (tipc || !cv) ? 0 : p.e_pend[c];
    // Off the dependent chain: the pivots of the lane's rows (R20) and their reciprocals
    // (Smith's formula for 1/d), the ProtectDivision thresholds, and the bound bw >= max |y|
    // over the pending in-tile rows (exact at the start).
    double2 inv[R];
    double td[R];
    double bw = 0.0;
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int r = sub + L * h;
      inv[h] = make_double2(0.0, 0.0);
      td[h] = 1.0;
      if (r <= top) {
        const double2 s = Ss[r * nt + r];
        const double t = Ts[r * nt + r].x;
        double2 d = make_double2(__dsub_rn(__dmul_rn(be, s.x), __dmul_rn(al.x, t)),
                                 __dsub_rn(__dmul_rn(be, s.y), __dmul_rn(al.y, t)));
        const double smin = fmax(kU * (be * zabs1(s) + aa * fabs(t)), kSmlnum);
        if (zabs1(d) < smin) d = make_double2(smin, 0.0);
        inv[h] = zdiv(make_double2(1.0, 0.0), d);
        td[h] = 0.5 * fmin(1.0, zabsm(d));
      }
      bw = fmax(bw, zabsm(y[h]));
    }
    bw = gmax(bw);
    const int itop = __reduce_max_sync(0xffffffffu, top);   // warp-uniform first row
    // the rows h L + s, s = L-1 .. 0, of register row h (h a compile-time constant, so that
    // every register row has a static index)
    auto rowblock = [&](auto hc) {
      constexpr int h = decltype(hc)::value;
      for (int s = min(L - 1, itop - h * L); s >= 0; --s) {
        const int i = h * L + s;
        const bool act = i <= top;
        const bool own = act && sub == s;
        // the tip's own row is 1 (R18); else ProtectDivision in the owner
        // lane, then x_i = y_i * (1/d_i)
        const bool tiprow = tipc && i == jl;
        int k = 0;
        if (own && !tiprow) k = protect_division(zabsm(y[h]), td[h]);
        k = __shfl_sync(0xffffffffu, k, s, L);
        if (k < 0) {
#pragma unroll
          for (int q = 0; q < R; ++q) y[q] = zldexp(y[q], k);
          bw = ldexp(bw, k);
          e += k;
        }
        if (own) y[h] = tiprow ? make_double2(1.0, 0.0) : zmul(y[h], inv[h]);
        double2 xi = make_double2(__shfl_sync(0xffffffffu, y[h].x, s, L), __shfl_sync(0xffffffffu, y[h].y, s, L));
        if (i == 0) break;   // h = 0, s = 0: the last row
        // ProtectUpdate of the in-tile rows above (R19 bound).  The bound bw
        // decides first; only when it cannot exclude a scaling is the exact maximum reduced,
        // so the decision is the one the exact maximum gives.
        const double tb = 2.0 * (be * cS[i] + aa * cT[i]);
        double ax = zabsm(xi);
        if (act && protect_update(bw, tb, ax) < 0) {
          double wm = 0.0;
#pragma unroll
          for (int q = 0; q < R; ++q)
            if (q < h || (q == h && sub < s)) wm = fmax(wm, zabsm(y[q]));
          wm = gmax(wm);
          const int k2 = protect_update(wm, tb, ax);
          if (k2 < 0) {
#pragma unroll
            for (int q = 0; q < R; ++q) y[q] = zldexp(y[q], k2);
            xi = zldexp(xi, k2);
            wm = ldexp(wm, k2);
            ax = zabsm(xi);
            e += k2;
          }
          bw = wm;
        }
        const double2 u = make_double2(be * xi.x, be * xi.y);   // x D
        const double2 v = zmul(al, xi);                          // x B
        // y_l <- y_l - S_li u + T_li v as 8 fused multiply-adds per row (the oracle rounds each
        // product: results agree to rounding, R22)
        if (act) {
#pragma unroll
          for (int q = 0; q < R; ++q) {
            if (q < h) y[q] = zaxpy2(y[q], Ss[i * nt + sub + L * q], u, Ts[i * nt + sub + L * q], v);
          }
          if (sub < s) y[h] = zaxpy2(y[h], Ss[i * nt + sub + L * h], u, Ts[i * nt + sub + L * h], v);
        }
        if (act) bw = bw + tb * ax;
      }
    };
    zfor_rev(std::make_integer_sequence<int, R>{}, rowblock);
    double nx = 0.0, hh = 0.0, sums = 0.0;
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int r = sub + L * h;
      if (r <= top) {
        xc[r] = y[h];
        nx = fmax(nx, zabsm(y[h]));
        hh = fmax(hh, 0.5 * fabs(y[h].x) + 0.5 * fabs(y[h].y));
        sums += be * cS[r] + aa * cT[r];
      }
    }
    nx = gmax(nx);
    hh = gmax(hh);
    sums = gsum(sums);
    if (cv && sub == 0) {
      p.e_seg[c] = e;
      p.nrmh_seg[c] = hh;
    }
    if (r0 == 0) continue;
    // Algorithm 3: one exponent for the pending rows after the update
    const int ep = (tipc || !cv) ? 0 : p.e_pend[c];
    const int g = min(ep, e);
    const double yh = ldexp((tipc || !cv) ? 0.0 : p.nYb[c], g - ep);
    const double xh = ldexp(nx, g - e);
    // R23 (k_zupdate): the partial sums of Im + Re accumulate from 2^sy (|Im Y| + |Re Y|) <=
    // 2 y^ and add up to sum_k (|Ar|+|Ai|)(|Wr|+|Wi|) <= 4 sums x^: ProtectUpdate(2 y^, 4 sums, x^)
    const double tau = 4.0 * sums;
    const int ed = protect_update(2.0 * yh, tau, xh);
    const int en = g + ed;
    const int sy = en - ep, sx = en - e;
    __syncwarp();
    if (cv && sub == 0) {
      p.e_pend[c] = en;
      // R21: the bound 2^ed (yh + tau xh), not a measurement; tau xh itself may exceed the
      // range when ed < 0, so that product is formed as protect_update does (scaled by 2^-1023)
      const double bnd = ed == 0 ? yh + tau * xh
                                 : ldexp(yh, ed) + ldexp(ldexp(tau, -512) * ldexp(xh, -511), ed + 1023);
      p.nYb[c] = bnd * (1.0 + 0x1p-40);
      p.sy[c] = sy;   // applied to the pending rows in k_zupdate's prologue
    }
    if (!cv) continue;
    // W(:, c) = [-sigma beta x ; sigma alpha x] in k_zupdate's stage layout, planes Re, Im and
    // Re + Im; rows past the tile (or past a tip) are zero
    double* Wt = p.W + (long long)(c / kZBN) * (2 * p.nkS) * (kZBBytes / 8) + (c % kZBN) * 4;
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int row = sub + L * h;
      if (row >= kZBK * p.nkS) continue;
      const bool z = row > top;
      const double2 xs = zldexp(y[h], sx);
      const double2 ws = z ? make_double2(0.0, 0.0) : make_double2(-(be * xs.x), -(be * xs.y));
      const double2 wt = z ? make_double2(0.0, 0.0) : zmul(al, xs);
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        const int kk = part ? kZBK * p.nkS + row : row;
        const double2 w = part ? wt : ws;
        double* o = Wt + (long long)(kk / kZBK) * (kZBBytes / 8) + ((kk % kZBK) >> 2) * (kZBN * 4) + (kk & 3);
        o[0] = w.x;
        o[kZWPlane] = w.y;
        o[2 * kZWPlane] = __dadd_rn(w.x, w.y);
      }
    }
  }
  // W is read next by bulk copies (the async proxy): order the generic writes before them
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------------------------------
// (3) The update of the pending rows as ONE complex contraction per step (PAPER.md:235's
// composition; reading R23): Y(rows, c) <- 2^sy[c] Y + [S_panel | T_panel] W(:, c) with
// W = [-sigma beta X_I ; sigma alpha X_I] (written by k_zdiag), by Gauss's three-multiplication
// form on the FP64 tensor instruction (DMMA.8x8x4):
//   T1 = Ar Wr,  T2 = Ai Wi,  T3 = (Ar + Ai)(Wr + Wi);   Re Y += T1 - T2,  Im Y += T3 - T1 - T2
// -- three real contractions sharing one staged panel and one staged W, each in three planes
// (Re, Im, Re + Im), 25 % fewer tensor instructions than the four-multiplication product.  The
// accumulators start from 2^sy Re Y, 0 and 2^sy (Im Y + Re Y), so the epilogue is
// Re = acc1 - acc2, Im = (acc3 - acc1) - acc2 (fixed order).  Bound (R23): every partial sum of
// acc3 is <= 2 y^ + sum_k (|Ar|+|Ai|)(|Wr|+|Wi|) <= 2 y^ + 4 sums x^ -- Algorithm 3's decision
// in k_zdiag is ProtectUpdate(2 y^, 4 sums, x^).
//
// k_zpack writes the panel of the step once in DMMA fragment order with its three planes
// ([64-row tile][chunk of 16 columns][8-row group][plane][k/4][lane]), so that a stage is one
// 24 KB bulk copy and every fragment load is one conflict-free 8-byte shared load (a TMA copy
// of the interleaved column-major panel gives 4-way conflicts on the 16-byte (Re, Im) loads).
// Pipeline as the real update (zz_update.cu): CTA tile 64 complex rows x 32 columns (aligned
// 64-row tiles from row 0; rows outside [row_lo, rows) are computed but not stored), four DMMA
// warps (32 rows x 16 columns each) and one producer warp, per stage 16 panel columns (24 KB)
// and the matching 12 KB of W, a 3-stage mbarrier ring.  The contraction is computed transposed (Y^T += W^T A^T): a
// lane's accumulators are two consecutive complex rows of one column (32-byte loads/stores).
// ------------------------------------------------------------------------------------
struct ZUpdParams {
  int rows, row_lo;   // complex rows [row_lo, rows) are updated
  int nkc;            // chunks of kZBK panel columns (S part, then T part)
  int c_begin, n_sel; // active columns
  int ntile0;         // first 32-column tile (c_begin / 32)
  int mtile0;         // first 64-row tile (row_lo / 64)
  double2* X; long long ldx;
  // K segments (a step group, PAPER.md:235's composition over several tiles): segment e has
  // its packed panel at A + e a_stride, its W at W + e w_stride and its sy at sy + e sy_stride,
  // each nkc chunks.  Y <- 2^(sum_e sy_e) Y + sum_e 2^(sum_{e' < e} sy_e') A_e W_e: the
  // contribution of tile L + e is scaled by the decisions of the later steps L + e - 1 .. L.
  const double* A;    // packed panel (k_zpack), segment 0
  const double* W;    // [n-tile][nkc][3][kZBK/4][32][4], segment 0
  const int* sy;
  int nseg;
  long long a_stride, w_stride;
  int sy_stride;
};

// panel of step I in fragment order: block (mt, kc) = 64 rows x 8 columns x 3 planes, element
// (row 8 g + cq, column 4 ks + rq, plane p) at ((g * 3 + p) * 2 + ks) * 32 + 4 cq + rq; columns
// kc < nkS from S, then T; columns past the tile (ragged last tile) and rows >= r0 are zero
__global__ void __launch_bounds__(256) k_zpack(const double2* __restrict__ S, long long lds,
                                               const double2* __restrict__ T, long long ldt, int r0, int nt, int nkS,
                                               double* __restrict__ A) {
  __shared__ double2 tile[kZBK][kZBM + 1];
  const int mt = blockIdx.x, kc = blockIdx.y;
  const bool isT = kc >= nkS;
  const double2* P = isT ? T : S;
  const long long ld = isT ? ldt : lds;
  const int k0 = (isT ? kc - nkS : kc) * kZBK;
  for (int idx = threadIdx.x; idx < kZBK * kZBM; idx += blockDim.x) {
    const int k = idx / kZBM, r = idx % kZBM;
    const int row = mt * kZBM + r;
    tile[k][r] = (row < r0 && k0 + k < nt) ? P[(long long)(r0 + k0 + k) * ld + row] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  double* out = A + ((long long)mt * gridDim.y + kc) * (kZABytes / 8);
  for (int o = threadIdx.x; o < kZABytes / 8; o += blockDim.x) {
    const int ln = o & 31, ks = (o >> 5) % kZKS, pl = ((o >> 5) / kZKS) % 3, g = (o >> 5) / (3 * kZKS);
    const double2 v = tile[ks * 4 + (ln & 3)][g * 8 + (ln >> 2)];
    out[o] = pl == 0 ? v.x : (pl == 1 ? v.y : __dadd_rn(v.x, v.y));
  }
  // read next by bulk copies (the async proxy)
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__global__ void __launch_bounds__(kZUThreads, 2) k_zupdate(ZUpdParams p, int n_mtiles, int n_ntiles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  double* sA = reinterpret_cast<double*>(smem);
  double* sB = reinterpret_cast<double*>(smem + kZStages * kZABytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kZStages * (kZABytes + kZBBytes));
  uint64_t* empty = full + kZStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkc = p.nkc;              // chunks per segment
  const int nkt = p.nseg * nkc;       // chunks in all
  int mt, nt;
  {
    const int tile = blockIdx.x, per = n_mtiles * kZNGroup;
    const int g = tile / per, loc = tile - g * per;
    const int gs = min(kZNGroup, n_ntiles - g * kZNGroup);
    mt = p.mtile0 + loc / gs;
    nt = g * kZNGroup + loc % gs;
  }
  const int m0 = mt * kZBM;                       // first complex row of the tile
  const int ntile = p.ntile0 + nt;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kZStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 4) {
    if (lane == 0) {
      const uint64_t pol_w = l2_policy(true);
      const double* wt = p.W + (long long)ntile * nkc * (kZBBytes / 8);
      const double* at = p.A + (long long)mt * nkc * (kZABytes / 8);
      int e = 0, lc = 0;
      for (int kc = 0; kc < nkt; ++kc) {
        const int s = kc % kZStages;
        if (kc >= kZStages) mbar_wait(&empty[s], ((kc / kZStages) - 1) & 1);
        mbar_expect_tx(&full[s], kZABytes + kZBBytes);
        bulk_load_h(sA + s * (kZABytes / 8), at + e * p.a_stride + (long long)lc * (kZABytes / 8), kZABytes, &full[s],
                    pol_w);
        bulk_load_h(sB + s * (kZBBytes / 8), wt + e * p.w_stride + (long long)lc * (kZBBytes / 8), kZBBytes, &full[s],
                    pol_w);
        if (++lc == nkc) { lc = 0; ++e; }
      }
    }
    return;
  }
  const int wm = warp >> 1, wn = warp & 1;
  const int rq = lane & 3, cq = lane >> 2;
  const uint64_t pol_c = l2_policy(false);
  // Per column: the exponent shift of the old Y (the sum of the group's decisions, applied in
  // the prologue) and of each segment's W (the later steps' decisions: exact powers of two,
  // applied to the staged fragments only in the rare case that a decision scaled).  (Holding
  // the old Y in registers for an epilogue add needs 200 registers: 1 CTA per SM, 1.6x slower.)
  double acc1[2][4][2], acc2[2][4][2], acc3[2][4][2];
  unsigned segscale = 0;   // warp-uniform: segments whose W some column of the warp rescales
#pragma unroll
  for (int ni = 0; ni < 2; ++ni) {
    const int c = ntile * kZBN + wn * 16 + ni * 8 + cq;
    const bool cv = c >= p.c_begin && c < p.n_sel;
    int sy = 0;
#pragma unroll
    for (int e = 0; e < kZMaxG; ++e) {
      if (e < p.nseg) {
        if (e > 0 && sy != 0) segscale |= 1u << e;
        int v = 0;
        ld1p_i(v, p.sy + (long long)e * p.sy_stride + (cv ? c : 0), cv);
        sy += v;
      }
    }
    const double* xc = reinterpret_cast<const double*>(p.X + (long long)(cv ? c : 0) * p.ldx);
    double v[4][4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int i0 = m0 + wm * 32 + mi * 8 + 2 * rq;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[mi][q] = 0.0;
      ld2h(v[mi][0], v[mi][1], xc + 2 * i0, cv && i0 < p.rows && i0 >= p.row_lo, pol_c);
      ld2h(v[mi][2], v[mi][3], xc + 2 * i0 + 2, cv && i0 + 1 < p.rows && i0 + 1 >= p.row_lo, pol_c);
    }
    if (sy != 0) {   // rare: a scaling decision of Algorithm 3 (exact powers of two)
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int q = 0; q < 4; ++q) v[mi][q] = ldexp(v[mi][q], sy);
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        acc1[ni][mi][h] = v[mi][2 * h];
        acc2[ni][mi][h] = 0.0;
        acc3[ni][mi][h] = __dadd_rn(v[mi][2 * h + 1], v[mi][2 * h]);
      }
    }
  }
  segscale = __reduce_or_sync(0xffffffffu, segscale);
  int e = 0, lc = 0;
  for (int kc = 0; kc < nkt; ++kc) {
    const int s = kc % kZStages;
    mbar_wait(&full[s], (kc / kZStages) & 1);
    // release the previous stage only now (see k_update_t)
    if (lane == 0 && kc >= 1 && kc - 1 + kZStages < nkt) mbar_arrive(&empty[(kc - 1) % kZStages]);
    const double* a = sA + s * (kZABytes / 8);
    const double* b = sB + s * (kZBBytes / 8);
    // one k-step of 4 panel columns: W and panel fragments, 24 DMMAs (SCALE: the rare case of
    // a later step in the group having scaled a column, its W fragments rescaled by 2^sc)
#define ZZ_ZCHUNK_KS(SCALE)                                                          \
  _Pragma("unroll") for (int ks = 0; ks < kZBK / 4; ++ks) {                          \
    double wr[2], wi[2], ws[2], fr[4], fi[4], fs[4];                                 \
    _Pragma("unroll") for (int ni = 0; ni < 2; ++ni) {                               \
      const int o = (ks * kZBN + wn * 16 + ni * 8 + cq) * 4 + rq;                    \
      wr[ni] = b[o];                                                                 \
      wi[ni] = b[kZWPlane + o];                                                      \
      ws[ni] = b[2 * kZWPlane + o];                                                  \
      if (SCALE) {                                                                   \
        wr[ni] = ldexp(wr[ni], sc[ni]);                                              \
        wi[ni] = ldexp(wi[ni], sc[ni]);                                              \
        ws[ni] = ldexp(ws[ni], sc[ni]);                                              \
      }                                                                              \
    }                                                                                \
    _Pragma("unroll") for (int mi = 0; mi < 4; ++mi) {                               \
      const int g = wm * 4 + mi;                                                     \
      fr[mi] = a[((g * 3 + 0) * kZKS + ks) * 32 + lane];                                \
      fi[mi] = a[((g * 3 + 1) * kZKS + ks) * 32 + lane];                                \
      fs[mi] = a[((g * 3 + 2) * kZKS + ks) * 32 + lane];                                \
    }                                                                                \
    _Pragma("unroll") for (int ni = 0; ni < 2; ++ni)                                 \
      _Pragma("unroll") for (int mi = 0; mi < 4; ++mi) {                             \
        dmma(acc1[ni][mi][0], acc1[ni][mi][1], wr[ni], fr[mi]);                      \
        dmma(acc2[ni][mi][0], acc2[ni][mi][1], wi[ni], fi[mi]);                      \
        dmma(acc3[ni][mi][0], acc3[ni][mi][1], ws[ni], fs[mi]);                      \
      }                                                                              \
  }
    if (!((segscale >> e) & 1)) {
      const int sc[2] = {0, 0};
      ZZ_ZCHUNK_KS(false)
    } else {   // rare: the prefix sum of the earlier segments' sy, reloaded
      int sc[2] = {0, 0};
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) {
        const int c = ntile * kZBN + wn * 16 + ni * 8 + cq;
        if (c >= p.c_begin && c < p.n_sel)
          for (int q = 0; q < e; ++q) sc[ni] += p.sy[(long long)q * p.sy_stride + c];
      }
      ZZ_ZCHUNK_KS(true)
    }
#undef ZZ_ZCHUNK_KS
    __syncwarp();
    if (++lc == nkc) { lc = 0; ++e; }
  }
#pragma unroll
  for (int ni = 0; ni < 2; ++ni) {
    const int c = ntile * kZBN + wn * 16 + ni * 8 + cq;
    const bool cv = c >= p.c_begin && c < p.n_sel;
    double* xc = reinterpret_cast<double*>(p.X + (long long)(cv ? c : 0) * p.ldx);
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int i0 = m0 + wm * 32 + mi * 8 + 2 * rq;
      double o[2][2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        o[h][0] = __dsub_rn(acc1[ni][mi][h], acc2[ni][mi][h]);
        o[h][1] = __dsub_rn(__dsub_rn(acc3[ni][mi][h], acc1[ni][mi][h]), acc2[ni][mi][h]);
      }
      st2h(xc + 2 * i0, o[0][0], o[0][1], cv && i0 < p.rows && i0 >= p.row_lo, pol_c);
      st2h(xc + 2 * i0 + 2, o[1][0], o[1][1], cv && i0 + 1 < p.rows && i0 + 1 >= p.row_lo, pol_c);
    }
  }
}

// (4) consistency and normalisation: e_c = min_I e_seg[I][c]; X <- ldexp(X, e_c - e_seg) / xmax
// with xmax = max (|Re|+|Im|) formed as 2 max(|Re|/2 + |Im|/2) (ZTGEVC's normalisation).
__global__ void __launch_bounds__(256) k_znorm(double2* X, long long ldx, int nb, int n_sel, const int* __restrict__ jcol,
                                              const int* __restrict__ e_seg, const double* __restrict__ nrmh_seg,
                                              int* col_scale_exp) {
  const int c = blockIdx.x;
  const int j = jcol[c];
  const int Jt = j / nb;
  __shared__ int s_e;
  __shared__ double s_rec;
  if (threadIdx.x == 0) {
    int ec = 0;
    for (int I = 0; I <= Jt; ++I) ec = min(ec, e_seg[(long long)I * n_sel + c]);
    double h = 0.0;
    for (int I = 0; I <= Jt; ++I) {
      const long long q = (long long)I * n_sel + c;
      h = fmax(h, ldexp(nrmh_seg[q], ec - e_seg[q]));
    }
    s_e = ec;
    s_rec = h > 0.0 ? 0.5 / h : 1.0;
    if (col_scale_exp) col_scale_exp[c] = ec;
  }
  __syncthreads();
  const int ec = s_e;
  const double rec = s_rec;
  double2* x = X + (long long)c * ldx;
  for (int i = threadIdx.x; i <= j; i += blockDim.x) {
    const int k = ec - e_seg[(long long)(i / nb) * n_sel + c];
    const double2 v = zldexp(x[i], k);
    x[i] = make_double2(v.x * rec, v.y * rec);
  }
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace
}  // namespace zz

using namespace zz;

#define ZCK(x)                                                              \
  do {                                                                      \
    cudaError_t _e = (x);                                                   \
    if (_e != cudaSuccess) return _e == cudaErrorMemoryAllocation ? ZZ_ERR_NOMEM : ZZ_ERR_CUDA; \
  } while (0)

extern "C" int zz_ztgevc(int m, const double* S_, int lds, const double* T_, int ldt, const int* select,
                         double* X_, int ldx, int* col_scale_exp) {
  if (m < 0) return -1;
  if (m > 0 && !S_) return -2;
  if (lds < std::max(1, m)) return -3;
  if (m > 0 && !T_) return -4;
  if (ldt < std::max(1, m)) return -5;
  if (m > 0 && !X_) return -7;
  if (ldx < std::max(1, m)) return -8;
  // COMPLEX*16 is read and written as 16-byte (re, im) pairs: the bases must be 16-byte
  // aligned (a misaligned access would be a sticky fault of the CUDA context)
  auto misaligned = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) != 0; };
  if (m > 0 && misaligned(S_)) return -2;
  if (m > 0 && misaligned(T_)) return -4;
  if (m > 0 && misaligned(X_)) return -7;
  cudaStream_t st;
  int mb_ctx, la_mode;
  zz_info_t* info;
  int r = ctx_acquire(&st, &mb_ctx, &la_mode, &info);
  if (r) return r;
  memset(info, 0, sizeof(*info));
  info->m = m;
  if (m == 0) return 0;
  const int nb = (mb_ctx >= 16 && mb_ctx <= kZMaxNB) ? mb_ctx : kZMaxNB;
  const int M = (m + nb - 1) / nb;
  std::vector<int> jcol;
  jcol.reserve(m);
  for (int j = 0; j < m; ++j)
    if (!select || select[j]) jcol.push_back(j);
  const int n = (int)jcol.size();
  info->n_sel = n;
  info->mb = nb;
  info->n_tiles = M;
  const double2* S = reinterpret_cast<const double2*>(S_);
  const double2* T = reinterpret_cast<const double2*>(T_);
  double2* X = reinterpret_cast<double2*>(X_);
  if (n == 0) return 0;
  // Step groups (zz_set_fusion, at most kZMaxG steps): the steps of a group I, I-1, ..., L run
  // their diagonal solves, each followed by a thin update of the group's remaining band (the
  // rows of tiles L .. X-1) with W_X, and then ONE update of all rows above tile L with
  // K = [tile L | ... | tile I] (k_zupdate segments).  The decisions use the pending bound
  // (R21), not a measured maximum, so they are the same as step by step; the contribution of
  // tile X is scaled by the later steps' decisions inside the contraction.  Every tile uses
  // nkS_max chunks (a ragged last tile is zero-padded), so the segments are uniform.
  // Default group length by the number of steps (measured, profiles/r02ak_zab.txt: m = 2000 is
  // fastest ungrouped, 4000 in pairs, 6000 in triples, 10000 in groups of 3-4: short wavefronts
  // are bound by the chain, which the group's band updates lengthen); zz_set_fusion overrides.
  const int G = ctx_fusion_explicit() ? std::max(1, std::min(kZMaxG, ctx_fusion()))
                                      : std::max(1, std::min(kZMaxG, (M + 16) / 32));
  // workspace (stream-ordered)
  const int nkS_max = (nb + kZBK - 1) / kZBK;
  const int n_nt = (n + kZBN - 1) / kZBN;
  const int NS = 2 * G;   // W / sy / panel sets: two groups (lookahead) of G slots
  const size_t wsz = (size_t)n_nt * 2 * nkS_max * (kZBBytes / 8);   // doubles per W set
  const size_t apk = (size_t)((m + kZBM - 1) / kZBM) * 2 * nkS_max * (kZABytes / 8);   // packed panel
  size_t off[13], tot = 0;
  const size_t sz[13] = {sizeof(int) * n, sizeof(double2) * n, sizeof(double) * n, sizeof(int) * n, sizeof(double) * n,
                         sizeof(int) * (size_t)M * n, sizeof(double) * (size_t)M * n, sizeof(double) * m,
                         sizeof(double) * m, sizeof(double) * NS * wsz, sizeof(int) * 4, sizeof(int) * NS * (size_t)n,
                         sizeof(double) * NS * apk};
  for (int i = 0; i < 13; ++i) { off[i] = tot; tot += align256(sz[i]); }
  // kept by the context between calls (a stream-ordered allocation returned its memory to the
  // driver at every call's final synchronisation: sporadic calls 10-15 ms longer at m = 10000)
  char* base = static_cast<char*>(ctx_zwork(tot));
  if (!base) return ZZ_ERR_NOMEM;
  int* d_jcol = reinterpret_cast<int*>(base + off[0]);
  double2* d_alpha = reinterpret_cast<double2*>(base + off[1]);
  double* d_beta = reinterpret_cast<double*>(base + off[2]);
  int* d_epend = reinterpret_cast<int*>(base + off[3]);
  double* d_nYb = reinterpret_cast<double*>(base + off[4]);
  int* d_eseg = reinterpret_cast<int*>(base + off[5]);
  double* d_nrmh = reinterpret_cast<double*>(base + off[6]);
  double* d_cmS = reinterpret_cast<double*>(base + off[7]);
  double* d_cmT = reinterpret_cast<double*>(base + off[8]);
  double* d_W = reinterpret_cast<double*>(base + off[9]);
  int* d_status = reinterpret_cast<int*>(base + off[10]);
  int* d_sy = reinterpret_cast<int*>(base + off[11]);
  double* d_A = reinterpret_cast<double*>(base + off[12]);
  int launches = 0;
  ZCK(cudaMemcpyAsync(d_jcol, jcol.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
  const int big = 0x7fffffff;
  ZCK(cudaMemcpyAsync(d_status, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  ZCK(cudaMemset2DAsync(X, sizeof(double2) * (size_t)ldx, 0, sizeof(double2) * (size_t)m, n, st));
  k_zprep<<<(std::max(m, n) + 255) / 256, 256, 0, st>>>(S, lds, T, ldt, m, d_jcol, n, d_alpha, d_beta, d_epend, d_nYb,
                                                       d_status);
  k_zcolmax<<<(m + 7) / 8, 256, 0, st>>>(S, lds, T, ldt, m, d_cmS, d_cmT);
  launches += 2;
  ZCK(cudaGetLastError());
  int hstatus = big;
  ZCK(cudaMemcpyAsync(&hstatus, d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
  ZCK(cudaStreamSynchronize(st));
  if (hstatus != big) return (hstatus & 1) == kZErrCplxDiag ? ZZ_ERR_CPLXDIAG : ZZ_ERR_NONFINITE;
  const size_t smem = sizeof(double2) * 2 * nb * nb + sizeof(double) * 2 * kZMaxNB;
  ZCK(cudaFuncSetAttribute(k_zdiag<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ZCK(cudaFuncSetAttribute(k_zdiag<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ZCK(cudaFuncSetAttribute(k_zupdate, cudaFuncAttributeMaxDynamicSharedMemorySize, kZUSmem));
  ZCK(cudaFuncSetAttribute(k_zupdate, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int nsm = 148;
  {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  // first active column of each step (columns with jcol >= r0); the active set only grows as
  // I decreases, so the empty steps are the top ones
  std::vector<int> csI(M);
  {
    int cs = n;
    for (int I = M - 1; I >= 0; --I) {
      while (cs > 0 && jcol[cs - 1] >= I * nb) --cs;
      csI[I] = cs;
    }
  }
  int Itop = M - 1;
  while (Itop >= 0 && csI[Itop] == n) --Itop;
  // Lookahead (DESIGN.md s.6 "Complex pencils"): the chain of a step group -- its solves, band
  // updates and the part of the previous group's update that covers its band -- runs on a
  // high-priority stream; the rest of the previous group's update (the rows above the band)
  // runs on the caller's stream beside it.  The decisions use the pending bound (R21), so the
  // chain needs nothing from the rest; W, sy and the packed panels alternate between two sets
  // of G slots by group, and the chain waits for the rest of the group before last (whose
  // rows its own band part updates next) before it writes the set that rest reads.
  const bool la = la_mode != 0 && Itop >= 1;   // zz_set_lookahead(0) turns it off
  cudaStream_t hp = nullptr;
  cudaEvent_t ev_dec = nullptr, ev_rest = nullptr;
  struct Guard {
    cudaStream_t& h; cudaEvent_t& a; cudaEvent_t& b; cudaStream_t st;
    ~Guard() {
      // on every exit (errors included) the work queued on the high-priority stream has
      // finished before the call returns (the context's workspace is reused by the next call)
      if (h) { cudaStreamSynchronize(h); cudaStreamDestroy(h); }
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
    }
  } guard{hp, ev_dec, ev_rest, st};
  if (la) {
    int lo, hi;
    ZCK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    ZCK(cudaStreamCreateWithPriority(&hp, cudaStreamNonBlocking, hi));
    ZCK(cudaEventCreateWithFlags(&ev_dec, cudaEventDisableTiming));
    ZCK(cudaEventCreateWithFlags(&ev_rest, cudaEventDisableTiming));
  }
  cudaStream_t cs_ = la ? hp : st;   // the chain's stream
  auto diag = [&](int I, int slot, int zero_begin) -> cudaError_t {
    const int r0 = I * nb, nt = std::min(nb, m - r0), cs = csI[I], n_act = n - cs;
    ZDiagParams p;
    p.I = I; p.r0 = r0; p.nt = nt; p.cs = cs; p.n_act = n_act; p.n_sel = n;
    p.S = S; p.lds = lds; p.T = T; p.ldt = ldt; p.X = X; p.ldx = ldx;
    p.jcol = d_jcol; p.alpha = d_alpha; p.beta = d_beta; p.cmS = d_cmS; p.cmT = d_cmT;
    p.e_pend = d_epend; p.nYb = d_nYb;
    p.e_seg = d_eseg + (size_t)I * n;
    p.nrmh_seg = d_nrmh + (size_t)I * n;
    p.W = d_W + (size_t)slot * wsz;
    p.nkS = nkS_max;
    p.sy = d_sy + (size_t)slot * n;
    p.zero_begin = std::min(zero_begin, cs);
    const int zb = (cs - p.zero_begin + kZWarps - 1) / kZWarps;
    // Two columns per warp while one pass of one CTA per SM covers the step, four beyond
    // (measured, profiles/r02am_zdiag_ab.txt: m = 2000 2.91 -> 2.43 ms with two, 2.75 with four;
    // m = 10000 77.0 -> 74.3 with two, 72.3 with four; bitwise the one-column kernel's results)
    const int cpw = n_act > nsm * kZWarps * 2 ? 4 : 2;
    const int ntask = (n_act + cpw - 1) / cpw;   // warp tasks
    // all warps of a CTA solve: the tasks are packed 16 to a CTA, so the other SMs stay with the
    // previous group's update (spreading them over the SMs first, fewer solving warps per CTA,
    // was slower from m = 2000: 2.45 -> 2.6 ms, 7.4 -> 8.0 ms at 4000; profiles/r02ap_zspread.txt)
    p.wact = kZWarps;
    const int grid = std::max(1, std::min(std::max((ntask + p.wact - 1) / p.wact, zb), nsm));   // one 132 KB CTA per SM
    if (cpw == 4) k_zdiag<4><<<grid, kZWarps * 32, smem, cs_>>>(p);
    else k_zdiag<2><<<grid, kZWarps * 32, smem, cs_>>>(p);
    ++launches;
    return cudaGetLastError();
  };
  // the panel of step I in fragment order (rows 0 .. r0 - 1), into panel slot `slot`
  auto pack = [&](int I, int slot) -> cudaError_t {
    const int r0 = I * nb, nt = std::min(nb, m - r0);
    k_zpack<<<dim3((r0 + kZBM - 1) / kZBM, 2 * nkS_max), 256, 0, cs_>>>(S, lds, T, ldt, r0, nt, nkS_max,
                                                                       d_A + (size_t)slot * apk);
    ++launches;
    return cudaGetLastError();
  };
  // Y(row0:row1, cs:n) <- 2^sy Y + sum_e [S_panel | T_panel]_e W_e for the nseg slots from
  // `slot` (tiles L, L+1, ...; cs = the first column active at tile L)
  auto update = [&](int L, int slot, int nseg, int row0, int row1, cudaStream_t us) -> cudaError_t {
    const int cs = csI[L];
    ZUpdParams up;
    up.row_lo = row0;
    up.rows = row1;
    up.nkc = 2 * nkS_max;
    up.c_begin = cs;
    up.n_sel = n;
    up.ntile0 = cs / kZBN;
    up.mtile0 = row0 / kZBM;
    up.X = X;
    up.ldx = ldx;
    up.A = d_A + (size_t)slot * apk;
    up.W = d_W + (size_t)slot * wsz;
    up.sy = d_sy + (size_t)slot * n;
    up.nseg = nseg;
    up.a_stride = (long long)apk;
    up.w_stride = (long long)wsz;
    up.sy_stride = n;
    const int n_mt = (row1 - 1) / kZBM - up.mtile0 + 1, n_ntl = n_nt - up.ntile0;
    if (row1 <= row0 || n_ntl <= 0) return cudaSuccess;
    // one tile per CTA: CTAs retire after each tile, so the high-priority diagonal solve of the
    // lookahead finds free SMs (measured: a persistent grid of 2 CTAs per SM was slower with it)
    k_zupdate<<<n_mt * n_ntl, kZUThreads, kZUSmem, us>>>(up, n_mt, n_ntl);
    ++launches;
    info->update_launches++;
    return cudaGetLastError();
  };
  // groups are fixed by the tile index counted from M-1 (not by the selection), so a column's
  // arithmetic does not depend on which other columns are computed; the last step of a group
  // needs rows above it (index >= 1)
  auto group_len = [&](int I) {
    int len = G - (M - 1 - I) % G;
    while (len > 1 && I - (len - 1) < 1) --len;
    return len;
  };
  if (la) {   // fork the chain's stream from the caller's
    ZCK(cudaEventRecord(ev_dec, st));
    ZCK(cudaStreamWaitEvent(hp, ev_dec, 0));
  }
  int gpar = 0;
  bool rest_pending = false;   // the previous group's rest update runs on st (lookahead)
  for (int I = Itop; I >= 0;) {
    if (I == 0) {               // the top rows: solve only
      ZCK(diag(0, gpar * G, csI[0]));
      break;
    }
    const int len = group_len(I), L = I - len + 1, sb = gpar * G;
    for (int X = I; X >= L; --X) {
      ZCK(diag(X, sb + (X - L), csI[L]));
      ZCK(pack(X, sb + (X - L)));
      if (X > L) ZCK(update(X, sb + (X - L), 1, L * nb, X * nb, cs_));   // the group's band
    }
    if (len >= 2) info->fused_pairs++;
    // the update of all rows above tile L with the group's len segments
    int rb = 0;                 // lookahead: rows [rb, L nb) are the next group's band
    if (la && L - 1 >= 1) rb = (L - group_len(L - 1)) * nb;
    if (la && rest_pending) ZCK(cudaStreamWaitEvent(hp, ev_rest, 0));
    if (la && rb > 0) {
      ZCK(update(L, sb, len, rb, L * nb, hp));
      ZCK(cudaEventRecord(ev_dec, hp));
      ZCK(cudaStreamWaitEvent(st, ev_dec, 0));
      ZCK(update(L, sb, len, 0, rb, st));
      ZCK(cudaEventRecord(ev_rest, st));
      rest_pending = true;
    } else {
      ZCK(update(L, sb, len, 0, L * nb, cs_));
      rest_pending = false;
    }
    gpar ^= la ? 1 : 0;
    I = L - 1;
  }
  if (la) {   // join the chain back into the caller's stream
    ZCK(cudaEventRecord(ev_dec, hp));
    ZCK(cudaStreamWaitEvent(st, ev_dec, 0));
  }
  k_znorm<<<n, 256, 0, st>>>(X, ldx, nb, n, d_jcol, d_eseg, d_nrmh, col_scale_exp);
  ++launches;
  ZCK(cudaGetLastError());
  info->total_launches = launches;
  ZCK(cudaStreamSynchronize(st));
  return 0;
}
