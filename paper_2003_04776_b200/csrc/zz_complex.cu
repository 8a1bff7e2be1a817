// zz_complex.cu -- right eigenvectors of a COMPLEX pencil (S,T) in generalized complex Schur
// form (the ZTGEVC analogue; PAPER.md:333 names complex pencils as the next step, SURVEY.md
// s.8(f) NEXT-4).  Every diagonal block is 1x1, so the method is Algorithm 1
// with complex entries: a wavefront over tiles I = M-1 .. 0 of
//   (2) a robust diagonal-tile solve per active eigenvector (k_zdiag, one warp per column,
//       the tile of S and T in shared memory, ProtectDivision / ProtectUpdate per row,
//       PAPER.md:175-200), which also takes the per-column scaling decision of Algorithm 3
//        and stages the scaled B operand [beta x ; -alpha x];
//   (3) the update of every pending row above the tile as ONE complex contraction
//       Y <- Y - [S_panel | T_panel] [sigma beta X_I ; -sigma alpha X_I]   (K = 2 nb),
//       a cuBLAS ZGEMM3M (Gauss's three-multiplication form, R23; ZGEMM with ZZ_Z3M=0) on
//       the DMMA pipe over a contiguous copy of the two panels;
//   (4) consistency and normalisation (max |Re|+|Im| = 1, ZTGEVC's convention).
// Readings R18-R21 of DESIGN.md; the pending-row maximum is carried as an upper bound
// (R21) instead of being measured, so the update needs no epilogue.
#include <cublas_v2.h>
#include <cuComplex.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "../../include/zz.h"
#include "zz_internal.cuh"

int ctx_acquire(cudaStream_t* st, cublasHandle_t* blas, int* mb, zz_info_t** info);

namespace zz {
namespace {

constexpr int kZMaxNB = 64;        // rows per tile: two rows per lane
constexpr int kZWarps = 32;        // columns (warps) per CTA of k_zdiag
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
  double2* B;        // 2 nt x n_act, column-major (ld 2 nt)
  int* sy;           // per column: exponent shift of the pending rows (<= 0)
  double tau_mul;    // 2 (four-multiplication product) or 4 (Gauss 3M, R23)
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
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
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

// A = [S(0:r0, r0:r0+nt) | T(0:r0, r0:r0+nt)], r0 x 2nt column-major (ld r0).
__global__ void k_zpanel(const double2* __restrict__ S, long long lds, const double2* __restrict__ T, long long ldt,
                         int r0, int nt, double2* __restrict__ A) {
  const int col = blockIdx.y;   // 0 .. 2nt-1
  const double2* src = col < nt ? S + (long long)(r0 + col) * lds : T + (long long)(r0 + col - nt) * ldt;
  double2* dst = A + (long long)col * r0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < r0; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

// Robust diagonal-tile solve + Algorithm 3's decision
// + the B operand of the update.  One warp per active column; lane l
// owns tile rows l and l + 32.
__global__ void __launch_bounds__(kZWarps * 32) k_zdiag(ZDiagParams p) {
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
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * kZWarps;
  for (int w = blockIdx.x * kZWarps + (threadIdx.x >> 5); w < p.n_act; w += nw) {
    const int c = p.cs + w;
    const int jl = p.jcol[c] - r0;               // >= nt: not a tip
    const bool tipc = jl < nt;
    const int top = tipc ? jl : nt - 1;
    const double2 al = p.alpha[c];
    const double be = p.beta[c];
    const double aa = fabs(al.x) + fabs(al.y);
    double2* xc = p.X + (long long)c * p.ldx + r0;
    double2 y0 = make_double2(0.0, 0.0), y1 = make_double2(0.0, 0.0);
    if (!tipc) {
      if (lane <= top) y0 = xc[lane];
      if (lane + 32 <= top) y1 = xc[lane + 32];
    }
    int e = tipc ? 0 : p.e_pend[c];
    // Off the dependent chain: the pivots of the lane's two rows (R20) and their reciprocals
    // (Smith's formula for 1/d), the ProtectDivision thresholds, and the bound bw >= max |y|
    // over the pending in-tile rows (exact at the start).
    double2 inv0 = make_double2(0.0, 0.0), inv1 = inv0;
    double td0 = 1.0, td1 = 1.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      if (r <= top) {
        const double2 s = Ss[r * nt + r];
        const double t = Ts[r * nt + r].x;
        double2 d = make_double2(__dsub_rn(__dmul_rn(be, s.x), __dmul_rn(al.x, t)),
                                 __dsub_rn(__dmul_rn(be, s.y), __dmul_rn(al.y, t)));
        const double smin = fmax(kU * (be * zabs1(s) + aa * fabs(t)), kSmlnum);
        if (zabs1(d) < smin) d = make_double2(smin, 0.0);
        const double2 iv = zdiv(make_double2(1.0, 0.0), d);
        const double td = 0.5 * fmin(1.0, zabsm(d));
        if (h == 0) { inv0 = iv; td0 = td; } else { inv1 = iv; td1 = td; }
      }
    }
    double bw = warp_max(fmax(zabsm(y0), zabsm(y1)));
    for (int i = top; i >= 0; --i) {
      const int own = i & 31;
      const bool hi = i >= 32;
      double2 xi;
      if (tipc && i == jl) {
        xi = make_double2(1.0, 0.0);
        if (lane == own) { if (hi) y1 = xi; else y0 = xi; }
      } else {
        // ProtectDivision in the owner lane, then x_i = y_i * (1/d_i)
        int k = 0;
        if (lane == own) k = protect_division(zabsm(hi ? y1 : y0), hi ? td1 : td0);
        k = __shfl_sync(0xffffffffu, k, own);
        if (k < 0) {
          y0 = zldexp(y0, k);
          y1 = zldexp(y1, k);
          bw = ldexp(bw, k);
          e += k;
        }
        if (lane == own) {
          if (hi) y1 = zmul(y1, inv1); else y0 = zmul(y0, inv0);
        }
        const double2 xo = hi ? y1 : y0;
        xi = make_double2(__shfl_sync(0xffffffffu, xo.x, own), __shfl_sync(0xffffffffu, xo.y, own));
      }
      if (i == 0) break;
      // ProtectUpdate of the in-tile rows above (R19 bound).  The bound bw
      // decides first; only when it cannot exclude a scaling is the exact maximum reduced,
      // so the decision is the one the exact maximum gives.
      const double tb = 2.0 * (be * cS[i] + aa * cT[i]);
      double ax = zabsm(xi);
      if (protect_update(bw, tb, ax) < 0) {
        double wm = 0.0;
        if (lane < i) wm = zabsm(y0);
        if (lane + 32 < i) wm = fmax(wm, zabsm(y1));
        wm = warp_max(wm);
        const int k2 = protect_update(wm, tb, ax);
        if (k2 < 0) {
          y0 = zldexp(y0, k2);
          y1 = zldexp(y1, k2);
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
      if (lane < i) y0 = zaxpy2(y0, Ss[i * nt + lane], u, Ts[i * nt + lane], v);
      if (lane + 32 < i) y1 = zaxpy2(y1, Ss[i * nt + lane + 32], u, Ts[i * nt + lane + 32], v);
      bw = bw + tb * ax;
    }
    if (lane <= top) xc[lane] = y0;
    if (lane + 32 <= top) xc[lane + 32] = y1;
    double nx = 0.0, h = 0.0, sums = 0.0;
    if (lane <= top) {
      nx = zabsm(y0);
      h = 0.5 * fabs(y0.x) + 0.5 * fabs(y0.y);
      sums = be * cS[lane] + aa * cT[lane];
    }
    if (lane + 32 <= top) {
      nx = fmax(nx, zabsm(y1));
      h = fmax(h, 0.5 * fabs(y1.x) + 0.5 * fabs(y1.y));
      sums += be * cS[lane + 32] + aa * cT[lane + 32];
    }
    nx = warp_max(nx);
    h = warp_max(h);
    sums = warp_sum(sums);
    if (lane == 0) {
      p.e_seg[c] = e;
      p.nrmh_seg[c] = h;
    }
    if (r0 == 0) continue;
    // Algorithm 3: one exponent for the pending rows after the update
    const int ep = tipc ? 0 : p.e_pend[c];
    const int g = min(ep, e);
    const double yh = ldexp(tipc ? 0.0 : p.nYb[c], g - ep);
    const double xh = ldexp(nx, g - e);
    const double tau = p.tau_mul * sums;
    const int ed = protect_update(yh, tau, xh);
    const int en = g + ed;
    const int sy = en - ep, sx = en - e;
    __syncwarp();
    if (lane == 0) {
      p.e_pend[c] = en;
      // R21: the bound 2^ed (yh + tau xh), not a measurement; tau xh itself may exceed the
      // range when ed < 0, so that product is formed as protect_update does (scaled by 2^-1023)
      const double bnd = ed == 0 ? yh + tau * xh
                                 : ldexp(yh, ed) + ldexp(ldexp(tau, -512) * ldexp(xh, -511), ed + 1023);
      p.nYb[c] = bnd * (1.0 + 0x1p-40);
    }
    if (lane == 0) p.sy[c] = sy;   // applied to the pending rows by k_zscale_pending
    double2* Bc = p.B + (long long)w * 2 * nt;
    const double2 x0 = zldexp(y0, sx), x1 = zldexp(y1, sx);
    if (lane < nt) {
      const bool z = lane > top;
      Bc[lane] = z ? make_double2(0.0, 0.0) : make_double2(be * x0.x, be * x0.y);
      const double2 q = zmul(al, x0);
      Bc[nt + lane] = z ? make_double2(0.0, 0.0) : make_double2(-q.x, -q.y);
    }
    if (lane + 32 < nt) {
      const bool z = lane + 32 > top;
      Bc[lane + 32] = z ? make_double2(0.0, 0.0) : make_double2(be * x1.x, be * x1.y);
      const double2 q = zmul(al, x1);
      Bc[nt + lane + 32] = z ? make_double2(0.0, 0.0) : make_double2(-q.x, -q.y);
    }
  }
}

// sigma_Y of Algorithm 3: Y(0:r0, c) <- 2^sy[c] Y(0:r0, c) for the columns whose decision
// scaled (rare); one warp per active column.  Runs on the update's stream, after the previous
// step's update has written those rows.
__global__ void k_zscale_pending(double2* X, long long ldx, int r0, int cs, int n_act, const int* __restrict__ sy) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= n_act) return;
  const int c = cs + w;
  const int k = sy[c];
  if (k >= 0) return;
  double2* yc = X + (long long)c * ldx;
  for (int i = threadIdx.x & 31; i < r0; i += 32) yc[i] = zldexp(yc[i], k);
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

struct ZWork {
  void* p = nullptr;
  size_t n = 0;
  cudaStream_t st = nullptr;
  cudaError_t alloc(size_t bytes, cudaStream_t s) {
    st = s;
    n = bytes;
    return cudaMallocAsync(&p, bytes, s);
  }
  ~ZWork() {
    if (p) cudaFreeAsync(p, st);
  }
};

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
  cudaStream_t st;
  cublasHandle_t blas;
  int mb_ctx;
  zz_info_t* info;
  int r = ctx_acquire(&st, &blas, &mb_ctx, &info);
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
  // workspace (stream-ordered)
  size_t off[13], tot = 0;
  const size_t sz[13] = {sizeof(int) * n, sizeof(double2) * n, sizeof(double) * n, sizeof(int) * n, sizeof(double) * n,
                         sizeof(int) * (size_t)M * n, sizeof(double) * (size_t)M * n, sizeof(double) * m,
                         sizeof(double) * m, sizeof(double2) * 4 * (size_t)nb * n,
                         sizeof(double2) * 2 * (size_t)nb * (size_t)m, sizeof(int) * 4, sizeof(int) * n};
  for (int i = 0; i < 13; ++i) { off[i] = tot; tot += align256(sz[i]); }
  ZWork wk;
  ZCK(wk.alloc(tot, st));
  char* base = static_cast<char*>(wk.p);
  int* d_jcol = reinterpret_cast<int*>(base + off[0]);
  double2* d_alpha = reinterpret_cast<double2*>(base + off[1]);
  double* d_beta = reinterpret_cast<double*>(base + off[2]);
  int* d_epend = reinterpret_cast<int*>(base + off[3]);
  double* d_nYb = reinterpret_cast<double*>(base + off[4]);
  int* d_eseg = reinterpret_cast<int*>(base + off[5]);
  double* d_nrmh = reinterpret_cast<double*>(base + off[6]);
  double* d_cmS = reinterpret_cast<double*>(base + off[7]);
  double* d_cmT = reinterpret_cast<double*>(base + off[8]);
  double2* d_B = reinterpret_cast<double2*>(base + off[9]);
  double2* d_A = reinterpret_cast<double2*>(base + off[10]);
  int* d_status = reinterpret_cast<int*>(base + off[11]);
  int* d_sy = reinterpret_cast<int*>(base + off[12]);
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
  ZCK(cudaFuncSetAttribute(k_zdiag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
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
  // Lookahead (DESIGN.md s.6 "Complex pencils"): the update of step I is split into the band
  // (the rows of tile I-1) and the rest; the solve of tile I-1 runs on a high-priority stream
  // beside the rest.  The scaling decisions use the pending bound (R21), so the solve needs
  // nothing from the rest; sigma_Y is applied by k_zscale_pending on the update stream.
  const char* la_env = getenv("ZZ_ZLOOKAHEAD");
  const bool la = (la_env ? atoi(la_env) != 0 : true) && Itop >= 1;
  cudaStream_t hp = nullptr;
  cudaEvent_t ev_band = nullptr, ev_diag = nullptr;
  struct Guard {
    cudaStream_t& h; cudaEvent_t& a; cudaEvent_t& b;
    ~Guard() { if (h) cudaStreamDestroy(h); if (a) cudaEventDestroy(a); if (b) cudaEventDestroy(b); }
  } guard{hp, ev_band, ev_diag};
  if (la) {
    int lo, hi;
    ZCK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    ZCK(cudaStreamCreateWithPriority(&hp, cudaStreamNonBlocking, hi));
    ZCK(cudaEventCreateWithFlags(&ev_band, cudaEventDisableTiming));
    ZCK(cudaEventCreateWithFlags(&ev_diag, cudaEventDisableTiming));
  }
  // Gauss's three-multiplication complex product (cublasZgemm3m, default; ZZ_Z3M=0 selects
  // ZGEMM): 25 % fewer real flops; its (Ar + Ai)(Br + Bi) partial sums are up to twice the
  // four-multiplication bound, so Algorithm 3's tau doubles (R23)
  const bool use3m = !(getenv("ZZ_Z3M") && atoi(getenv("ZZ_Z3M")) == 0);
  const size_t bsz = 2 * (size_t)nb * n;
  auto diag = [&](int I, cudaStream_t s) -> cudaError_t {
    const int r0 = I * nb, nt = std::min(nb, m - r0), cs = csI[I], n_act = n - cs;
    ZDiagParams p;
    p.I = I; p.r0 = r0; p.nt = nt; p.cs = cs; p.n_act = n_act; p.n_sel = n;
    p.S = S; p.lds = lds; p.T = T; p.ldt = ldt; p.X = X; p.ldx = ldx;
    p.jcol = d_jcol; p.alpha = d_alpha; p.beta = d_beta; p.cmS = d_cmS; p.cmT = d_cmT;
    p.e_pend = d_epend; p.nYb = d_nYb;
    p.e_seg = d_eseg + (size_t)I * n;
    p.nrmh_seg = d_nrmh + (size_t)I * n;
    p.B = d_B + (size_t)(I & 1) * bsz;
    p.sy = d_sy;
    p.tau_mul = use3m ? 4.0 : 2.0;
    const int grid = std::min((n_act + kZWarps - 1) / kZWarps, nsm);   // one 132 KB CTA per SM
    k_zdiag<<<grid, kZWarps * 32, smem, s>>>(p);
    ++launches;
    return cudaGetLastError();
  };
  const cuDoubleComplex mone = make_cuDoubleComplex(-1.0, 0.0), one = make_cuDoubleComplex(1.0, 0.0);
  // Y(row0:row0+rows, cs:n) <- Y - [S_panel | T_panel](row0:row0+rows, :) [sigma beta X_I ; -sigma alpha X_I]
  auto gemm = [&](int I, int row0, int rows) -> int {
    const int r0 = I * nb, nt = std::min(nb, m - r0), cs = csI[I], n_act = n - cs;
    if ((use3m ? cublasZgemm3m : cublasZgemm)(blas, CUBLAS_OP_N, CUBLAS_OP_N, rows, n_act, 2 * nt, &mone,
                    reinterpret_cast<const cuDoubleComplex*>(d_A + row0), r0,
                    reinterpret_cast<const cuDoubleComplex*>(d_B + (size_t)(I & 1) * bsz), 2 * nt, &one,
                    reinterpret_cast<cuDoubleComplex*>(X + (size_t)cs * ldx + row0), ldx) != CUBLAS_STATUS_SUCCESS)
      return ZZ_ERR_CUDA;
    ++launches;
    info->update_launches++;
    return 0;
  };
  if (Itop >= 0) ZCK(diag(Itop, st));
  for (int I = Itop; I >= 0; --I) {
    const int r0 = I * nb, nt = std::min(nb, m - r0), cs = csI[I], n_act = n - cs;
    if (la && I < Itop) ZCK(cudaStreamWaitEvent(st, ev_diag, 0));
    if (r0 == 0) break;
    k_zscale_pending<<<(n_act + 7) / 8, 256, 0, st>>>(X, ldx, r0, cs, n_act, d_sy);
    k_zpanel<<<dim3((r0 + 255) / 256 > 64 ? 64 : (r0 + 255) / 256, 2 * nt), 256, 0, st>>>(S, lds, T, ldt, r0, nt, d_A);
    launches += 2;
    ZCK(cudaGetLastError());
    if (la) {
      const int rb = r0 - nb;   // tile I-1 is a full tile
      if ((r = gemm(I, rb, nb))) return r;
      ZCK(cudaEventRecord(ev_band, st));
      ZCK(cudaStreamWaitEvent(hp, ev_band, 0));
      ZCK(diag(I - 1, hp));
      ZCK(cudaEventRecord(ev_diag, hp));
      if (rb > 0 && (r = gemm(I, 0, rb))) return r;
    } else {
      if ((r = gemm(I, 0, r0))) return r;
      ZCK(diag(I - 1, st));
    }
  }
  k_znorm<<<n, 256, 0, st>>>(X, ldx, nb, n, d_jcol, d_eseg, d_nrmh, col_scale_exp);
  ++launches;
  ZCK(cudaGetLastError());
  info->total_launches = launches;
  ZCK(cudaStreamSynchronize(st));
  return 0;
}
