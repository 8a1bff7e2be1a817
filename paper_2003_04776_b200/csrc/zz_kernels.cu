// zz_kernels.cu -- sm_100a kernels of the robust eigenvector path other than the update:
// structure scan, eigenvalue pairs, panel norms, the robust diagonal-block solve (tips and
// right-hand sides) with the per-column scaling decision, and the consistency /
// normalisation pass.  Readings R1..R17 refer to DESIGN.md.
#include <math.h>
#include <stdint.h>

#include "zz_internal.cuh"
#include "zz_device.cuh"

namespace zz {

#define FULL 0xffffffffu

// ------------------------------------------------------------------------------------
// Structure scan: gather the subdiagonal S(j+1, j), j < m-1.
// ------------------------------------------------------------------------------------
__global__ void k_subdiag(const double* __restrict__ S, long long lds, int m, double* sub) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m - 1) sub[j] = S[(long long)j * lds + j + 1];
}
cudaError_t launch_subdiag(const double* S, long long lds, int m, double* sub, cudaStream_t st) {
  if (m < 2) return cudaSuccess;
  k_subdiag<<<(m + 255) / 256, 256, 0, st>>>(S, lds, m, sub);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// Eigenvalue pairs (alpha, beta), alpha = a + i b (readings R2, R3),
// normalised by an exact power of two so that max(beta, |a|+|b|) in [1/2, 1).  Every
// operation is an explicit round-to-nearest intrinsic (no contraction), so the pairs --
// and hence the pivots beta S_ii - alpha T_ii -- are fixed bit patterns (reading R17).
// ------------------------------------------------------------------------------------
__device__ void normalise_pair(double& a, double& b, double& beta, int& kind) {
  double h = dmaxd(__dmul_rn(0.5, beta), __dadd_rn(__dmul_rn(0.5, fabs(a)), __dmul_rn(0.5, fabs(b))));
  if (h == 0.0) { kind = kIndefinite; return; }
  int k;
  frexp(h, &k);
  a = ldexp(a, -(k + 1));
  b = ldexp(b, -(k + 1));
  beta = ldexp(beta, -(k + 1));
}

// returns 0 ok, 1 real eigenvalues (not a complex pair)
__device__ int pair_2x2(double s11, double s21, double s12, double s22, double t11, double t12,
                        double t22, double& a, double& b, double& beta) {
  double ms = dmaxd(dmaxd(fabs(s11), fabs(s12)), dmaxd(fabs(s21), fabs(s22)));
  double mt = dmaxd(dmaxd(fabs(t11), fabs(t12)), fabs(t22));
  if (!(ms > 0.0) || !(mt > 0.0)) return 1;
  int ks, kt;
  frexp(ms, &ks);
  frexp(mt, &kt);
  s11 = ldexp(s11, -ks); s21 = ldexp(s21, -ks); s12 = ldexp(s12, -ks); s22 = ldexp(s22, -ks);
  t11 = ldexp(t11, -kt); t12 = ldexp(t12, -kt); t22 = ldexp(t22, -kt);
  if (t11 == 0.0 || t22 == 0.0) return 1;
  // eigenvalues of N = T_blk^{-1} S_blk: p +- i q (reading R3)
  double n21 = __ddiv_rn(s21, t22);
  double n11 = __ddiv_rn(__dsub_rn(s11, __dmul_rn(t12, n21)), t11);
  double n12 = __ddiv_rn(__dsub_rn(s12, __dmul_rn(t12, __ddiv_rn(s22, t22))), t11);
  double n22 = __ddiv_rn(s22, t22);
  double d = __dmul_rn(__dsub_rn(n11, n22), 0.5);
  double disc = __dadd_rn(__dmul_rn(d, d), __dmul_rn(n12, n21));
  if (!(disc < 0.0)) return 1;
  a = __dadd_rn(n22, d);
  b = __dsqrt_rn(-disc);
  beta = ldexp(1.0, kt - ks);
  return 0;
}

__global__ void k_pairs(const double* __restrict__ S, long long lds, const double* __restrict__ T,
                        long long ldt, int p0, int nblk, DevPlan P) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nblk) return;
  const int p = p0 + idx;
  int j = P.blk_start[p], sz = P.blk_size[p];
  double a, b, beta;
  int kind = kReal, err = 0;
  if (sz == 1) {
    double s = S[(long long)j * lds + j], t = T[(long long)j * ldt + j];
    if (!isfinite(s) || !isfinite(t)) err = 1;
    a = s; b = 0.0; beta = t;
    if (beta < 0) { a = -a; beta = -beta; }
    normalise_pair(a, b, beta, kind);
  } else {
    double s11 = S[(long long)j * lds + j], s21 = S[(long long)j * lds + j + 1];
    double s12 = S[(long long)(j + 1) * lds + j], s22 = S[(long long)(j + 1) * lds + j + 1];
    double t11 = T[(long long)j * ldt + j], t12 = T[(long long)(j + 1) * ldt + j];
    double t22 = T[(long long)(j + 1) * ldt + j + 1];
    if (!isfinite(s11) || !isfinite(s21) || !isfinite(s12) || !isfinite(s22) || !isfinite(t11) ||
        !isfinite(t12) || !isfinite(t22))
      err = 1;
    else if (pair_2x2(s11, s21, s12, s22, t11, t12, t22, a, b, beta))
      err = 2;
    else {
      kind = kPairFirst;
      normalise_pair(a, b, beta, kind);
    }
  }
  if (err) {
    atomicMin(&P.status[0], p * 4 + err);
    return;
  }
  int c = P.blk_col[p];
  if (c < 0) return;
  if (kind == kIndefinite) atomicAdd(&P.status[2], 1);
  P.col_a[c] = a; P.col_b[c] = b; P.col_beta[c] = beta; P.col_kind[c] = kind;
  if (sz == 2) {
    P.col_a[c + 1] = a; P.col_b[c + 1] = b; P.col_beta[c + 1] = beta; P.col_kind[c + 1] = kPairSecond;
  }
}
cudaError_t launch_pairs(const double* S, long long lds, const double* T, long long ldt, int p0, int nblk,
                         const DevPlan& P, cudaStream_t st) {
  if (nblk <= 0) return cudaSuccess;
  k_pairs<<<(nblk + 127) / 128, 128, 0, st>>>(S, lds, T, ldt, p0, nblk, P);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// Max |entry| of the upper part (+ subdiagonal) of S and T (rare pre-scale path, R6).
// ------------------------------------------------------------------------------------
__global__ void k_maxabs(const double* __restrict__ S, long long lds, const double* __restrict__ T,
                         long long ldt, int m, unsigned long long* out) {
  double ms = 0.0, mt = 0.0;
  for (int j = blockIdx.x; j < m; j += gridDim.x) {
    int ie = min(j + 1, m - 1);
    for (int i = threadIdx.x; i <= ie; i += blockDim.x) {
      ms = fmax(ms, fabs(S[(long long)j * lds + i]));
      mt = fmax(mt, fabs(T[(long long)j * ldt + i]));
    }
  }
  for (int o = 16; o; o >>= 1) {
    ms = fmax(ms, __shfl_xor_sync(FULL, ms, o));
    mt = fmax(mt, __shfl_xor_sync(FULL, mt, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out[0], (unsigned long long)__double_as_longlong(ms));
    atomicMax(&out[1], (unsigned long long)__double_as_longlong(mt));
  }
}
cudaError_t launch_maxabs(const double* S, long long lds, const double* T, long long ldt, int m,
                          unsigned long long* out, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_maxabs<<<min(m, 4096), 256, 0, st>>>(S, lds, T, ldt, m, out);
  return cudaGetLastError();
}

// scaled copy of the upper part (+ subdiagonal): B = 2^-k A (rare pre-scale / repack path)
__global__ void k_scale_copy(const double* __restrict__ A, long long lda, int m, int k, double* B,
                             long long ldb) {
  for (int j = blockIdx.x; j < m; j += gridDim.x) {
    int ie = min(j + 1, m - 1);
    for (int i = threadIdx.x; i < m; i += blockDim.x)
      B[(long long)j * ldb + i] = (i <= ie) ? ldexp(A[(long long)j * lda + i], -k) : 0.0;
  }
}
cudaError_t launch_scale_copy(const double* A, long long lda, int m, int k, double* B, long long ldb,
                              cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_scale_copy<<<min(m, 8192), 256, 0, st>>>(A, lda, m, k, B, ldb);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// Panel norms: for every tile column J >= 1,
//   cS[J] = max_{i < ts_J} sum_{k in tile J} |S_ik|   (the infinity norm of the panel
// above the diagonal tile), cT likewise.  Also dS[J], dT[J] = the largest row sum of the
// upper part of the diagonal tile (used only for the pre-scale test, reading R6).
// One thread per row; consecutive threads read consecutive rows of a column (coalesced).
// ------------------------------------------------------------------------------------
__global__ void k_panel_norms(const double* __restrict__ S, long long lds,
                              const double* __restrict__ T, long long ldt,
                              const int* __restrict__ tile_start, int J0, double* cS, double* cT,
                              double* dS, double* dT) {
  int J = J0 + blockIdx.y;
  int k0 = tile_start[J], k1 = tile_start[J + 1];
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.x * blockDim.x >= k1) return;
  bool diag = (i >= k0);
  int kb = diag ? max(k0, i - 1) : k0;
  double s = 0.0, t = 0.0;
  if (i < k1) {
    const double* sp = S + (long long)i;
    const double* tp = T + (long long)i;
    int k = kb;
#pragma unroll 16
    for (; k < k1; ++k) {
      s += fabs(sp[(long long)k * lds]);
      t += fabs(tp[(long long)k * ldt]);
    }
  }
  // warp max, split by region
  double sp_ = diag ? 0.0 : s, tp_ = diag ? 0.0 : t;
  double sd_ = diag ? s : 0.0, td_ = diag ? t : 0.0;
  for (int o = 16; o; o >>= 1) {
    sp_ = fmax(sp_, __shfl_xor_sync(FULL, sp_, o));
    tp_ = fmax(tp_, __shfl_xor_sync(FULL, tp_, o));
    sd_ = fmax(sd_, __shfl_xor_sync(FULL, sd_, o));
    td_ = fmax(td_, __shfl_xor_sync(FULL, td_, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (sp_ > 0) atomicMax((unsigned long long*)&cS[J], (unsigned long long)__double_as_longlong(sp_));
    if (tp_ > 0) atomicMax((unsigned long long*)&cT[J], (unsigned long long)__double_as_longlong(tp_));
    if (sd_ > 0) atomicMax((unsigned long long*)&dS[J], (unsigned long long)__double_as_longlong(sd_));
    if (td_ > 0) atomicMax((unsigned long long*)&dT[J], (unsigned long long)__double_as_longlong(td_));
  }
}
// tile 0's diagonal part
__global__ void k_diag0_norms(const double* __restrict__ S, long long lds,
                              const double* __restrict__ T, long long ldt,
                              const int* __restrict__ tile_start, double* dS, double* dT) {
  int k1 = tile_start[1];
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0, t = 0.0;
  if (i < k1) {
    // unrolled: the loads of 16 columns are in flight together (the sums keep their order)
#pragma unroll 16
    for (int k = max(0, i - 1); k < k1; ++k) {
      s += fabs(S[(long long)k * lds + i]);
      t += fabs(T[(long long)k * ldt + i]);
    }
  }
  for (int o = 16; o; o >>= 1) {
    s = fmax(s, __shfl_xor_sync(FULL, s, o));
    t = fmax(t, __shfl_xor_sync(FULL, t, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax((unsigned long long*)&dS[0], (unsigned long long)__double_as_longlong(s));
    atomicMax((unsigned long long*)&dT[0], (unsigned long long)__double_as_longlong(t));
  }
}
cudaError_t launch_panel_norms(const double* S, long long lds, const double* T, long long ldt, int M,
                               const int* tile_start_host, const DevPlan& P, cudaStream_t st, int J0, int nJ) {
  // cS, cT, dS, dT are 4 consecutive arrays of M doubles (zeroed by the caller); panels
  // J0 .. J0+nJ-1 (J = 0 is the first tile's diagonal part only)
  double* dS = P.cS + 2 * (long long)M;
  double* dT = P.cS + 3 * (long long)M;
  if (nJ <= 0) return cudaSuccess;
  if (J0 == 0) {
    int k1 = tile_start_host[1];
    k_diag0_norms<<<(k1 + 255) / 256, 256, 0, st>>>(S, lds, T, ldt, P.tile_start, dS, dT);
    J0 = 1;
    nJ -= 1;
  }
  if (nJ > 0) {
    int rows = tile_start_host[J0 + nJ];
    dim3 grid((rows + 255) / 256, nJ);
    k_panel_norms<<<grid, 256, 0, st>>>(S, lds, T, ldt, P.tile_start, J0, P.cS, P.cT, dS, dT);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// Robust diagonal-block solve (Kernel 1 tips and Kernel 3 solves, PAPER.md:150-163, 282;
// Alg. 1 lines P:137) fused with the per-column scaling decision of the
// following update (Algs. 2/3) and the formation of its B operand.
//
// One warp per eigenvector (real column or complex pair); lane l holds rows
// l, l+32, ..., of the tile in registers.  The diagonal tile of S and T (upper part and
// subdiagonal) is staged once per CTA in shared memory, column-major packed.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int poff(int j) { return j * (j + 3) / 2; }

template <int NQ>
__device__ __forceinline__ double get_row(const double (&y)[NQ], int k) {
  int q = k >> 5;
  double v = y[0];
#pragma unroll
  for (int s = 1; s < NQ; ++s)
    if (q == s) v = y[s];
  return __shfl_sync(FULL, v, k & 31);
}
template <int NQ>
__device__ __forceinline__ void set_row(double (&y)[NQ], int k, double v, int lane) {
  int q = k >> 5;
#pragma unroll
  for (int s = 0; s < NQ; ++s)
    if (q == s && lane == (k & 31)) y[s] = v;
}
template <int NQ>
__device__ __forceinline__ void scale_all(double (&yr)[NQ], double (&yi)[NQ], int k) {
#pragma unroll
  for (int s = 0; s < NQ; ++s) {
    yr[s] = ldexp(yr[s], k);
    yi[s] = ldexp(yi[s], k);
  }
}

// upper bound (within 2^-20 relative) of the max over lanes of a non-negative double
__device__ __forceinline__ double warp_max_bound(double v) {
  unsigned hi = (unsigned)__double2hiint(v);
  hi = __reduce_max_sync(FULL, hi);
  return __hiloint2double((int)hi, (int)0xFFFFFFFFu);
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// shared context of one warp's eigenvector
template <int NQ, bool PAIR>
struct Vec {
  double yr[NQ], yi[NQ];
  int e;   // accumulated local exponent of the segment
  __device__ __forceinline__ cpx get(int k) const {
    cpx z;
    z.re = get_row<NQ>(yr, k);
    z.im = PAIR ? get_row<NQ>(yi, k) : 0.0;
    return z;
  }
  __device__ __forceinline__ void put(int k, cpx z, int lane) {
    set_row<NQ>(yr, k, z.re, lane);
    if (PAIR) set_row<NQ>(yi, k, z.im, lane);
  }
  __device__ __forceinline__ void scale(int k) {
    if (k < 0) {
#pragma unroll
      for (int s = 0; s < NQ; ++s) {
        yr[s] = ldexp(yr[s], k);
        if (PAIR) yi[s] = ldexp(yi[s], k);
      }
      e += k;
    }
  }
};

// Robust division of the value z (already scaled with the vector) by d (reading R9).
template <int NQ, bool PAIR>
__device__ __forceinline__ cpx pdiv(Vec<NQ, PAIR>& v, cpx& z, cpx d) {
  if (!PAIR) {
    int k = protect_division(fabs(z.re), fabs(d.re));
    if (k < 0) { v.scale(k); z.re = ldexp(z.re, k); }
    return mkc(__ddiv_rn(z.re, d.re), 0.0);
  }
  int k = protect_division(nmax(z), __dmul_rn(0.5, dmind(1.0, nmax(d))));
  if (k < 0) { v.scale(k); z.re = ldexp(z.re, k); z.im = ldexp(z.im, k); }
  return cdivx(z, d);
}

struct Tile {
  const double* Sp;
  const double* Tp;
  const double* cmS;
  const double* cmT;
  const signed char* fl;
  __device__ __forceinline__ double s(int i, int j) const { return Sp[poff(j) + i]; }
  __device__ __forceinline__ double t(int i, int j) const { return Tp[poff(j) + i]; }
};

// in-tile update of the pending rows [0, ks) with the solved block rows [ks, ke]
template <int NQ, bool PAIR>
__device__ __forceinline__ void update_above(Vec<NQ, PAIR>& v, const Tile& tl, int ks, int ke, double a,
                                             double b, double beta, double ab, int lane) {
  if (ks <= 0) return;
  cpx x0 = v.get(ks);
  cpx x1 = (ke > ks) ? v.get(ke) : mkc(0.0, 0.0);
  // ProtectUpdate(max pending, t, |x|) over the block
  double xn = dmaxd(nmax(x0), nmax(x1));
  double t = 0.0;
  for (int k = ks; k <= ke; ++k)
    t = __dadd_rn(t, __dadd_rn(__dmul_rn(beta, tl.cmS[k]), __dmul_rn(ab, tl.cmT[k])));
  double lm = 0.0;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    int row = lane + 32 * q;
    if (row < ks) lm = fmax(lm, PAIR ? fmax(fabs(v.yr[q]), fabs(v.yi[q])) : fabs(v.yr[q]));
  }
  double ymax = warp_max_bound(lm);
  int eu = protect_update(ymax, t, xn);
  if (eu < 0) {
    v.scale(eu);
    x0.re = ldexp(x0.re, eu); x0.im = ldexp(x0.im, eu);
    x1.re = ldexp(x1.re, eu); x1.im = ldexp(x1.im, eu);
  }
  for (int k = ks; k <= ke; ++k) {
    cpx x = (k == ks) ? x0 : x1;
    // u = x D (beta x), w = x B (alpha x)
    double ur = beta * x.re, ui = beta * x.im;
    double wr = PAIR ? (a * x.re - b * x.im) : a * x.re;
    double wi = PAIR ? (a * x.im + b * x.re) : 0.0;
    const double* sc = tl.Sp + poff(k);
    const double* tc = tl.Tp + poff(k);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      int row = lane + 32 * q;
      if (row < ks) {
        double sv = sc[row], tv = tc[row];
        v.yr[q] = fma(tv, wr, fma(-sv, ur, v.yr[q]));
        if (PAIR) v.yi[q] = fma(tv, wi, fma(-sv, ui, v.yi[q]));
      }
    }
  }
}

// 1x1 row j: (beta S_jj - alpha T_jj) x_j = y_j
template <int NQ, bool PAIR>
__device__ __forceinline__ void solve1(Vec<NQ, PAIR>& v, const Tile& tl, int j, double a, double b,
                                       double beta, double ab, int lane) {
  double sjj = tl.s(j, j), tjj = tl.t(j, j);
  cpx d = mkc(__fma_rn(-a, tjj, __dmul_rn(beta, sjj)), __dmul_rn(-b, tjj));
  double smin = dmaxd(__dmul_rn(kU, __dadd_rn(__dmul_rn(beta, fabs(sjj)), __dmul_rn(ab, fabs(tjj)))), kSmlnum);
  if (n1(d) < smin) d = mkc(smin, 0.0);
  cpx z = v.get(j);
  cpx x = pdiv<NQ, PAIR>(v, z, d);
  v.put(j, x, lane);
}

// 2x2 rows (j, j+1): complete pivoting on |Re|+|Im|, pivots below smin -> smin (R9)
template <int NQ, bool PAIR>
__device__ __forceinline__ void solve2(Vec<NQ, PAIR>& v, const Tile& tl, int j, double a, double b,
                                       double beta, double ab, int lane) {
  double s11 = tl.s(j, j), s21 = tl.s(j + 1, j), s12 = tl.s(j, j + 1), s22 = tl.s(j + 1, j + 1);
  double t11 = tl.t(j, j), t12 = tl.t(j, j + 1), t22 = tl.t(j + 1, j + 1);
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
  int i1 = j + pr, i2 = j + 1 - pr;
  cpx w1 = v.get(i1), w2 = v.get(i2);
  // forward step y2 <- y2 - l y1
  {
    double wn = dmaxd(nmax(w1), nmax(w2));
    int k = protect_update(wn, 2.0, wn);
    if (k < 0) {
      v.scale(k);
      w1 = mkc(ldexp(w1.re, k), ldexp(w1.im, k));
      w2 = mkc(ldexp(w2.re, k), ldexp(w2.im, k));
    }
  }
  w2 = csubx(w2, cmulx(l, w1));
  // z2 = y2 / u22
  int e0 = v.e;
  cpx z2 = pdiv<NQ, PAIR>(v, w2, u22);
  if (v.e != e0) w1 = mkc(ldexp(w1.re, v.e - e0), ldexp(w1.im, v.e - e0));
  // z1 = (y1 - cc z2) / p
  {
    int k = protect_update(nmax(w1), n1(cc), nmax(z2));
    if (k < 0) {
      v.scale(k);
      w1 = mkc(ldexp(w1.re, k), ldexp(w1.im, k));
      z2 = mkc(ldexp(z2.re, k), ldexp(z2.im, k));
    }
  }
  cpx nn = csubx(w1, cmulx(cc, z2));
  e0 = v.e;
  cpx z1 = pdiv<NQ, PAIR>(v, nn, p);
  if (v.e != e0) z2 = mkc(ldexp(z2.re, v.e - e0), ldexp(z2.im, v.e - e0));
  v.put(j + pc, z1, lane);
  v.put(j + 1 - pc, z2, lane);
}

template <int NQ, bool PAIR>
__device__ void solve_item(const DiagParams& p, const Tile& tl, int c, int lane) {
  const DevPlan& P = p.P;
  const int nt = p.nt;
  const double a = P.col_a[c], b = PAIR ? P.col_b[c] : 0.0, beta = P.col_beta[c];
  const int kind = P.col_kind[c];
  const bool tip = c < p.tip_col_end;
  const double ab = __dadd_rn(fabs(a), fabs(b));
  Vec<NQ, PAIR> v;
  v.e = 0;
  const double* xc = p.X + (long long)c * p.ldx + p.t0;
  const double* xc1 = xc + p.ldx;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    int row = lane + 32 * q;
    bool ld = !tip && row < nt;
    v.yr[q] = ld ? xc[row] : 0.0;
    v.yi[q] = (PAIR && ld) ? xc1[row] : 0.0;
  }
  int j;
  if (kind == kIndefinite) {
    // indefinite eigenvalue: the unit vector e_r (reading R13), no substitution
#pragma unroll
    for (int q = 0; q < NQ; ++q) { v.yr[q] = 0.0; v.yi[q] = 0.0; }
    if (tip) v.put(P.col_r[c] - p.t0, mkc(1.0, 0.0), lane);
    j = -1;
  } else if (tip) {
    int rr = P.col_r[c] - p.t0;
    if (!PAIR) {
      v.put(rr, mkc(1.0, 0.0), lane);
      update_above<NQ, PAIR>(v, tl, rr, rr, a, b, beta, ab, lane);
      j = rr - 1;
    } else {
      // tip of a complex pair (reading R10)
      double pp = __dmul_rn(beta, tl.s(rr, rr - 1));
      cpx q = mkc(__fma_rn(-a, tl.t(rr, rr), __dmul_rn(beta, tl.s(rr, rr))), __dmul_rn(-b, tl.t(rr, rr)));
      cpx zr, zr1;
      if (fabs(pp) >= n1(q)) {
        zr = mkc(1.0, 0.0);
        zr1 = mkc(__ddiv_rn(-q.re, pp), __ddiv_rn(-q.im, pp));
      } else {
        zr1 = mkc(1.0, 0.0);
        cpx z = cdivx(mkc(pp, 0.0), q);
        zr = mkc(-z.re, -z.im);
      }
      v.put(rr, zr, lane);
      v.put(rr - 1, zr1, lane);
      update_above<NQ, PAIR>(v, tl, rr - 1, rr, a, b, beta, ab, lane);
      j = rr - 2;
    }
  } else {
    j = nt - 1;
  }
  // bottom-up substitution over the 1x1 / 2x2 blocks of the tile
  while (j >= 0) {
    bool two = tl.fl[j] == kRowBot2;
    int js = two ? j - 1 : j;
    if (two) solve2<NQ, PAIR>(v, tl, js, a, b, beta, ab, lane);
    else solve1<NQ, PAIR>(v, tl, j, a, b, beta, ab, lane);
    update_above<NQ, PAIR>(v, tl, js, j, a, b, beta, ab, lane);
    j = js - 1;
  }
  // store the solved segment and its norms
  double* xo = p.X + (long long)c * p.ldx + p.t0;
  double lm = 0.0, lh = 0.0;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    int row = lane + 32 * q;
    if (row < nt) {
      xo[row] = v.yr[q];
      if (PAIR) xo[row + p.ldx] = v.yi[q];
      lm = fmax(lm, PAIR ? fmax(fabs(v.yr[q]), fabs(v.yi[q])) : fabs(v.yr[q]));
      lh = fmax(lh, PAIR ? __dadd_rn(__dmul_rn(0.5, fabs(v.yr[q])), __dmul_rn(0.5, fabs(v.yi[q])))
                         : __dmul_rn(0.5, fabs(v.yr[q])));
    }
  }
  double nrm = warp_max(lm), nrmh = warp_max(lh);
  const int ep = tip ? 0 : P.e_pend[c];
  const int es = ep + v.e;
  const long long so = (long long)p.I * p.n_sel + c;
  if (lane == 0) {
    P.e_seg[so] = es;
    P.nrm_seg[so] = nrm;
    P.nrmh_seg[so] = nrmh;
    if (PAIR) { P.e_seg[so + 1] = es; P.nrm_seg[so + 1] = nrm; P.nrmh_seg[so + 1] = nrmh; }
  }
  if (!p.do_update) return;
  // scaling decision of the update at this step (Alg. 3 P:253-259 with Alg. 2 P:228-232;
  // reading R5): align to gamma = min exponent, then ProtectUpdate.
  // pending max of the column (a pair: of both of its columns)
  double nyv = tip ? 0.0 : __longlong_as_double((long long)P.nY[(long long)p.nY_in * p.n_sel + c]);
  if (PAIR && !tip) nyv = dmaxd(nyv, __longlong_as_double((long long)P.nY[(long long)p.nY_in * p.n_sel + c + 1]));
  int g = min(ep, es);
  double yh = ldexp(nyv, g - ep), xh = ldexp(nrm, g - es);
  double tau = __dadd_rn(__dmul_rn(beta, p.P.cS[p.I]), __dmul_rn(ab, p.P.cT[p.I]));
  int ed = protect_update(yh, tau, xh);
  int en = g + ed;
  int sx = en - es;
  if (lane == 0) {
    P.sY[c] = en - ep;
    P.e_pend[c] = en;
    P.nY[(long long)(1 - p.nY_in) * p.n_sel + c] = 0ull;
    if (PAIR) {
      P.sY[c + 1] = en - ep;
      P.e_pend[c + 1] = en;
      P.nY[(long long)(1 - p.nY_in) * p.n_sel + c + 1] = 0ull;
    }
  }
  // B operand of the update: W = [-2^sx X_I D ; 2^sx X_I B], written in
  // the update kernel's stage layout [ntile][kc][BK/4][BN][4].
  const int kext = p.nks * kBK;
  const long long tstride = (long long)(2 * p.nks) * (kBN * kBK);
  // element (k, col) of W in the update kernel's stage layout; a pair may straddle tiles
  auto wp = [&](int col, int chunk, int kk) -> double* {
    return p.P.W + (long long)(col / kBN) * tstride + (long long)chunk * (kBN * kBK) +
           (long long)(kk >> 2) * (kBN * 4) + (col % kBN) * 4 + (kk & 3);
  };
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    int k = lane + 32 * q;
    if (k < kext) {
      double xr = (k < nt) ? ldexp(v.yr[q], sx) : 0.0;
      double xi = (PAIR && k < nt) ? ldexp(v.yi[q], sx) : 0.0;
      int kc = k / kBK, kk = k % kBK;
      *wp(c, kc, kk) = -(beta * xr);
      if (!PAIR) {
        *wp(c, kc + p.nks, kk) = a * xr;
      } else {
        *wp(c + 1, kc, kk) = -(beta * xi);
        *wp(c, kc + p.nks, kk) = a * xr - b * xi;
        *wp(c + 1, kc + p.nks, kk) = b * xr + a * xi;
      }
    }
  }
}

template <int NQ>
__global__ void __launch_bounds__(512, 1) k_diag(DiagParams p) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int nt = p.nt;
  const int plen = nt * (nt + 3) / 2;
  double* Sp = reinterpret_cast<double*>(smraw);
  double* Tp = Sp + plen;
  double* cmS = Tp + plen;
  double* cmT = cmS + nt;
  signed char* fl = reinterpret_cast<signed char*>(cmT + nt);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // stage the diagonal tile (upper part + subdiagonal), column-major packed
  for (int j = warp; j < nt; j += nw) {
    int len = min(j + 2, nt);
    const double* sc = p.S + (long long)(p.t0 + j) * p.lds + p.t0;
    const double* tc = p.T + (long long)(p.t0 + j) * p.ldt + p.t0;
    for (int i = lane; i < len; i += 32) {
      Sp[poff(j) + i] = sc[i];
      Tp[poff(j) + i] = tc[i];
    }
  }
  for (int i = threadIdx.x; i < nt; i += blockDim.x) fl[i] = p.P.row_flag[p.t0 + i];
  __syncthreads();
  // in-tile column bounds above each block (reading R6)
  for (int j = threadIdx.x; j < nt; j += blockDim.x) {
    int top = (fl[j] == kRowBot2) ? j - 1 : j;
    double ms = 0.0, mt = 0.0;
    for (int i = 0; i < top; ++i) {
      ms = fmax(ms, fabs(Sp[poff(j) + i]));
      mt = fmax(mt, fabs(Tp[poff(j) + i]));
    }
    cmS[j] = ms;
    cmT[j] = mt;
  }
  __syncthreads();
  Tile tl;
  tl.Sp = Sp; tl.Tp = Tp; tl.cmS = cmS; tl.cmT = cmT; tl.fl = fl;
  for (int it = p.item_begin + blockIdx.x * nw + warp; it < p.n_items; it += gridDim.x * nw) {
    int c = p.P.item_col[it];
    int kind = p.P.col_kind[c];
    if (kind == kPairFirst) solve_item<NQ, true>(p, tl, c, lane);
    else solve_item<NQ, false>(p, tl, c, lane);
  }
}

size_t diag_smem_bytes(int nt) {
  size_t plen = (size_t)nt * (nt + 3) / 2;
  return (2 * plen + 2 * (size_t)nt) * sizeof(double) + (size_t)nt + 16;
}

static int g_num_sms = 0;

cudaError_t launch_diag(const DiagParams& p, cudaStream_t st) {
  if (p.n_items <= p.item_begin) return cudaSuccess;
  if (!g_num_sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  size_t smem = diag_smem_bytes(p.nt);
  int nq = (p.nt + 31) / 32;
  int threads = 512, nw = threads / 32;
  int items = p.n_items - p.item_begin;
  int grid = (items + nw - 1) / nw;
  if (grid > g_num_sms) grid = g_num_sms;
  cudaError_t err = cudaSuccess;
#define ZZ_DIAG_CASE(Q)                                                                        \
  case Q:                                                                                     \
    err = cudaFuncSetAttribute(k_diag<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (err != cudaSuccess) return err;                                                       \
    k_diag<Q><<<grid, threads, smem, st>>>(p);                                                \
    break;
  switch (nq) {
    ZZ_DIAG_CASE(1)
    ZZ_DIAG_CASE(2)
    ZZ_DIAG_CASE(3)
    ZZ_DIAG_CASE(4)
    ZZ_DIAG_CASE(5)
    default: return cudaErrorInvalidValue;
  }
#undef ZZ_DIAG_CASE
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// Consistency and normalisation (LAPACK normalisation, reading R11):
// e_c = min over the column's segments of e_seg; each segment is brought to e_c by an
// exact power of two, then the column (pair) is multiplied by 1/xmax, where xmax is
// max|x| (real) or max(|x|+|y|) (pair), formed as 2 max(|x|/2+|y|/2).
// ------------------------------------------------------------------------------------
__global__ void k_col_final(int n_sel, int M, DevPlan P, int* col_scale_exp, int* exp_tmp,
                            double* rec_tmp, int* stats) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_sel) return;
  int J = P.col_tile[c];
  int ec = 0;
  for (int I = 0; I <= J; ++I) ec = min(ec, P.e_seg[(long long)I * n_sel + c]);
  double h = 0.0;
  for (int I = 0; I <= J; ++I) {
    long long o = (long long)I * n_sel + c;
    h = fmax(h, ldexp(P.nrmh_seg[o], ec - P.e_seg[o]));
  }
  double rec = (h > 0.0) ? __ddiv_rn(0.5, h) : 1.0;
  exp_tmp[c] = ec;
  rec_tmp[c] = rec;
  // L_c of SURVEY.md s.8(c) O9: h is half the LAPACK measure (|x| or |x|+|y|) of the column
  // at exponent e_c, so log2(2h) - e_c is the log2 of the tip-normalised vector's maximum
  P.logmax[c] = (h > 0.0) ? log2(h) + 1.0 - (double)ec : -INFINITY;
  if (col_scale_exp) col_scale_exp[c] = ec;
  if (ec < 0) {
    atomicAdd(&stats[0], 1);
    atomicMin(&stats[1], ec);
  }
}

__global__ void k_apply_norm(int m, int n_sel, double* X, long long ldx, DevPlan P,
                             const int* __restrict__ exp_tmp, const double* __restrict__ rec_tmp) {
  int c = blockIdx.y;
  int r = P.col_r[c];
  int ec = exp_tmp[c];
  double rec = rec_tmp[c];
  double* xc = X + (long long)c * ldx;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    double v = 0.0;
    if (i <= r) {
      int I = P.row_tile[i];
      int k = ec - P.e_seg[(long long)I * n_sel + c];
      double x = xc[i];
      if (k != 0) x = ldexp(x, k);
      v = x * rec;
    }
    xc[i] = v;
  }
}

cudaError_t launch_normalize(int m, int n_sel, int M, double* X, long long ldx, int* col_scale_exp,
                             const DevPlan& P, int* exp_tmp, double* rec_tmp, cudaStream_t st) {
  if (n_sel <= 0 || m <= 0) return cudaSuccess;
  k_col_final<<<(n_sel + 127) / 128, 128, 0, st>>>(n_sel, M, P, col_scale_exp, exp_tmp, rec_tmp,
                                                   P.status + 4);
  int bx = (m + 1023) / 1024;
  if (bx > 8) bx = 8;
  dim3 grid(bx, n_sel);
  k_apply_norm<<<grid, 256, 0, st>>>(m, n_sel, X, ldx, P, exp_tmp, rec_tmp);
  return cudaGetLastError();
}

}  // namespace zz
