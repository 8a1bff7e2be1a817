// zz_back.cu -- back-transformation W = V X of the eigenvectors (xTGEVC HOWMNY='B'; PAPER.md:28-32
// with SURVEY.md reading A1: S = U^T A V, T = U^T B V, S z = lambda T z gives A (V z) =
// lambda B (V z)), followed by LAPACK's normalisation of the back-transformed vectors:
// max_i |w_i| = 1 for a real column, max_i (|Re w_i| + |Im w_i|) = 1 for a complex pair.
//
// B200 design.  X is block-upper-triangular (column c is zero below its last row r_c, and
// the columns are in block order, so r_c is non-decreasing): W(:, J) = V(:, 0:K_J) X(0:K_J, J)
// for every 64-column tile J with K_J = 1 + max r_c over the tile -- about m^3 flop for all
// eigenvectors instead of the 2 m^3 of a dense product.  One FP64 tensor-core contraction
// (DMMA.8x8x4, mma.sync.m8n8k4.f64; sm_100a has no FP64 tcgen05 kind) with the pipeline of
// the robust update (zz_update.cu): CTA tile 128 rows x 64 columns, two CTAs per SM, one
// producer warp feeding a 4-stage mbarrier ring -- V by TMA (16 boxes of 8 rows x 16
// columns per chunk), X by one 8 KB bulk copy per chunk from a tile-packed copy
// [tile][chunk][4][64][4] written by k_back_pack -- and four DMMA warps (64 x 32 each)
// computing W^T = X^T V^T, so a lane holds two consecutive rows of one column of W (16-byte
// stores).  The K loop of a tile runs over its own K_J chunks only; tiles with the longest K
// are scheduled first.  The epilogue writes W and the per-column max |w| (atomicMax on the
// double's bits: exact, order-independent), which normalises the real columns directly;
// pairs take their |Re| + |Im| maximum in the normalisation pass.
#include <cuda.h>
#include <stdint.h>

#include "zz_internal.cuh"
#include "zz_pipe.cuh"

namespace zz {

namespace {

constexpr int kBkStages = 4;
constexpr int kBkA = kBM * kBK * 8;       // V chunk [BM/8][BK][8]
constexpr int kBkB = kBN * kBK * 8;       // X chunk [BK/4][BN][4]
constexpr int kBkThreads = 5 * 32;        // 4 DMMA warps + 1 producer warp
constexpr int kBkSmem = kBkStages * (kBkA + kBkB) + 2 * kBkStages * 8 + kBN * 8;
constexpr int kBkGroup = 64;              // N tiles per group of the CTA order

// X (m x n_sel, ldx) -> [tile J][chunk kc < nkc[J]][BK/4][64][4]: element (row r, column c) of
// tile J at woff[J] + (r / 16) * 1024 + ((r % 16) / 4) * 256 + (c % 64) * 4 + (r % 4); zeros
// past m and n_sel.  One CTA per (chunk, tile): 8 KB out, contiguous.
__global__ void __launch_bounds__(256) k_back_pack(const double* __restrict__ X, long long ldx, int m, int n_sel,
                                                   const int* __restrict__ nkc, const long long* __restrict__ woff,
                                                   double* __restrict__ Xp) {
  const int J = blockIdx.y, kc = blockIdx.x;
  if (kc >= nkc[J]) return;
  double* out = Xp + woff[J] + (long long)kc * (kBN * kBK);
  for (int o = threadIdx.x; o < kBN * kBK; o += blockDim.x) {
    const int rr = o & 3, col = (o >> 2) & 63, kq = o >> 8;
    const int r = kc * kBK + kq * 4 + rr, c = J * kBN + col;
    out[o] = (r < m && c < n_sel) ? X[(long long)c * ldx + r] : 0.0;
  }
}

__global__ void __launch_bounds__(kBkThreads, 2)
    k_back_gemm(const __grid_constant__ CUtensorMap tmV, const double* __restrict__ Xp, const int* __restrict__ nkc,
                const long long* __restrict__ woff, int m, int n_sel, int n_mtiles, int n_ntiles, double* __restrict__ W,
                long long ldw, unsigned long long* __restrict__ colmax_out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  double* sA = reinterpret_cast<double*>(smem);
  double* sB = reinterpret_cast<double*>(smem + kBkStages * kBkA);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBkStages * (kBkA + kBkB));
  uint64_t* empty = full + kBkStages;
  unsigned long long* colmax = reinterpret_cast<unsigned long long*>(empty + kBkStages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CTA order: groups of kBkGroup N tiles, the longest-K tiles (highest J) first; inside a
  // group the M tiles are the slow index (consecutive CTAs share a V panel in L2)
  int mt, jt;
  {
    const int tile = blockIdx.x;
    const int per = n_mtiles * kBkGroup;
    const int g = tile / per, loc = tile - g * per;
    const int gs = min(kBkGroup, n_ntiles - g * kBkGroup);
    mt = loc / gs;
    jt = n_ntiles - 1 - (g * kBkGroup + loc % gs);
  }
  const int nk = nkc[jt];
  const int m0 = mt * kBM, n0 = jt * kBN;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBkStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < kBN) colmax[threadIdx.x] = 0ull;
  __syncthreads();
  if (warp == 4) {
    // ---------------- producer: TMA (V chunk) + bulk copy (X chunk) ----------------
    if (lane == 0) {
      const uint64_t pol_x = l2_policy(true);
      const double* xt = Xp + woff[jt];
      for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % kBkStages;
        if (kc >= kBkStages) mbar_wait(&empty[s], ((kc / kBkStages) - 1) & 1);
        mbar_expect_tx(&full[s], kBkA + kBkB);
        double* a = sA + s * (kBM * kBK);
#pragma unroll 4
        for (int mo = 0; mo < kBM / 8; ++mo) tma_load_2d(a + mo * (kBK * 8), &tmV, m0 + mo * 8, kc * kBK, &full[s]);
        bulk_load_h(sB + s * (kBN * kBK), xt + (long long)kc * (kBN * kBK), kBkB, &full[s], pol_x);
      }
    }
    return;
  }
  // ---------------- consumers: 2 (rows) x 2 (columns) warps, 64 x 32 each ----------------
  const int wm = warp >> 1, wn = warp & 1;
  const int rq = lane & 3, cq = lane >> 2;
  const uint64_t pol_c = l2_policy(false);
  double acc[4][8][2];
#pragma unroll
  for (int ni = 0; ni < 4; ++ni)
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) acc[ni][mi][0] = acc[ni][mi][1] = 0.0;
  const int wc = wn * 32;
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc % kBkStages;
    mbar_wait(&full[s], (kc / kBkStages) & 1);
    // the previous stage is released only now (see k_update_t: an arrive scheduled among
    // the DMMAs of its own chunk could let a refill race the last fragment loads)
    if (lane == 0 && kc >= 1 && kc - 1 + kBkStages < nk) mbar_arrive(&empty[(kc - 1) % kBkStages]);
    const double* a = sA + s * (kBM * kBK);
    const double* b = sB + s * (kBN * kBK);
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      double fw[4], fs[8];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) fw[ni] = b[(ks * kBN + wc + ni * 8 + cq) * 4 + rq];
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) fs[mi] = a[((wm * 8 + mi) * kBK + ks * 4 + rq) * 8 + cq];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) dmma(acc[ni][mi][0], acc[ni][mi][1], fw[ni], fs[mi]);
    }
    __syncwarp();
  }
  // ---------------- epilogue: store W, per-column max |w| ----------------
#pragma unroll
  for (int ni = 0; ni < 4; ++ni) {
    const int c = n0 + wc + ni * 8 + cq;
    const bool cvalid = c < n_sel;
    double* wcol = W + (long long)(cvalid ? c : 0) * ldw;
    double cm = 0.0;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int i0 = m0 + wm * 64 + mi * 8 + 2 * rq;
      const double v0 = acc[ni][mi][0], v1 = acc[ni][mi][1];
      st2h(wcol + i0, v0, v1, cvalid && i0 + 1 < m, pol_c);
      st1h(wcol + i0, v0, cvalid && i0 + 1 == m, pol_c);
      if (i0 < m) cm = fmax(cm, fabs(v0));
      if (i0 + 1 < m) cm = fmax(cm, fabs(v1));
    }
    cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, 1));
    cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, 2));
    if (rq == 0 && cvalid && cm > 0.0) atomicMax(&colmax[c - n0], (unsigned long long)__double_as_longlong(cm));
  }
  asm volatile("bar.sync 1, %0;" ::"n"(4 * 32) : "memory");
  if (threadIdx.x < kBN) {
    const int c = n0 + threadIdx.x;
    const unsigned long long v = colmax[threadIdx.x];
    if (v != 0ull && c < n_sel) atomicMax(&colmax_out[c], v);
  }
}

constexpr int kNormThreads = 256;

// LAPACK's normalisation: a real column by 1/max|w| (from the GEMM epilogue), a pair by
// 1/max(|Re| + |Im|) (one CTA per pair reads both columns); one multiply per entry.  The CTA
// of a pair's second column returns at once.
__global__ void __launch_bounds__(kNormThreads) k_back_norm(double* __restrict__ W, long long ldw, int m,
                                                            const int* __restrict__ col_kind,
                                                            const unsigned long long* __restrict__ colmax) {
  const int c = blockIdx.x;
  const int kind = col_kind[c];
  if (kind == kPairSecond) return;
  const bool pair = kind == kPairFirst;
  double* w0 = W + (long long)c * ldw;
  double* w1 = pair ? w0 + ldw : w0;
  __shared__ double red[kNormThreads / 32];
  double mx;
  if (!pair) {
    mx = __longlong_as_double((long long)colmax[c]);
  } else {
    mx = 0.0;
    for (int i = threadIdx.x; i < m; i += kNormThreads) mx = fmax(mx, fabs(w0[i]) + fabs(w1[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
      mx = threadIdx.x < kNormThreads / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (threadIdx.x == 0) red[0] = mx;
    }
    __syncthreads();
    mx = red[0];
  }
  if (!(mx > 0.0)) return;           // a zero column (V singular) stays zero
  const double r = 1.0 / mx;
  for (int i = threadIdx.x; i < m; i += kNormThreads) {
    w0[i] *= r;
    if (pair) w1[i] *= r;
  }
}

}  // namespace

size_t back_pack_doubles(const int* nkc_host, int n_ntiles) {
  size_t t = 0;
  for (int J = 0; J < n_ntiles; ++J) t += (size_t)nkc_host[J] * (kBN * kBK);
  return t;
}

cudaError_t launch_back_gemm(const CUtensorMap* tmV, const double* X, long long ldx, int m, int n_sel,
                             const int* nkc, const long long* woff, int max_nkc, double* Xp, double* W,
                             long long ldw, unsigned long long* colmax, cudaStream_t st) {
  if (m <= 0 || n_sel <= 0) return cudaSuccess;
  const int n_ntiles = (n_sel + kBN - 1) / kBN, n_mtiles = (m + kBM - 1) / kBM;
  k_back_pack<<<dim3(max_nkc, n_ntiles), 256, 0, st>>>(X, ldx, m, n_sel, nkc, woff, Xp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(k_back_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, kBkSmem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_back_gemm, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_back_gemm<<<n_mtiles * n_ntiles, kBkThreads, kBkSmem, st>>>(*tmV, Xp, nkc, woff, m, n_sel, n_mtiles, n_ntiles, W,
                                                                  ldw, colmax);
  return cudaGetLastError();
}

cudaError_t launch_back_norm(double* W, long long ldw, int m, int n_sel, const int* col_kind,
                             const unsigned long long* colmax, cudaStream_t st) {
  if (n_sel <= 0 || m <= 0) return cudaSuccess;
  k_back_norm<<<n_sel, kNormThreads, 0, st>>>(W, ldw, m, col_kind, colmax);
  return cudaGetLastError();
}

}  // namespace zz
