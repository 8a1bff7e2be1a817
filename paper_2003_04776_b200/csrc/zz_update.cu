// zz_update.cu -- the robust update (Kernel 2 of PAPER.md:153-157, Alg. 1 line P:140) as
// one fused FP64 contraction per wavefront step I (the composition of PAPER.md:235):
//
//   Y[0:ts_I, c] <- 2^sY[c] Y[0:ts_I, c] + [S(0:ts_I, tile I) | T(0:ts_I, tile I)] W[:, c]
//   W = [-2^sX X_I D ; 2^sX X_I B]    (formed by the diagonal solve, zz_kernels.cu)
//
// with the per-column exponents sY/sX chosen by ProtectUpdate (Algs. 2 and 3,
// PAPER.md:216-262), and an epilogue that writes the new max|Y| per column (the norm the
// next step's scaling decision needs).
//
// B200 design: FP64 has no tcgen05 kind on sm_100a; the tensor path is DMMA.8x8x4
// (mma.sync.m8n8k4.f64), measured at 37.0 TFLOP/s = the DFMA peak (profiles/).  The CTA
// tile is 128 rows x 64 columns, K is consumed in chunks of 16 through a 4-stage
// TMA / bulk-copy pipeline with mbarriers; one producer warp, four DMMA warps (64 x 32
// each).  The contraction is computed transposed (C^T = W^T S^T) so that each lane's two
// accumulators are two consecutive rows of a column of X: 16-byte loads/stores of C.
#include <cuda.h>
#include <stdint.h>
#include <stdlib.h>

#include "zz_internal.cuh"
#include "zz_pipe.cuh"

namespace zz {

constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK * 8;     // S or T chunk: [BM/8][BK][8] doubles
constexpr int kBBytes = kBN * kBK * 8;     // W chunk:      [BK/4][BN][4] doubles
constexpr int kNGroup = 64;                // N tiles per group of the CTA order (tile_coords)

// 2 (rows) x 2 (columns) consumer warps of 64 x 32 consume a 128 x 64 tile; one producer warp.
// BMC = 64 / 32: half / quarter tiles (warps of 32 / 16 rows x 32) for launches with fewer
// CTAs than SMs (thin band updates, small steps): more CTAs, each at the full DMMA rate of its
// SM, and the same DMMA sequence per accumulator, so bitwise the same result.
template <int BMC = kBM>
struct UT {
  static constexpr int BN = 64;
  static constexpr int CW = 4;                              // consumer warps
  static constexpr int MI = BMC / 16;                       // 8-row blocks per consumer warp
  static constexpr int THREADS = (CW + 1) * 32;
  static constexpr int ABYTES = BMC * kBK * 8;
  static constexpr int BBYTES = BN * kBK * 8;
  static constexpr int STAGE = ABYTES + BBYTES;
  static constexpr int SMEM = kStages * STAGE + 2 * kStages * 8 + BN * 8;
};

// CTA order: groups of `ng` N tiles; inside a group the M tiles are the slow index and the
// group's N tiles the fast one.  Consecutive CTAs share one S/T panel block (A reuse in L2)
// while the group's W columns stay in L2 for the sweep over all M tiles (with three
// segments W no longer fits L2 whole: the ungrouped order re-read it from DRAM per M tile).
// ng <= 0: one group (M-major over all N tiles).
__device__ __forceinline__ void tile_coords(int tile, int n_mtiles, int n_ntl, int ng, int& mt, int& ntl) {
  if (ng <= 0 || ng >= n_ntl) {
    mt = tile / n_ntl;
    ntl = tile % n_ntl;
    return;
  }
  const int per = n_mtiles * ng;          // CTAs of a full group
  const int g = tile / per, loc = tile - g * per;
  const int gs = min(ng, n_ntl - g * ng);  // N tiles in this group (the last may be short)
  mt = loc / gs;
  ntl = g * ng + loc % gs;
}

template <int MODE = 0, int BMC = kBM>
__global__ void __launch_bounds__(UT<BMC>::THREADS, 2)
    k_update_t(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmT, UpdParams p,
               int n_mtiles, int n_tiles) {
  using C = UT<BMC>;
  constexpr int WN = 2;
  extern __shared__ __align__(1024) unsigned char smem[];
  double* sA = reinterpret_cast<double*>(smem);
  double* sB = reinterpret_cast<double*>(smem + kStages * C::ABYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * C::STAGE);
  uint64_t* empty = full + kStages;
  unsigned long long* colmax = reinterpret_cast<unsigned long long*>(empty + kStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // MODE 1 (two-step fused update): a second K segment; MODE 2 (thin update): first row row_lo
  constexpr bool SEG2 = MODE == 1 || MODE == 3;   // MODE 3: segments and a first row (lookahead band)
  // K chunks: segment 0 (t0, nks, W), then the group's further segments (MODE 1)
  const int nkca = 2 * p.nks;
  int nkc = nkca;
  if (SEG2) {
#pragma unroll
    for (int e = 0; e < kMaxGroup - 1; ++e) nkc += (e < p.nxs) ? 2 * p.xnks[e] : 0;
  }
  const int n_ntl = n_tiles / n_mtiles;
  const int row_lo = (MODE >= 2) ? p.row_lo : 0;   // MODE 3: the lookahead's band part
  const int mbase = row_lo & ~1;                         // 16-byte aligned first row pair
  // W is stored per 64-column block: [ntile64][kc][BK/4][64][4] (per segment)


  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < C::BN) colmax[threadIdx.x] = 0ull;
  __syncthreads();

  if (warp == C::CW) {
    // ---------------- producer: TMA (S/T chunks) + bulk copies (W chunk) ----------------
    if (lane == 0) {
      const uint64_t pol_w = l2_policy(true);
      int g = 0;
      {
        const int tile = blockIdx.x;
        int mt, ntl;
        tile_coords(tile, n_mtiles, n_ntl, kNGroup, mt, ntl);
        const int m0 = mbase + mt * BMC;
        const int nb64 = p.ntile0 + ntl * (C::BN / kBN);   // first 64-column block
        const int nblk = min(C::BN / kBN, p.ntile_end - nb64);         // 64-column blocks present
        for (int kc = 0; kc < nkc; ++kc, ++g) {
          const int s = g % kStages;
          if (g >= kStages) mbar_wait(&empty[s], ((g / kStages) - 1) & 1);
          mbar_expect_tx(&full[s], C::ABYTES + nblk * kBBytes);
          // segment of chunk kc (static indices: the parameter arrays stay in constant space)
          int kl = kc, nks_s = p.nks, t0_s = p.t0;
          const double* w_s = p.W;
          if (SEG2 && kc >= nkca) {
            int base = nkca;
            bool found = false;
#pragma unroll
            for (int e = 0; e < kMaxGroup - 1; ++e) {
              const int n2 = (e < p.nxs) ? 2 * p.xnks[e] : 0;
              if (!found && kc < base + n2) {
                found = true;
                kl = kc - base;
                nks_s = p.xnks[e];
                t0_s = p.xt0[e];
                w_s = p.xW[e];
              }
              base += n2;
            }
          }
          const CUtensorMap* tm = (kl < nks_s) ? &tmS : &tmT;
          const int kcol = t0_s + (kl % nks_s) * kBK;
          double* a = sA + s * (BMC * kBK);
          // S/T chunk as [BM/8][BK][8]: 16 (8) TMA boxes of 8 rows x 16 columns
#pragma unroll 4
          for (int mo = 0; mo < BMC / 8; ++mo) tma_load_2d(a + mo * (kBK * 8), tm, m0 + mo * 8, kcol, &full[s]);
          for (int q = 0; q < nblk; ++q)
            bulk_load_h(sB + s * (C::BN * kBK) + q * (kBN * kBK),
                        w_s + (long long)(nb64 + q) * ((long long)(2 * nks_s) * (kBN * kBK)) +
                            (long long)kl * (kBN * kBK),
                        kBBytes, &full[s], pol_w);
        }
      }
    }
    return;
  }

  // ---------------- consumers: 2 (rows) x WN (columns) warps, 64 x 32 each ----------------
  const int wm = warp / WN, wn = warp % WN;
  const int rq = lane & 3, cq = lane >> 2;
  const uint64_t pol_c = l2_policy(false);
  const uint64_t pol_s = pol_c;
  int g = 0;
  {
    const int tile = blockIdx.x;
    int mt, ntl;
    tile_coords(tile, n_mtiles, n_ntl, kNGroup, mt, ntl);
    const int m0 = mbase + mt * BMC;
    const int n0 = (p.ntile0 + ntl * (C::BN / kBN)) * kBN;
    constexpr int MI = C::MI;
    double acc[4][MI][2];
    // accumulators start from the scaled pending values 2^sY[c] Y (exact): all loads first
    int sy[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int c = n0 + wn * 32 + ni * 8 + cq;
      const bool ld = (c >= p.c_begin) && (c < p.n_sel) && (c >= p.first_end);
      sy[ni] = 0;
      ld1p_i(sy[ni], p.sY + (ld ? c : 0), ld);
      const double* xc = p.X + (long long)(ld ? c : 0) * p.ldx;
      // one 16-byte load per row pair (X is 16-byte aligned with an even ldx on this path),
      // all issued before any is consumed
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const int i0 = m0 + wm * (BMC / 2) + mi * 8 + 2 * rq;
        acc[ni][mi][0] = 0.0;
        acc[ni][mi][1] = 0.0;
        // a pair straddling the last row is loaded whole (row p.rows exists: p.rows < m <=
        // ldx); that accumulator row is never stored nor counted in the column maximum
        ld2h(acc[ni][mi][0], acc[ni][mi][1], xc + i0, ld && (i0 < p.rows) && (i0 + 1 >= row_lo), pol_c);
      }
    }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      if (sy[ni] != 0) {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          acc[ni][mi][0] = ldexp(acc[ni][mi][0], sy[ni]);
          acc[ni][mi][1] = ldexp(acc[ni][mi][1], sy[ni]);
        }
      }
    }
    const double* bw = sB + (wn >> 1) * (kBN * kBK);   // this warp's 64-column block of W
    const int wc = (wn & 1) * 32;
    for (int kc = 0; kc < nkc; ++kc, ++g) {
      const int s = g % kStages;
      mbar_wait(&full[s], (g / kStages) & 1);
      // Release the previous stage only now, not at the end of its own iteration: ptxas may
      // schedule an mbarrier arrive above the DMMAs of the chunk, i.e. while the last shared-
      // memory fragment loads are still in flight, and a fast TMA refill of that stage then
      // races them (observed as run-to-run differences of whole 8-row boxes with K > 16
      // chunks).  Every DMMA of chunk kc-1 has issued -- its fragments have landed -- before
      // this point.  (The last kStages chunks have no refill to release.)
      if (lane == 0 && kc >= 1 && kc - 1 + kStages < nkc) mbar_arrive(&empty[(g - 1) % kStages]);
      const double* a = sA + s * (BMC * kBK);
      const double* b = bw + s * (C::BN * kBK);
#pragma unroll
      for (int ks = 0; ks < kBK / 4; ++ks) {
        double fw[4], fs[MI];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) fw[ni] = b[(ks * kBN + wc + ni * 8 + cq) * 4 + rq];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) fs[mi] = a[((wm * MI + mi) * kBK + ks * 4 + rq) * 8 + cq];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) dmma(acc[ni][mi][0], acc[ni][mi][1], fw[ni], fs[mi]);
      }
      __syncwarp();
    }

    // ---------------- epilogue: store Y, per-column max over the next pending rows ----------------
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int c = n0 + wn * 32 + ni * 8 + cq;
      const bool cvalid = (c >= p.c_begin) && (c < p.n_sel);
      double* xc = p.X + (long long)(cvalid ? c : 0) * p.ldx;
      double cm = 0.0;
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const int i0 = m0 + wm * (BMC / 2) + mi * 8 + 2 * rq;
        const double v0 = acc[ni][mi][0], v1 = acc[ni][mi][1];
        // rows [row_lo, rows) only: a pair may straddle either end
        const bool both = cvalid && (i0 + 1 < p.rows) && (i0 >= row_lo);
        st2h(xc + i0, v0, v1, both, pol_s);
        st1h(xc + i0, v0, cvalid && i0 + 1 == p.rows && i0 >= row_lo, pol_s);
        if (MODE >= 2) st1h(xc + i0 + 1, v1, cvalid && i0 + 1 == row_lo && i0 + 1 < p.rows, pol_s);
        if (i0 < p.max_row) cm = fmax(cm, fabs(v0));
        if (i0 + 1 < p.max_row) cm = fmax(cm, fabs(v1));
      }
      cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, 1));
      cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, 2));
      if (rq == 0 && cvalid && cm > 0.0)
        atomicMax(&colmax[c - n0], (unsigned long long)__double_as_longlong(cm));
    }
    asm volatile("bar.sync 1, %0;" ::"n"(C::CW * 32) : "memory");
    if (threadIdx.x < C::BN) {
      const int c = n0 + threadIdx.x;
      const unsigned long long v = colmax[threadIdx.x];
      if (v != 0ull && c >= p.c_begin && c < p.n_sel) atomicMax(&p.nY_out[c], v);
      colmax[threadIdx.x] = 0ull;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(C::CW * 32) : "memory");
  }
}


static int g_sms_u = 0;

template <int MODE, int BMC>
static cudaError_t launch_tt(const CUtensorMap* tmS, const CUtensorMap* tmT, UpdParams p, int n_mtiles, int n_ntiles64,
                             cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_update_t<MODE, BMC>, cudaFuncAttributeMaxDynamicSharedMemorySize, UT<BMC>::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_update_t<MODE, BMC>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  p.ntile_end = p.ntile0 + n_ntiles64;
  const int n_tiles = n_mtiles * n_ntiles64;   // one (m-tile, n-tile) per CTA
  k_update_t<MODE, BMC><<<n_tiles, UT<BMC>::THREADS, UT<BMC>::SMEM, st>>>(*tmS, *tmT, p, n_mtiles, n_tiles);
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_t(const CUtensorMap* tmS, const CUtensorMap* tmT, UpdParams p, int n_mtiles, int n_ntiles64,
                            cudaStream_t st) {
  if (!g_sms_u) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms_u, cudaDevAttrMultiProcessorCount, dev);
  }
  if (n_mtiles * n_ntiles64 < g_sms_u) {
    // fewer CTAs than SMs: half (quarter) tiles, twice (four times) the CTAs
    const int mbase = ((MODE >= 2) ? p.row_lo : 0) & ~1;
    const int n_m64 = (p.rows - mbase + 63) / 64;
    if (n_m64 * n_ntiles64 < g_sms_u) return launch_tt<MODE, 32>(tmS, tmT, p, (p.rows - mbase + 31) / 32, n_ntiles64, st);
    return launch_tt<MODE, 64>(tmS, tmT, p, n_m64, n_ntiles64, st);
  }
  return launch_tt<MODE, kBM>(tmS, tmT, p, n_mtiles, n_ntiles64, st);
}

// MODE 0: one step; 1: a step group's update (further K segments); 2: thin update of a band
// (first row row_lo); 3: segments and a first row (the lookahead's band part).  X must be
// 16-byte aligned with an even ldx (zz_api.cu solves any other X in an aligned workspace).
cudaError_t launch_update(const CUtensorMap* tmS, const CUtensorMap* tmT, const UpdParams& p,
                          int n_mtiles, int n_ntiles, cudaStream_t st) {
  if (n_mtiles <= 0 || n_ntiles <= 0) return cudaSuccess;
  if (!p.vec) return cudaErrorInvalidValue;
  if (p.nxs > 0 && p.row_lo > 0) return launch_t<3>(tmS, tmT, p, n_mtiles, n_ntiles, st);
  if (p.nxs > 0) return launch_t<1>(tmS, tmT, p, n_mtiles, n_ntiles, st);
  if (p.row_lo > 0) return launch_t<2>(tmS, tmT, p, n_mtiles, n_ntiles, st);
  return launch_t<0>(tmS, tmT, p, n_mtiles, n_ntiles, st);
}

}  // namespace zz
