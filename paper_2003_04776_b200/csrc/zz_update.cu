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

namespace zz {

constexpr int kStages = 4;
constexpr int kCWarps = 4;                 // DMMA (consumer) warps
constexpr int kThreads = (kCWarps + 1) * 32;
constexpr int kABytes = kBM * kBK * 8;     // S or T chunk: [BM/8][BK][8] doubles
constexpr int kBBytes = kBN * kBK * 8;     // W chunk:      [BK/4][BN][4] doubles
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kSmemBytes = kStages * kStageBytes + 2 * kStages * 8 + kBN * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kCWarps * 32) : "memory");
}

// v1: one CTA per (n-tile, m-tile); C loads and stores guarded by branches.
__global__ void __launch_bounds__(kThreads, 2)
    k_update_v1(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmT, UpdParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  double* sA = reinterpret_cast<double*>(smem);
  double* sB = reinterpret_cast<double*>(smem + kStages * kABytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  unsigned long long* colmax = reinterpret_cast<unsigned long long*>(empty + kStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntile = p.ntile0 + blockIdx.x;
  const int n0 = ntile * kBN, m0 = blockIdx.y * kBM;
  const int nkc = 2 * p.nks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < kBN) colmax[threadIdx.x] = 0ull;
  __syncthreads();

  if (warp == kCWarps) {
    // ---------------- producer: TMA (S/T chunks) + bulk copy (W chunk) ----------------
    if (lane == 0) {
      const double* wt = p.W + (long long)ntile * nkc * (kBN * kBK);
      for (int kc = 0; kc < nkc; ++kc) {
        const int s = kc % kStages;
        if (kc >= kStages) mbar_wait(&empty[s], ((kc / kStages) - 1) & 1);
        mbar_expect_tx(&full[s], kStageBytes);
        const CUtensorMap* tm = (kc < p.nks) ? &tmS : &tmT;
        const int kcol = p.t0 + (kc % p.nks) * kBK;
        double* a = sA + s * (kBM * kBK);
#pragma unroll 4
        for (int mo = 0; mo < kBM / 8; ++mo) tma_load_2d(a + mo * (kBK * 8), tm, m0 + mo * 8, kcol, &full[s]);
        bulk_load(sB + s * (kBN * kBK), wt + (long long)kc * (kBN * kBK), kBBytes, &full[s]);
      }
    }
    return;
  }

  // ---------------- consumers: 4 warps, 2 (rows) x 2 (columns), 64 x 32 each ----------------
  const int wm = warp >> 1, wn = warp & 1;
  const int rq = lane & 3, cq = lane >> 2;
  double acc[4][8][2];
  // accumulators start from the scaled pending values: 2^sY[c] * Y (exact)
#pragma unroll
  for (int ni = 0; ni < 4; ++ni) {
    const int c = n0 + wn * 32 + ni * 8 + cq;
    const bool cvalid = (c >= p.c_begin) && (c < p.n_sel);
    const bool ld = cvalid && (c >= p.first_end);
    const int sy = ld ? p.sY[c] : 0;
    const double* xc = p.X + (long long)c * p.ldx;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int i0 = m0 + wm * 64 + mi * 8 + 2 * rq;
      double v0 = 0.0, v1 = 0.0;
      if (ld && i0 < p.rows) {
        if (p.vec && i0 + 1 < p.rows) {
          double2 t = *reinterpret_cast<const double2*>(xc + i0);
          v0 = t.x; v1 = t.y;
        } else {
          v0 = xc[i0];
          if (i0 + 1 < p.rows) v1 = xc[i0 + 1];
        }
        if (sy != 0) { v0 = ldexp(v0, sy); v1 = ldexp(v1, sy); }
      }
      acc[ni][mi][0] = v0;
      acc[ni][mi][1] = v1;
    }
  }

  for (int kc = 0; kc < nkc; ++kc) {
    const int s = kc % kStages;
    mbar_wait(&full[s], (kc / kStages) & 1);
    // release the previous stage only now (see k_update_t)
    if (lane == 0 && kc >= 1 && kc - 1 + kStages < nkc) mbar_arrive(&empty[(kc - 1) % kStages]);
    const double* a = sA + s * (kBM * kBK);
    const double* b = sB + s * (kBN * kBK);
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      double fw[4], fs[8];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) fw[ni] = b[(ks * kBN + wn * 32 + ni * 8 + cq) * 4 + rq];
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) fs[mi] = a[((wm * 8 + mi) * kBK + ks * 4 + rq) * 8 + cq];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) dmma(acc[ni][mi][0], acc[ni][mi][1], fw[ni], fs[mi]);
    }
    __syncwarp();
  }

  // ---------------- epilogue: store Y, per-column max over the next pending rows ----------------
#pragma unroll
  for (int ni = 0; ni < 4; ++ni) {
    const int c = n0 + wn * 32 + ni * 8 + cq;
    const bool cvalid = (c >= p.c_begin) && (c < p.n_sel);
    double* xc = p.X + (long long)c * p.ldx;
    double cm = 0.0;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int i0 = m0 + wm * 64 + mi * 8 + 2 * rq;
      const double v0 = acc[ni][mi][0], v1 = acc[ni][mi][1];
      if (cvalid && i0 < p.rows) {
        if (p.vec && i0 + 1 < p.rows) {
          *reinterpret_cast<double2*>(xc + i0) = make_double2(v0, v1);
        } else {
          xc[i0] = v0;
          if (i0 + 1 < p.rows) xc[i0 + 1] = v1;
        }
      }
      if (i0 < p.max_row) cm = fmax(cm, fabs(v0));
      if (i0 + 1 < p.max_row) cm = fmax(cm, fabs(v1));
    }
    cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, 1));
    cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, 2));
    if (rq == 0 && cvalid && cm > 0.0)
      atomicMax(&colmax[c - n0], (unsigned long long)__double_as_longlong(cm));
  }
  consumer_sync();
  if (threadIdx.x < kBN) {
    const int c = n0 + threadIdx.x;
    const unsigned long long v = colmax[threadIdx.x];
    if (v != 0ull && c >= p.c_begin && c < p.n_sel) atomicMax(&p.nY_out[c], v);
  }
}

// predicated global accesses (no branch around a load: every C load of a lane is issued
// before the first one is consumed)
__device__ __forceinline__ void ld2p(double& x, double& y, const double* p, bool pr) {
  asm("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q ld.global.v2.f64 {%0, %1}, [%2];\n}"
      : "+d"(x), "+d"(y) : "l"(p), "r"((int)pr));
}
__device__ __forceinline__ void ld1p(double& x, const double* p, bool pr) {
  asm("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q ld.global.f64 %0, [%1];\n}" : "+d"(x) : "l"(p), "r"((int)pr));
}
__device__ __forceinline__ void st2p(double* p, double x, double y, bool pr) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q st.global.v2.f64 [%0], {%1, %2};\n}"
               ::"l"(p), "d"(x), "d"(y), "r"((int)pr) : "memory");
}
__device__ __forceinline__ void st1p(double* p, double x, bool pr) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global.f64 [%0], %1;\n}"
               ::"l"(p), "d"(x), "r"((int)pr) : "memory");
}

// the same with an L2 eviction-priority policy (createpolicy): the C tiles stream through L2
// once per step (evict_first) while W is re-read by every m-tile of the step (evict_last)
__device__ __forceinline__ uint64_t l2_policy(bool last, bool on) {
  uint64_t pol;
  if (!on)
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  else if (last)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void ld2h(double& x, double& y, const double* p, bool pr, uint64_t pol) {
  asm("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %4;\n}"
      : "+d"(x), "+d"(y) : "l"(p), "r"((int)pr), "l"(pol));
}
__device__ __forceinline__ void st2h(double* p, double x, double y, bool pr, uint64_t pol) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %4;\n}"
               ::"l"(p), "d"(x), "d"(y), "r"((int)pr), "l"(pol) : "memory");
}
__device__ __forceinline__ void st1h(double* p, double x, bool pr, uint64_t pol) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global.L2::cache_hint.f64 [%0], %1, %3;\n}"
               ::"l"(p), "d"(x), "r"((int)pr), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_load_h(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void ld1p_i(int& x, const int* p, bool pr) {
  asm("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q ld.global.b32 %0, [%1];\n}" : "+r"(x) : "l"(p), "r"((int)pr));
}

// S/T panel of step I in fragment order: block (mt, kc) holds rows mt*128 .. +127 and the 16
// columns of chunk kc (S for kc < nks, T after), element (row 8g + c, column 4s + r) at
// ((g * 4 + s) * 8 + c) * 4 + r -- lane (c, r) of a DMMA B fragment reads consecutive doubles.
// Rows >= rows and columns >= nt are zero.  One CTA per block, staged through shared memory
// (coalesced column-major reads, contiguous writes).
__global__ void __launch_bounds__(256) k_pack(const double* __restrict__ S, long long lds, const double* __restrict__ T,
                                              long long ldt, int rows, int t0, int nt, int nks, double* __restrict__ Apk) {
  __shared__ double tile[16][129];
  const int mt = blockIdx.x, kc = blockIdx.y;
  const double* A = (kc < nks) ? S : T;
  const long long lda = (kc < nks) ? lds : ldt;
  const int c0 = (kc % nks) * kBK;
  for (int idx = threadIdx.x; idx < 16 * 128; idx += 256) {
    const int col = idx >> 7, r = idx & 127;
    const int gr = mt * kBM + r, gc = c0 + col;
    tile[col][r] = (gr < rows && gc < nt) ? A[(long long)(t0 + gc) * lda + gr] : 0.0;
  }
  __syncthreads();
  double* out = Apk + ((long long)mt * (2 * nks) + kc) * (kBM * kBK);
  for (int o = threadIdx.x; o < kBM * kBK; o += 256) {
    const int rr = o & 3, c = (o >> 2) & 7, sidx = (o >> 5) & 3, g = o >> 7;
    out[o] = tile[sidx * 4 + rr][g * 8 + c];
  }
}

size_t pack_bytes(int rows, int nks) { return (size_t)((rows + kBM - 1) / kBM) * 2 * nks * kBM * kBK * 8; }

cudaError_t launch_pack(const double* S, long long lds, const double* T, long long ldt, int rows, int t0, int nt,
                        int nks, double* Apk, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  dim3 grid((rows + kBM - 1) / kBM, 2 * nks);
  k_pack<<<grid, 256, 0, st>>>(S, lds, T, ldt, rows, t0, nt, nks, Apk);
  return cudaGetLastError();
}

// Persistent: each CTA walks the (m-tile, n-tile) grid with stride gridDim.x; the producer
// warp runs ahead into the next tile while the consumers finish the current epilogue.
// WN column warps x 2 row warps consume a 128 x (32 WN) tile; WN = 4 is one 288-thread CTA
// per SM sharing each S/T stage between 128 columns (half the A traffic of WN = 2).
template <int WN, int BOX = 8>
struct UT {
  static constexpr int BN = 32 * WN;
  static constexpr int CW = 2 * WN;                         // consumer warps
  static constexpr int THREADS = (CW + 1) * 32;
  static constexpr int BBYTES = BN * kBK * 8;               // W chunk: BN/64 blocks [BK/4][64][4]
  static constexpr int STAGE = kABytes + BBYTES;
  static constexpr int SMEM = kStages * STAGE + 2 * kStages * 8 + BN * 8;
  static constexpr int MINB = (WN == 2) ? 2 : 1;
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

template <int WN, int BOX, int MODE = 0>
__global__ void __launch_bounds__(UT<WN>::THREADS, UT<WN>::MINB)
    k_update_t(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmT, UpdParams p,
               int n_mtiles, int n_tiles) {
  using C = UT<WN, BOX>;
  extern __shared__ __align__(1024) unsigned char smem[];
  double* sA = reinterpret_cast<double*>(smem);
  double* sB = reinterpret_cast<double*>(smem + kStages * kABytes);
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
  const long long wtile = (long long)nkca * (kBN * kBK);


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
      const uint64_t pol_w = l2_policy(true, p.l2hint & 1);
      int g = 0;
      {
        const int tile = blockIdx.x;
        int mt, ntl;
        tile_coords(tile, n_mtiles, n_ntl, p.ngroup, mt, ntl);
        const int m0 = mbase + mt * kBM;
        const int nb64 = p.ntile0 + ntl * (C::BN / kBN);   // first 64-column block
        const int nblk = min(C::BN / kBN, p.ntile_end - nb64);         // 64-column blocks present
        for (int kc = 0; kc < nkc; ++kc, ++g) {
          const int s = g % kStages;
          if (g >= kStages) mbar_wait(&empty[s], ((g / kStages) - 1) & 1);
          mbar_expect_tx(&full[s], kABytes + nblk * kBBytes);
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
          double* a = sA + s * (kBM * kBK);
          if (BOX == 0) {
            // packed panel (k_pack): one 16 KB bulk copy per stage
            bulk_load(a, p.Apk + ((long long)(m0 / kBM) * nkc + kc) * (kBM * kBK), kABytes, &full[s]);
          } else {
            // S/T chunk as [BM/BOX][BK][BOX] (BOX = 4: conflict-free fragment loads)
#pragma unroll 4
            for (int mo = 0; mo < kBM / BOX; ++mo)
              tma_load_2d(a + mo * (kBK * BOX), tm, m0 + mo * BOX, kcol, &full[s]);
          }
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
  const uint64_t pol_c = l2_policy(false, p.l2hint & 2);
  const uint64_t pol_s = l2_policy(false, p.l2hint & 4);
  int g = 0;
  {
    const int tile = blockIdx.x;
    int mt, ntl;
    tile_coords(tile, n_mtiles, n_ntl, p.ngroup, mt, ntl);
    const int m0 = mbase + mt * kBM;
    const int n0 = (p.ntile0 + ntl * (C::BN / kBN)) * kBN;
    double acc[4][8][2];
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
      for (int mi = 0; mi < 8; ++mi) {
        const int i0 = m0 + wm * 64 + mi * 8 + 2 * rq;
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
        for (int mi = 0; mi < 8; ++mi) {
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
      const double* a = sA + s * (kBM * kBK);
      const double* b = bw + s * (C::BN * kBK);
#pragma unroll
      for (int ks = 0; ks < kBK / 4; ++ks) {
        double fw[4], fs[8];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) fw[ni] = b[(ks * kBN + wc + ni * 8 + cq) * 4 + rq];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) {
          if (BOX == 0) {
            fs[mi] = a[(((wm * 8 + mi) * 4 + ks) * 8 + cq) * 4 + rq];
          } else if (BOX == 8) {
            fs[mi] = a[((wm * 8 + mi) * kBK + ks * 4 + rq) * 8 + cq];
          } else {
            const int grp = wm * 16 + mi * 2 + (cq >> 2);
            fs[mi] = a[(grp * kBK + ks * 4 + rq) * 4 + (cq & 3)];
          }
        }
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int mi = 0; mi < 8; ++mi) dmma(acc[ni][mi][0], acc[ni][mi][1], fw[ni], fs[mi]);
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
      for (int mi = 0; mi < 8; ++mi) {
        const int i0 = m0 + wm * 64 + mi * 8 + 2 * rq;
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

static int g_upd_sms = 0;

int update_version() {
  static const int ver = getenv("ZZ_UPD") ? atoi(getenv("ZZ_UPD")) : 2;
  return ver;
}
int update_box_rows() { return update_version() == 3 ? 4 : 8; }
bool update_packs() { return update_version() == 5; }

template <int WN, int BOX, int MODE = 0>
static cudaError_t launch_t(const CUtensorMap* tmS, const CUtensorMap* tmT, UpdParams p, int n_mtiles, int n_ntiles64,
                            cudaStream_t st, int persist) {
  using C = UT<WN, BOX>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_update_t<WN, BOX, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_update_t<WN, BOX, MODE>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int per = C::BN / kBN;
  const int n_ntl = (n_ntiles64 + per - 1) / per;
  p.ntile_end = p.ntile0 + n_ntiles64;
  const int n_tiles = n_mtiles * n_ntl;
  const int grid = n_tiles;   // one tile per CTA (a persistent tile loop measured no faster)
  (void)persist;
  k_update_t<WN, BOX, MODE><<<grid, C::THREADS, C::SMEM, st>>>(*tmS, *tmT, p, n_mtiles, n_tiles);
  return cudaGetLastError();
}

static cudaError_t launch_update_impl(const CUtensorMap* tmS, const CUtensorMap* tmT, const UpdParams& p,
                                      int n_mtiles, int n_ntiles, cudaStream_t st, int ver, int persist);

cudaError_t launch_update(const CUtensorMap* tmS, const CUtensorMap* tmT, const UpdParams& p,
                          int n_mtiles, int n_ntiles, cudaStream_t st) {
  // ZZ_UPD: 2 (default) = 128 x 64 tiles, 2 CTAs per SM, batched predicated C loads;
  // 3 = the same with 4-row TMA boxes (conflict-free S/T fragment loads); 4 = 128 x 128
  // tiles with 8 consumer warps (1 CTA per SM); 1 = the first version (branchy C loads).
  // ZZ_UPD_PERSIST=k: k CTAs per SM walk the tiles.  (Variants are measured in profiles/.)
  const int ver = update_version();
  static const int persist = getenv("ZZ_UPD_PERSIST") ? atoi(getenv("ZZ_UPD_PERSIST")) : 0;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_update_v1, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_update_v1, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_upd_sms, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  if (n_mtiles <= 0 || n_ntiles <= 0) return cudaSuccess;
  // ZZ_L2HINT (bits): 1 = W evict_last, 2 = C loads evict_first, 4 = C stores evict_first
  static const int l2hint = getenv("ZZ_L2HINT") ? atoi(getenv("ZZ_L2HINT")) : 7;
  // ZZ_NGROUP: N tiles per CTA-order group (tile_coords; 0 = ungrouped)
  static const int ngroup = getenv("ZZ_NGROUP") ? atoi(getenv("ZZ_NGROUP")) : 64;
  UpdParams q = p;
  q.l2hint = l2hint;
  q.ngroup = ngroup;
  return launch_update_impl(tmS, tmT, q, n_mtiles, n_ntiles, st, ver, persist);
}

static cudaError_t launch_update_impl(const CUtensorMap* tmS, const CUtensorMap* tmT, const UpdParams& p,
                                      int n_mtiles, int n_ntiles, cudaStream_t st, int ver, int persist) {
  // the template kernels move C in 16-byte pairs: X 16-byte aligned with an even ldx
  if (ver == 2 && p.vec) {
    if (p.nxs > 0 && p.row_lo > 0) return launch_t<2, 8, 3>(tmS, tmT, p, n_mtiles, n_ntiles, st, persist);
    if (p.nxs > 0) return launch_t<2, 8, 1>(tmS, tmT, p, n_mtiles, n_ntiles, st, persist);
    if (p.row_lo > 0) return launch_t<2, 8, 2>(tmS, tmT, p, n_mtiles, n_ntiles, st, persist);
    return launch_t<2, 8>(tmS, tmT, p, n_mtiles, n_ntiles, st, persist);
  }
  if (ver == 3 && p.vec) return launch_t<2, 4>(tmS, tmT, p, n_mtiles, n_ntiles, st, persist);
  if (ver == 4 && p.vec) return launch_t<4, 8>(tmS, tmT, p, n_mtiles, n_ntiles, st, persist);
  if (ver == 5 && p.vec && p.Apk) return launch_t<2, 0>(tmS, tmT, p, n_mtiles, n_ntiles, st, persist);
  dim3 g1(n_ntiles, n_mtiles);
  k_update_v1<<<g1, kThreads, kSmemBytes, st>>>(*tmS, *tmT, p);
  return cudaGetLastError();
}

}  // namespace zz
