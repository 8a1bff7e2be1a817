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
__device__ __noinline__ double scale2_slow3(double x, int k) {
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
  double2* bn;     // per block b: (||S_bb||_inf, ||T_bb||_inf) of the block's diagonal sub-block
  int* bs;         // block b = rows [bs[b], bs[b+1]); bs[b] = 8b - (row 8b is a 2x2 bottom)
  unsigned char* teams;   // per team of warps: team_bytes(W, nblk) (see Team)
  double* ptab;           // per warp: pivot table (G stage 1; the substitution's prepared pivots)
  unsigned char* gring;   // one warp per task: the G producers' ring (GRing), else unused
  signed char* fl; // row flags
};

// One solved block as its owner warp publishes it to the other warps of its team.
struct Pub {
  double x[72];        // [9 slots][8 columns]: the block's rows (the owner's slab), after all
                       // of the block's scalings
  double bound[8];     // per column: running bound of the pending rows after the block
  int kseg[8], eu[8];  // per column: the block's two segment scalings (in this order)
  int ex[8];           // per column: exponent of the segment after the block (relative to e_pend)
  int flag;            // 2 gen: published; 2 gen - 1: the owner asks for the pending maximum
  int cnt;             // warps that answered the request
  int pad[2];
};
static_assert(sizeof(Pub) % 16 == 0, "Pub alignment");

// Per team: the publication records (one per block; W = 1: one, the warp's slab), the
// prepared pivots of the slow path (only the warp solving the current block uses them) and
// two reduction areas (initial bound; segment norms).
__host__ __device__ __forceinline__ size_t team_bytes(int W, int nblk) {
  return sizeof(Pub) * (size_t)(W == 1 ? 1 : nblk) + sizeof(double) * 8 * (size_t)W +
         sizeof(double) * 16 * (size_t)W + sizeof(double) * 8 * (size_t)W;
}
constexpr size_t kPtabBytes = sizeof(double) * 576;   // per warp: pivot table [9][8][8]

__host__ __device__ __forceinline__ size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ __forceinline__ size_t gring_bytes() { return 4 * 5632 + 64; }   // kGSlots x kGSlotBytes + flags
__host__ __device__ __forceinline__ size_t smem3(int nt, int nteams, size_t tb, int nwarps) {
  return a16(sizeof(double2) * (size_t)(nt * (nt + 3) / 2 + kPad3)) + a16(sizeof(double2) * (size_t)nt) +
         a16(sizeof(double2) * 17) + a16(sizeof(double2) * 17) + a16(sizeof(int) * 18) + a16(tb) * nteams +
         kPtabBytes * nwarps + (nteams == nwarps ? gring_bytes() : 0) + a16((size_t)nt);
}
__device__ __forceinline__ Sm3 carve3(unsigned char* base, int nt, int nteams, size_t tb, int nwarps) {
  Sm3 s;
  size_t o = 0;
  s.ST = reinterpret_cast<double2*>(base + o); o += a16(sizeof(double2) * (size_t)(nt * (nt + 3) / 2 + kPad3));
  s.cm = reinterpret_cast<double2*>(base + o); o += a16(sizeof(double2) * (size_t)nt);
  s.tau = reinterpret_cast<double2*>(base + o); o += a16(sizeof(double2) * 17);
  s.bn = reinterpret_cast<double2*>(base + o); o += a16(sizeof(double2) * 17);
  s.bs = reinterpret_cast<int*>(base + o); o += a16(sizeof(int) * 18);
  s.teams = base + o; o += a16(tb) * nteams;
  s.ptab = reinterpret_cast<double*>(base + o); o += kPtabBytes * nwarps;
  s.gring = base + o; o += (nteams == nwarps ? gring_bytes() : 0);
  s.fl = reinterpret_cast<signed char*>(base + o);
  return s;
}

// A team: W warps solving one task together (warp w owns a contiguous range of blocks).
struct Team {
  int W, w;        // team size, this warp's index in it
  int bar;         // named barrier of the team (W > 1)
  int gen;         // task + 1: the generation of the publication flags
  Pub* pub;
  double* pslab;   // this warp's pivot table [9][8][8]
  double* red0;    // [W][8] initial bound
  double* red1;    // [W][8][2] segment norms
  double* red2;    // [W][8] pending maxima (answers to an owner's request)
};

#ifdef ZZ_VARIANT_TRACE
__device__ long long g_trace[512];
#define ZZ_TR(i) do { if (blockIdx.x == 0 && tm.gen == 1 && lane == 0) g_trace[(i)] = clock64(); } while (0)
#define ZZ_TR0() do { if (blockIdx.x == 0 && threadIdx.x == 0) g_trace[180] = clock64(); } while (0)
#else
#define ZZ_TR(i) do { } while (0)
#define ZZ_TR0() do { } while (0)
#endif

__device__ __forceinline__ void team_sync(const Team& tm) {
  if (tm.W > 1) asm volatile("bar.sync %0, %1;" ::"r"(tm.bar), "r"(tm.W * 32) : "memory");
}
// publication flag: release by the owner (after a __syncwarp over the writes), acquire by a reader
__device__ __forceinline__ void pub_release(int* flag, int gen) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(flag)), "r"(gen)
               : "memory");
}
__device__ __forceinline__ int ld_relaxed(const int* flag) {
  int v;
  asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(flag)) : "memory");
  return v;
}
// (spins use relaxed loads and one acquire fence once the awaited value is seen)
// wait until *flag == v1 (or, if v0 != 0, == v0); returns the value seen (all lanes)
__device__ __forceinline__ int pub_wait(const int* flag, int v1, int lane, int v0 = 0) {
  int v;
  do {   // warp-uniform: every lane loads the same word (one broadcast load)
    v = ld_relaxed(flag);
  } while (v != v1 && (v0 == 0 || v != v0));
  asm volatile("fence.acq_rel.cta;" ::: "memory");
  return v;
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
// Fast block solve (the tile's critical path): x = D^{-1} y for the rows of one
// block, D = beta S_bb - alpha T_bb, through the block-local inverse G = D^{-1}.  G
// depends on the column's eigenvalue and the staged tile only, not on y, so its rows are
// formed with independent instructions; the dependency chain through a block is then one
// short matrix-vector product instead of a row-by-row substitution.  Lanes: a real column's
// lane t forms the G rows of slots t, t + 4 (and 8 for t = 0); a complex pair's eight lanes
// u = 4 comp + t the row of slot u (and 8 for u = 0).  A row of G is formed right-looking:
// g_J = acc_J D_JJ^{-1}, then acc_l -= g_J D_Jl for l > J; a 2x2 diagonal block by its
// explicit inverse.  Pivots are the protected ones of the substitution (R8: |d| < smin ->
// smin).  The result is used only if it cannot overflow and G is well conditioned relative
// to D: for every row, (sum_J |G_qJ|) max|y| <= 2^1000 and (sum_J |G_qJ|) ||D_bb|| <= 2^40
// (an Inf or NaN fails both); the caller then takes the protected substitution
// (ProtectDivision / ProtectUpdate) for the column instead.  Returns that verdict for this
// lane's rows; xr/xi receive the lane's solution rows.
// ------------------------------------------------------------------------------------
// power of two sc with sc ||D_bb|| in [1/2, 1) (clamped to [2^-500, 2^500]): G is formed for
// sc D (no subnormal entries at any scale of the pencil; results equivariant under
// (S, T) -> 2^k (S, T)) and x = sc (G' y)
__device__ __forceinline__ double gscale(double dn) {
  int pe;
  frexp(dn, &pe);
  return (dn > 0.0) ? pow2k(-max(-500, min(500, pe))) : 1.0;
}

struct GRows {
  double ar[9], ai[9], br[9];                     // rows A (complex for pairs) and B (real)
  double cr7, ci7, cr8, ci8;                      // row C: slots 7 and 8
};

// Stage 1 of gprep_block: the inverses of the diagonal 1x1 / 2x2 blocks of one column (R8
// perturbation as in the substitution), written to the warp's pivot table ptab[slot][column][4]:
// 1x1 slot J: (1/d) at [J][0..1]; 2x2 block (J, J+1): real -- inv at [J][0..3] (row-major);
// pair -- inv row 0 at [J][0..3], row 1 at [J+1][0..3] (complex).  A rolled loop (compact code:
// the diagonal solve is bound by instruction fetch when its code is unrolled).
// G producers (one or two tasks per CTA): the CTA's idle warps form the rows of G of the task's
// blocks (the same gpiv/gprep arithmetic as the solving warp, so results do not depend on who
// formed them) into a ring of shared-memory slots; the solving warp only loads them.
constexpr int kGSlots = 4;
constexpr int kGVals = 22;                 // doubles per lane per block (see gstore / gload)
constexpr size_t kGSlotBytes = sizeof(double) * kGVals * 32;
struct GRing {
  double* slot;    // [ns][kGVals][32]
  int* ready;      // [ns]: block id + 1 of the rows in the slot
  int* done;       // [ns]: block id + 1 of the last rows the solving warp consumed
  int ns;          // slots (kGSlots / tasks per CTA)
};

template <bool PAIR>
__device__ __forceinline__ void gpiv_block(const Sm3& sm, int r0, int q0, int qe, double a, double b, double beta,
                                        double ab, int u, int col, double* ptab) {
  const int nl = PAIR ? 8 : 4;
#pragma unroll 1
  for (int J = u; J < qe; J += nl) {
    if (J < q0) continue;
    const int j = r0 + J;
    const int fJ = sm.fl[j];
    if (fJ == kRowBot2) continue;
    double* pt = ptab + (J * 8 + col) * 4;
    if (fJ == kRowTop2) {
      const double2 e00 = sm.ST[poff3(j) + j], e10 = sm.ST[poff3(j) + j + 1];
      const double2 e01 = sm.ST[poff3(j + 1) + j], e11 = sm.ST[poff3(j + 1) + j + 1];
      const double maxs = dmaxd(dmaxd(fabs(e00.x), fabs(e10.x)), dmaxd(fabs(e01.x), fabs(e11.x)));
      const double maxt = dmaxd(dmaxd(fabs(e00.y), fabs(e01.y)), fabs(e11.y));
      const double smin = dmaxd(__dmul_rn(kU, __dadd_rn(__dmul_rn(beta, maxs), __dmul_rn(ab, maxt))), kSmlnum);
      const cpx d00 = mkc(__fma_rn(-a, e00.y, __dmul_rn(beta, e00.x)), -b * e00.y);
      const cpx d01 = mkc(__fma_rn(-a, e01.y, __dmul_rn(beta, e01.x)), -b * e01.y);
      const double d10 = __dmul_rn(beta, e10.x);
      const cpx d11 = mkc(__fma_rn(-a, e11.y, __dmul_rn(beta, e11.x)), -b * e11.y);
      const double pv = dmaxd(dmaxd(n1(d00), n1(d01)), dmaxd(fabs(d10), n1(d11)));
      // the block scaled by a power of two sc ~ 1/pv (D^-1 = sc (sc D)^-1): no overflow or
      // underflow at any scale, so results are equivariant under (S, T) -> 2^k (S, T)
      int pe;
      frexp(pv, &pe);
      const double sc = pow2k(-max(-1000, min(1000, pe)));
      const cpx s00 = mkc(d00.re * sc, d00.im * sc), s11 = mkc(d11.re * sc, d11.im * sc);
      const cpx s01 = mkc(d01.re * sc, d01.im * sc);
      const double s10 = d10 * sc;
      if (!PAIR) {
        double det = fma(s00.re, s11.re, -(s01.re * s10));
        if (fabs(det) < smin * sc) det = smin * sc;
        const double rd = __drcp_rn(det) * sc;
        pt[0] = s11.re * rd;
        pt[1] = -s01.re * rd;
        pt[2] = -s10 * rd;
        pt[3] = s00.re * rd;
      } else {
        cpx det = csubx(cmulx(s00, s11), mkc(s01.re * s10, s01.im * s10));
        if (n1(det) < smin * sc) det = mkc(smin * sc, 0.0);
        cpx rd;   // 1 / det (Smith)
        if (fabs(det.re) >= fabs(det.im)) {
          const double sr = det.im * __drcp_rn(det.re), r = __drcp_rn(fma(det.im, sr, det.re));
          rd = mkc(r, -sr * r);
        } else {
          const double sr = det.re * __drcp_rn(det.im), r = __drcp_rn(fma(det.re, sr, det.im));
          rd = mkc(sr * r, -r);
        }
        rd = mkc(rd.re * sc, rd.im * sc);
        const cpx i00 = cmulx(s11, rd), i11 = cmulx(s00, rd);
        const cpx i01 = cmulx(mkc(-s01.re, -s01.im), rd), i10 = mkc(-s10 * rd.re, -s10 * rd.im);
        pt[0] = i00.re; pt[1] = i00.im; pt[2] = i01.re; pt[3] = i01.im;
        pt[32] = i10.re; pt[33] = i10.im; pt[34] = i11.re; pt[35] = i11.im;   // slot J+1
      }
    } else {
      const double2 dd = sm.ST[poff3(j) + j];
      cpx d = mkc(__fma_rn(-a, dd.y, __dmul_rn(beta, dd.x)), __dmul_rn(-b, dd.y));
      const double smin =
          dmaxd(__dmul_rn(kU, __dadd_rn(__dmul_rn(beta, fabs(dd.x)), __dmul_rn(ab, fabs(dd.y)))), kSmlnum);
      if (n1(d) < smin) d = mkc(smin, 0.0);
      if (!PAIR) {
        pt[0] = __drcp_rn(d.re);
      } else if (fabs(d.re) >= fabs(d.im)) {
        const double sr = d.im * __drcp_rn(d.re), r = __drcp_rn(fma(d.im, sr, d.re));
        pt[0] = r;
        pt[1] = -sr * r;
      } else {
        const double sr = d.re * __drcp_rn(d.im), r = __drcp_rn(fma(d.re, sr, d.im));
        pt[0] = sr * r;
        pt[1] = -r;
      }
    }
  }
}

// Stage 2: this lane's rows of G = D^{-1} for the block (slots [q0, qe)), right-looking:
// g_J = acc_J D_JJ^{-1} (from the pivot table), acc_l -= g_J D_Jl for l > J.
template <bool PAIR>
__device__ __forceinline__ void gprep_block(const Sm3& sm, int g8, int q0, int qe, int nt, double a, double b,
                                            double beta, double ab, int u, int col, double* ptab, GRows& gr) {
  const int r0 = g8 - 1;                          // row of slot 0
  __syncwarp();   // the pivot table (gpiv_block) is complete
  // entry (slot J, slot l) at sm.ST[off[l] + J]; columns past the tile are clamped (their
  // entries only feed accumulators of slots >= qe, which are never read)
  int off[9];
#pragma unroll
  for (int l = 0; l < 9; ++l) off[l] = poff3(min(r0 + l, nt - 1)) + r0;
  const int qA = u, qB = PAIR ? 99 : u + 4;       // slots of this lane's G rows (C: slot 8)
  const bool hasC = (u == 0) && qe == 9;
  double (&ar)[9] = gr.ar, (&ai)[9] = gr.ai, (&br)[9] = gr.br;
  double &cr7 = gr.cr7, &ci7 = gr.ci7, &cr8 = gr.cr8, &ci8 = gr.ci8;
  cr7 = 0.0; ci7 = 0.0; cr8 = 1.0; ci8 = 0.0;
#pragma unroll
  for (int J = 0; J < 9; ++J) {
    ar[J] = (J == qA) ? 1.0 : 0.0;
    ai[J] = 0.0;
    br[J] = (J == qB) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int J = 0; J < 9; ++J) {
    if (J < q0 || J >= qe) continue;
    const int fJ = sm.fl[r0 + J];
    if (fJ == kRowBot2) continue;                 // solved with the top row of its block
    const double* pt = ptab + (J * 8 + col) * 4;
    if (J < 8 && fJ == kRowTop2) {
      // ---- 2x2 diagonal block (J, J+1): [g_J, g_J+1] = [acc_J, acc_J+1] inv ----
      if (!PAIR) {
        const double2 p01 = *reinterpret_cast<const double2*>(pt), p23 = *reinterpret_cast<const double2*>(pt + 2);
        const double i00 = p01.x, i01 = p01.y, i10 = p23.x, i11 = p23.y;
#define ZZ_ROW2R(x0, x1)                                              \
  {                                                                   \
    const double g0_ = fma(x1, i10, x0 * i00), g1_ = fma(x1, i11, x0 * i01); \
    x0 = g0_;                                                         \
    x1 = g1_;                                                         \
  }
        ZZ_ROW2R(ar[J], ar[J + 1]);
        if (J >= 3) ZZ_ROW2R(br[J], br[J + 1]);
        if (J == 7 && hasC) ZZ_ROW2R(cr7, cr8);
#undef ZZ_ROW2R
      } else {
        const double2 q0v = *reinterpret_cast<const double2*>(pt), q1v = *reinterpret_cast<const double2*>(pt + 2);
        const double2 q2v = *reinterpret_cast<const double2*>(pt + 32), q3v = *reinterpret_cast<const double2*>(pt + 34);
        const cpx i00 = mkc(q0v.x, q0v.y), i01 = mkc(q1v.x, q1v.y), i10 = mkc(q2v.x, q2v.y), i11 = mkc(q3v.x, q3v.y);
#define ZZ_ROW2C(r0v, i0v, r1v, i1v)                                                        \
  {                                                                                         \
    const double g0r = fma(-i1v, i10.im, fma(r1v, i10.re, fma(-i0v, i00.im, r0v * i00.re))); \
    const double g0i = fma(i1v, i10.re, fma(r1v, i10.im, fma(i0v, i00.re, r0v * i00.im)));   \
    const double g1r = fma(-i1v, i11.im, fma(r1v, i11.re, fma(-i0v, i01.im, r0v * i01.re))); \
    const double g1i = fma(i1v, i11.re, fma(r1v, i11.im, fma(i0v, i01.re, r0v * i01.im)));   \
    r0v = g0r; i0v = g0i; r1v = g1r; i1v = g1i;                                             \
  }
        ZZ_ROW2C(ar[J], ai[J], ar[J + 1], ai[J + 1]);
        if (J == 7 && hasC) ZZ_ROW2C(cr7, ci7, cr8, ci8);
#undef ZZ_ROW2C
      }
#pragma unroll
      for (int l = 0; l < 9; ++l) {   // constant trip count: unrolled after J is
        if (l >= J + 2) {
          const double2 f0 = sm.ST[off[l] + J], f1 = sm.ST[off[l] + J + 1];
          const double D0r = __fma_rn(-a, f0.y, __dmul_rn(beta, f0.x)), D1r = __fma_rn(-a, f1.y, __dmul_rn(beta, f1.x));
          if (!PAIR) {
            ar[l] = fma(-ar[J + 1], D1r, fma(-ar[J], D0r, ar[l]));
            if (J >= 3) br[l] = fma(-br[J + 1], D1r, fma(-br[J], D0r, br[l]));
          } else {
            const double D0i = -b * f0.y, D1i = -b * f1.y;
            ar[l] = fma(ai[J + 1], D1i, fma(-ar[J + 1], D1r, fma(ai[J], D0i, fma(-ar[J], D0r, ar[l]))));
            ai[l] = fma(-ar[J + 1], D1i, fma(-ai[J + 1], D1r, fma(-ar[J], D0i, fma(-ai[J], D0r, ai[l]))));
          }
        }
      }
    } else {
      // ---- 1x1 pivot ----
      if (!PAIR) {
        const double r = pt[0];
        ar[J] *= r;
        if (J >= 3) br[J] *= r;
        if (J == 7 && hasC) cr7 *= r;
        if (J == 8 && hasC) cr8 *= r;
      } else {
        const double2 rv = *reinterpret_cast<const double2*>(pt);
        const cpx rd = mkc(rv.x, rv.y);
#define ZZ_MULR(vr_, vi_)                                                            \
  {                                                                                 \
    const double nr_ = fma(-vi_, rd.im, vr_ * rd.re), ni_ = fma(vi_, rd.re, vr_ * rd.im); \
    vr_ = nr_;                                                                      \
    vi_ = ni_;                                                                      \
  }
        ZZ_MULR(ar[J], ai[J]);
        if (J == 7 && hasC) ZZ_MULR(cr7, ci7);
        if (J == 8 && hasC) ZZ_MULR(cr8, ci8);
#undef ZZ_MULR
      }
#pragma unroll
      for (int l = 0; l < 9; ++l) {
        if (l >= J + 1) {
          const double2 f = sm.ST[off[l] + J];
          const double Dr = __fma_rn(-a, f.y, __dmul_rn(beta, f.x));
          if (!PAIR) {
            ar[l] = fma(-ar[J], Dr, ar[l]);
            if (J >= 3) br[l] = fma(-br[J], Dr, br[l]);
            if (J == 7 && l == 8 && hasC) cr8 = fma(-cr7, Dr, cr8);
          } else {
            const double Di = -b * f.y;
            ar[l] = fma(ai[J], Di, fma(-ar[J], Dr, ar[l]));
            ai[l] = fma(-ar[J], Di, fma(-ai[J], Dr, ai[l]));
            if (J == 7 && l == 8 && hasC) {
              const double nr = fma(ci7, Di, fma(-cr7, Dr, cr8));
              ci8 = fma(-cr7, Di, fma(-ci7, Dr, ci8));
              cr8 = nr;
            }
          }
        }
      }
    }
  }
  __syncwarp();   // the pivot table is reused (slow path, next block)
}

// a lane's rows of G in a ring slot (element i of lane l at [i][l]: conflict-free)
template <bool PAIR>
__device__ __forceinline__ void gstore(const GRows& gr, double* sl, int lane) {
#pragma unroll
  for (int J = 0; J < 9; ++J) sl[J * 32 + lane] = gr.ar[J];
  if (!PAIR) {
#pragma unroll
    for (int J = 3; J < 9; ++J) sl[(6 + J) * 32 + lane] = gr.br[J];
    sl[15 * 32 + lane] = gr.cr7;
    sl[16 * 32 + lane] = gr.cr8;
  } else {
#pragma unroll
    for (int J = 0; J < 9; ++J) sl[(9 + J) * 32 + lane] = gr.ai[J];
    sl[18 * 32 + lane] = gr.cr7;
    sl[19 * 32 + lane] = gr.ci7;
    sl[20 * 32 + lane] = gr.cr8;
    sl[21 * 32 + lane] = gr.ci8;
  }
}
template <bool PAIR>
__device__ __forceinline__ void gload(GRows& gr, const double* sl, int lane) {
#pragma unroll
  for (int J = 0; J < 9; ++J) {
    gr.ar[J] = sl[J * 32 + lane];
    gr.ai[J] = 0.0;
    gr.br[J] = 0.0;
  }
  if (!PAIR) {
#pragma unroll
    for (int J = 3; J < 9; ++J) gr.br[J] = sl[(6 + J) * 32 + lane];
    gr.cr7 = sl[15 * 32 + lane];
    gr.cr8 = sl[16 * 32 + lane];
    gr.ci7 = 0.0;
    gr.ci8 = 0.0;
  } else {
#pragma unroll
    for (int J = 0; J < 9; ++J) gr.ai[J] = sl[(9 + J) * 32 + lane];
    gr.cr7 = sl[18 * 32 + lane];
    gr.ci7 = sl[19 * 32 + lane];
    gr.cr8 = sl[20 * 32 + lane];
    gr.ci8 = sl[21 * 32 + lane];
  }
}

// x = G y for this lane's rows and the overflow / conditioning verdict (see gprep_block)
template <bool PAIR>
__device__ __forceinline__ bool gapply_block(const GRows& gr, const double* wslab, int q0, int qe, int tq, double dn,
                                             double sc, int team, int u, double (&xr)[3], double (&xi)[3]) {
  const int qB = PAIR ? 99 : u + 4, qA = u;
  const bool hasC = (u == 0) && qe == 9;
  const int pt = PAIR ? (team & ~1) : team;       // slab column of Re (Im at pt + 1)
  const double (&ar)[9] = gr.ar, (&ai)[9] = gr.ai, (&br)[9] = gr.br;
  const double cr7 = gr.cr7, ci7 = gr.ci7, cr8 = gr.cr8, ci8 = gr.ci8;
  // ---- x = G y (sources in ascending slot order), row sums of |G| ----
  double ymax = 0.0, sA = 0.0, sB = 0.0;
  double xar = 0.0, xai = 0.0, xbr = 0.0, xcr = 0.0, xci = 0.0;
#pragma unroll
  for (int J = 0; J < 9; ++J) {
    if (J >= q0 && J < qe && J < tq) {   // (a tip block: the leading rows only)
      const double yr = wslab[J * 8 + pt], yi = PAIR ? wslab[J * 8 + pt + 1] : 0.0;
      ymax = dmaxd(ymax, PAIR ? dmaxd(fabs(yr), fabs(yi)) : fabs(yr));
      if (!PAIR) {
        xar = fma(ar[J], yr, xar);
        sA += fabs(ar[J]);
        if (J >= 3) {
          xbr = fma(br[J], yr, xbr);
          sB += fabs(br[J]);
        }
      } else {
        xar = fma(-ai[J], yi, fma(ar[J], yr, xar));
        xai = fma(ai[J], yr, fma(ar[J], yi, xai));
        sA += fabs(ar[J]) + fabs(ai[J]);
      }
      if (J == 7 && hasC) {
        xcr = fma(-ci7, yi, fma(cr7, yr, xcr));
        xci = fma(ci7, yr, fma(cr7, yi, xci));
      }
      if (J == 8 && hasC) {
        xcr = fma(-ci8, yi, fma(cr8, yr, xcr));
        xci = fma(ci8, yr, fma(cr8, yi, xci));
      }
    }
  }
  const double sC = (qe == 9) ? (fabs(cr7) + fabs(ci7) + fabs(cr8) + fabs(ci8)) : 0.0;
  const double yb = PAIR ? 2.0 * ymax : ymax;
  const double lim = 0x1p1000 / sc;   // |x| = sc |G' y| <= 2^1000
  bool ok = true;
  if (qA >= q0 && qA < qe) ok = ok && (sA * yb <= lim) && (sA * dn <= 0x1p40);
  if (!PAIR && qB < qe) ok = ok && (sB * yb <= lim) && (sB * dn <= 0x1p40);
  if (hasC) ok = ok && (sC * yb <= lim) && (sC * dn <= 0x1p40);
  xr[0] = xar * sc; xi[0] = xai * sc;
  xr[1] = xbr * sc; xi[1] = 0.0;
  xr[2] = xcr * sc; xi[2] = xci * sc;
  return ok;
}

// max |value| over the rows [r0, r1) of the column held by this warp (position p holds group
// (p - rot) mod G; pairs: over both components)
template <int G, bool PAIR>
__device__ __forceinline__ double range_max(const Seg<G>& s, int rot, int t, int r0, int r1) {
  double m = 0.0;
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int g = (q - rot + G) % G;
    const int r = 8 * g + 2 * t;
    if (r >= r0 && r < r1) m = fmax(m, fabs(s.y[q][0]));
    if (r + 1 >= r0 && r + 1 < r1) m = fmax(m, fabs(s.y[q][1]));
  }
  m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 1));
  m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 2));
  if (PAIR) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 4));
  return m;
}

// DMMA update of the groups g in [gmin, k) held by this warp (position q holds group
// top - (G-1-q)) with the solution of block k: Y(8 columns x 8 rows) += A (8 x 4) . [S | T]^T
// over the block's source rows 8k + 4 kk + t (kk = 0, 1) and its straddling top row 8k - 1
// (kk = 2) -- the instruction sequence of the block's owner, for every warp.
template <int G>
__device__ __forceinline__ void dmma_block(Seg<G>& s, int top, int k, int gmin, bool st, const Sm3& sm, int nt,
                                           int t, int team, const double (&aS)[3], const double (&aT)[3]) {
  const int g8 = 8 * k;
  // source chunk outermost: consecutive DMMAs belong to different groups (independent
  // accumulators), so they issue back to back instead of waiting on each other; per group the
  // order of the products (kk = 0, 1, 2; S then T) is unchanged
#pragma unroll
  for (int kk = 0; kk < 3; ++kk) {
    if (kk == 2 && !st) continue;
    const int src0 = (kk < 2) ? g8 + 4 * kk : g8 - 4;
    const double2* col = sm.ST + poff3(min(src0 + t, nt - 1)) + team;
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int g = top - (G - 1 - q);
      if (g >= gmin && g < k) {
        const double2 v = col[8 * g];
        dmma3(s.y[q][0], s.y[q][1], aS[kk], v.x);
        dmma3(s.y[q][0], s.y[q][1], aT[kk], v.y);
      }
    }
  }
}

// A fragments of block k's update from its publication: lane (team, t) holds its column's
// coefficients [-beta x | alpha x] for source row src0 + t (the owner forms the same values
// from its registers).
template <bool PAIR>
__device__ __forceinline__ void pub_frags(const double* x, const Sm3& sm, int k, double a, double b, double beta,
                                          int team, int t, int comp, double (&aS)[3], double (&aT)[3]) {
  const int g8 = 8 * k, e0 = sm.bs[k + 1];
  const bool st = sm.bs[k] < g8;
#pragma unroll
  for (int kk = 0; kk < 3; ++kk) {
    const int slot = (kk < 2) ? 1 + 4 * kk + t : 0;
    const bool in = (kk < 2) ? (g8 + 4 * kk + t < e0) : (st && t == 3);
    const double v = in ? x[slot * 8 + team] : 0.0;
    const double o = (PAIR && in) ? x[slot * 8 + (team ^ 1)] : 0.0;
    const double xr = PAIR ? (comp ? o : v) : v, xi = PAIR ? (comp ? v : o) : 0.0;
    aS[kk] = -(beta * v);
    aT[kk] = PAIR ? (comp ? (a * xi + b * xr) : (a * xr - b * xi)) : a * xr;
  }
}

// The protected substitution of one block (P:142-146 with ProtectDivision / ProtectUpdate,
// P:175-200): the rows of the block in the warp's slab, solved 1x1 / 2x2 block by 1x1 / 2x2
// block bottom-up with in-block updates against the running bound.  Out of line: the block-local
// inverse handles almost every block, and the diagonal solve is bound by instruction fetch.
struct SlowSt { double bound, xnb; int ex, kseg; };

template <bool PAIR>
__device__ __forceinline__ SlowSt slow_block(const Sm3& sm, double* wslab, double* pslab, int g8, int q0, int s0,
                                          int e0, double a, double b, double beta, double ab, bool tip, int tipr,
                                          int team, int t, int comp, SlowSt st) {
  double bound = st.bound, xnb = st.xnb;
  int ex = st.ex, kseg = st.kseg;
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
  st.bound = bound; st.xnb = xnb; st.ex = ex; st.kseg = kseg;
  return st;
}

// ------------------------------------------------------------------------------------
// A G producer (warp h of nh idle warps of a CTA holding one or two tasks): the rows of G of the
// task's blocks nblk-1-h, nblk-1-h-nh, ... (the first while the solving warp loads its
// right-hand side), with exactly the solving warp's arithmetic, into the ring slot block % ns
// once the solving warp has consumed the slot's previous rows.
// ------------------------------------------------------------------------------------
template <bool PAIR>
__device__ __forceinline__ void gproduce_task(const Diag2Params& p, const Sm3& sm, int nblk, int task, int lane,
                                              int h, int nh, double* ptab, const GRing& ring) {
  const DevPlan& P = p.P;
  const int team = lane >> 2, t = lane & 3;
  const int comp = PAIR ? (team & 1) : 0;
  const int cpt = p.cpt;
  const int slot = PAIR ? (team >> 1) : team;
  const int item = PAIR ? task * (cpt / 2) + slot : task * cpt + slot;
  const int n_items = PAIR ? p.n_pair : p.n_real;
  const bool valid = item < n_items && slot < (PAIR ? cpt / 2 : cpt);
  const int c0 = valid ? (PAIR ? p.pair_items[item] : p.real_items[item]) : -1;
  double a = 0.0, b = 0.0, beta = 0.0;
  if (valid) {
    a = P.col_a[c0];
    b = PAIR ? P.col_b[c0] : 0.0;
    beta = P.col_beta[c0];
  }
  const double ab = __dadd_rn(fabs(a), fabs(b));
  const int u = PAIR ? comp * 4 + t : t, col = PAIR ? (team & ~1) : team;
  for (int k = nblk - 1 - h; k >= 0; k -= nh) {
    const int g8 = 8 * k, q0 = sm.bs[k] - (g8 - 1), qe = sm.bs[k + 1] - (g8 - 1);
    const double2 bnv = sm.bn[k];
    const double gsc = gscale(__dadd_rn(__dmul_rn(beta, bnv.x), __dmul_rn(ab, bnv.y)));
    gpiv_block<PAIR>(sm, g8 - 1, q0, qe, a * gsc, b * gsc, beta * gsc, ab * gsc, u, col, ptab);
    GRows gr;
    gprep_block<PAIR>(sm, g8, q0, qe, p.nt, a * gsc, b * gsc, beta * gsc, ab * gsc, u, col, ptab, gr);
    const int si = k % ring.ns;
    if (k + ring.ns <= nblk - 1) pub_wait(&ring.done[si], k + ring.ns + 1, lane);
    gstore<PAIR>(gr, ring.slot + si * (kGVals * 32), lane);
    __syncwarp();
    if (lane == 0) pub_release(&ring.ready[si], k + 1);
  }
}

// ------------------------------------------------------------------------------------
// One task: 8 real columns (PAIR = false) or 4 complex pairs (PAIR = true) of tile I.
// ------------------------------------------------------------------------------------
template <int G, bool PAIR, bool TEAMS>
__device__ __forceinline__ void solve_task(const Diag2Params& p, const Sm3& sm, int nblk, int task, int lane,
                                        const Team& tm, const GRing ring) {
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
  // pending exponent of the column (read before any warp of the team writes the new one)
  const int ep = (valid && !tip) ? P.e_pend[c] : 0;
  const int nt = p.nt;
  const int pbase = lane & ~3;           // first lane of this column's team
  constexpr int CUR = G - 1, PRV = G - 2;

  // ---- the team (W warps per task; W = 1: one warp): warp w owns the blocks [lo, hi) and
  // their rows [rlo, rhi); the chain of blocks runs bottom-up through the warps W-1, ..., 0.
  // Every warp applies the published solution of each block below its range to its rows
  // (the same DMMA instructions on the same operands as the block's owner would issue), so
  // the arithmetic of a column does not depend on W.  Group lo-1 is kept as well when it
  // holds the top row of a 2x2 block that straddles into block lo. ----
  const int W = TEAMS ? tm.W : 1, w = TEAMS ? tm.w : 0;   // (one warp: the team code compiles away)
  const int lo = (w * nblk) / W, hi = ((w + 1) * nblk) / W;
  const int rlo = sm.bs[lo], rhi = sm.bs[hi];
  const int gmin = (lo > 0 && rlo < 8 * lo) ? lo - 1 : lo;
  Pub* const pub = tm.pub;
  // ---- right-hand side (tips start from zero) ----
  Seg<G> s;
  {
    const double* xc = p.X + (long long)(valid ? c : 0) * p.ldx + p.t0;
    const bool ld = valid && !tip;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int r = 8 * g + 2 * t;
      const bool mine = ld && g >= gmin && g < hi;
      s.y[g][0] = (mine && r < nt) ? xc[r] : 0.0;
      s.y[g][1] = (mine && r + 1 < nt) ? xc[r + 1] : 0.0;
    }
  }
  int rot = 0;
  while (rot < G - hi) { s.rotate(); ++rot; }   // group hi-1 -> position G-1
  int ex = 0;   // exponent of the segment relative to e_pend (stored = 2^ex true)
  // running upper bound of max |pending| (Alg. 3's y^): initially the exact maximum over
  // the tile's rows (a max is exact and order-independent: the same for every W)
  double bound = range_max<G, PAIR>(s, rot, t, rlo, rhi);
  // the pivots of this warp's first block (the rcp chains of G's stage 1), formed before the
  // chain reaches it (W > 1: while the warps below solve their blocks); the others in turn
  int pre_blk = -1;
  if (W > 1 && hi > lo) {
    const int k = hi - 1, g8k = 8 * k;
    const double2 bk = sm.bn[k];
    const double sck = gscale(__dadd_rn(__dmul_rn(beta, bk.x), __dmul_rn(ab, bk.y)));
    gpiv_block<PAIR>(sm, g8k - 1, sm.bs[k] - (g8k - 1), sm.bs[k + 1] - (g8k - 1), a * sck, b * sck, beta * sck, ab * sck,
                     PAIR ? comp * 4 + t : t, PAIR ? (team & ~1) : team, tm.pslab);
    pre_blk = k;
  }
  ZZ_TR(200 + w);
  if (W > 1) {
    if (t == 0) tm.red0[w * 8 + team] = bound;
    team_sync(tm);
    if (hi == nblk) {
      bound = 0.0;
      for (int v = 0; v < W; ++v) bound = dmaxd(bound, tm.red0[v * 8 + team]);
    }
    // the blocks below this warp's range: their scalings and updates, in the chain's order
    for (int k = nblk - 1; k >= hi; --k) {
      Pub& pk = pub[k];
      const int v = pub_wait(&pk.flag, 2 * tm.gen, lane, 2 * tm.gen - 1);
      ZZ_TR(k * 8 + 5);
      const int k1 = pk.kseg[team];
      if (k1 < 0) s.scale(k1);
      if (v != 2 * tm.gen) {
        // the owner asks for the exact maximum of the pending rows (after the block's
        // in-block scaling): this warp's rows are all above block k
        const double mx = range_max<G, PAIR>(s, rot, t, rlo, rhi);
        if (t == 0) tm.red2[w * 8 + team] = mx;
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          atomicAdd(&pk.cnt, 1);
        }
        pub_wait(&pk.flag, 2 * tm.gen, lane);
      }
      const int k2 = pk.eu[team];
      if (k2 < 0) s.scale(k2);
      if (k > 0) {
        double aS[3], aT[3];
        pub_frags<PAIR>(pk.x, sm, k, a, b, beta, team, t, comp, aS, aT);
        dmma_block<G>(s, hi - 1, k, gmin, sm.bs[k] < 8 * k, sm, nt, t, team, aS, aT);
        // the top row of a block that straddles into block hi belongs to that block's owner
        if (k == hi && sm.bs[k] < 8 * k && t == 3) s.y[G - 1][1] = 0.0;   // group hi-1 at position G-1
      }
      ZZ_TR(k * 8 + 6);
    }
    ZZ_TR(220 + w);
    if (hi < nblk && hi > lo) {
      bound = pub[hi].bound[team];
      ex = pub[hi].ex[team];
    }
  }

  for (int blk = hi - 1; blk >= lo; --blk) {
    double* const wslab = pub[W == 1 ? 0 : blk].x;
    double* const pslab = tm.pslab;
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
    __syncwarp();
    // ---- fast path: the block-local inverse (gsolve_block); the tip's own block and
    // columns whose check fails take the protected substitution below ----
    ZZ_TR(blk * 8 + 0);
    double xfr[3], xfi[3];
    const double2 bnv = sm.bn[blk];
    const double dn0 = __dadd_rn(__dmul_rn(beta, bnv.x), __dmul_rn(ab, bnv.y));
    const double gsc = gscale(dn0), dn = dn0 * gsc;   // G is formed for gsc D (gscale)
    const int u = PAIR ? comp * 4 + t : t;
    GRows gpre;
    if (ring.slot != nullptr) {
      // the rows of G formed by the CTA's producer warps (gproduce_task)
      const int si = blk % ring.ns;
      pub_wait(&ring.ready[si], blk + 1, lane);
      gload<PAIR>(gpre, ring.slot + si * (kGVals * 32), lane);
      __syncwarp();
      if (lane == 0) pub_release(&ring.done[si], blk + 1);
      ZZ_TR(256 + blk * 8 + 0);
    } else {
      if (blk != pre_blk)
        gpiv_block<PAIR>(sm, g8 - 1, q0, e0 - (g8 - 1), a * gsc, b * gsc, beta * gsc, ab * gsc, u,
                         PAIR ? (team & ~1) : team, pslab);
      ZZ_TR(256 + blk * 8 + 0);
      gprep_block<PAIR>(sm, g8, q0, e0 - (g8 - 1), nt, a * gsc, b * gsc, beta * gsc, ab * gsc, u,
                        PAIR ? (team & ~1) : team, pslab, gpre);
    }
    ZZ_TR(256 + blk * 8 + 1);
    // ---- the tip's own block (Kernel 1; reading R10): the eigenvalue rows get the tip
    // values, the rows above them in the block are x = G y with G restricted to the leading
    // rows (its entries there do not involve the singular pivot) and y = -D(rows, tip rows) x_tip
    // (tips start from zero; the slab takes y, and back the zeros if the substitution runs) ----
    const bool tipblk = tip && tipr >= s0 && tipr < e0;
    int tq = 99;
    cpx xt0 = mkc(0.0, 0.0), xt1 = mkc(0.0, 0.0);
    if (tipblk) {
      const int rr = tipr, top = PAIR ? rr - 1 : rr;
      tq = top - (g8 - 1);
      if (!PAIR) {
        xt0 = mkc(1.0, 0.0);
      } else {
        const double2 d21 = sm.ST[poff3(rr - 1) + rr], d22 = sm.ST[poff3(rr) + rr];
        const double pp = __dmul_rn(beta, d21.x);
        const cpx qq = mkc(__fma_rn(-a, d22.y, __dmul_rn(beta, d22.x)), __dmul_rn(-b, d22.y));
        if (fabs(pp) >= n1(qq)) {
          xt1 = mkc(1.0, 0.0);
          xt0 = mkc(__ddiv_rn(-qq.re, pp), __ddiv_rn(-qq.im, pp));
        } else {
          xt0 = mkc(1.0, 0.0);
          const cpx z = cdivx(mkc(pp, 0.0), qq);
          xt1 = mkc(-z.re, -z.im);
        }
      }
      for (int r = t; r < tq; r += 4) {   // slot r of the column: lane r & 3
        if (r < q0) continue;
        const int j = g8 - 1 + r;
        const double2 f0 = sm.ST[poff3(top) + j];
        cpx yv = cmulx(mkc(__fma_rn(-a, f0.y, __dmul_rn(beta, f0.x)), __dmul_rn(-b, f0.y)), xt0);
        if (PAIR) {
          const double2 f1 = sm.ST[poff3(rr) + j];
          const cpx d1 = mkc(__fma_rn(-a, f1.y, __dmul_rn(beta, f1.x)), __dmul_rn(-b, f1.y));
          const cpx p1 = cmulx(d1, xt1);
          yv = mkc(__dadd_rn(yv.re, p1.re), __dadd_rn(yv.im, p1.im));
        }
        wslab[r * 8 + team] = PAIR ? (comp ? -yv.im : -yv.re) : -yv.re;
      }
    }
    __syncwarp();
    bool okc = gapply_block<PAIR>(gpre, wslab, q0, e0 - (g8 - 1), tq, dn, gsc, team, u, xfr, xfi);
    ZZ_TR(256 + blk * 8 + 2);
#ifdef ZZ_VARIANT_NOFAST
    okc = false;
#endif
    {   // one verdict per column (pair: both columns); every lane shuffles
      int v = okc ? 1 : 0;
      v &= __shfl_xor_sync(0xffffffffu, v, 1);
      v &= __shfl_xor_sync(0xffffffffu, v, 2);
      if (PAIR) v &= __shfl_xor_sync(0xffffffffu, v, 4);
      okc = (v != 0) || !valid;
    }
    int kseg = 0;
    ZZ_TR(blk * 8 + 1);
    if (tipblk && !okc)   // the substitution starts the tip from zero itself
      for (int r = t; r < tq; r += 4) wslab[r * 8 + team] = 0.0;
    if (__any_sync(0xffffffffu, !okc)) {
    const double bound0 = bound;
    const int ex0 = ex;
    {
      SlowSt ss;
      ss.bound = bound; ss.xnb = xnb; ss.ex = ex; ss.kseg = kseg;
      ss = slow_block<PAIR>(sm, wslab, pslab, g8, q0, s0, e0, a, b, beta, ab, tip, tipr, team, t, comp, ss);
      bound = ss.bound; xnb = ss.xnb; ex = ss.ex; kseg = ss.kseg;
    }
    if (okc) {   // the substitution ran for other columns of the warp: keep the fast result
      bound = bound0;
      ex = ex0;
      kseg = 0;
    }
    }   // protected substitution
    ZZ_TR(blk * 8 + 2);
    if (okc) {
      const int qe = e0 - (g8 - 1);
      const int pt = PAIR ? (team & ~1) : team;
      if (tipblk) {   // the tip rows and the zeros below them
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int q = (i == 0) ? u : (i == 1 ? u + 4 : 8);
          const cpx v = (q == tq) ? xt0 : ((PAIR && q == tq + 1) ? xt1 : mkc(0.0, 0.0));
          if (q >= tq) {
            xfr[i] = v.re;
            xfi[i] = v.im;
          }
        }
      }
      double xm = 0.0;
      if (u >= q0 && u < qe) {
        wslab[u * 8 + pt] = xfr[0];
        if (PAIR) wslab[u * 8 + pt + 1] = xfi[0];
        xm = PAIR ? dmaxd(fabs(xfr[0]), fabs(xfi[0])) : fabs(xfr[0]);
      }
      if (!PAIR && u + 4 < qe) {
        wslab[(u + 4) * 8 + team] = xfr[1];
        xm = dmaxd(xm, fabs(xfr[1]));
      }
      if (u == 0 && qe == 9) {
        wslab[64 + pt] = xfr[2];
        if (PAIR) wslab[64 + pt + 1] = xfi[2];
        xm = dmaxd(xm, PAIR ? dmaxd(fabs(xfr[2]), fabs(xfi[2])) : fabs(xfr[2]));
      }
      xnb = xm;
    }
    {   // max |x| over the block's rows of the column (fast result)
      double xm = okc ? xnb : 0.0;
      xm = dmaxd(xm, __shfl_xor_sync(0xffffffffu, xm, 1));
      xm = dmaxd(xm, __shfl_xor_sync(0xffffffffu, xm, 2));
      if (PAIR) xm = dmaxd(xm, __shfl_xor_sync(0xffffffffu, xm, 4));
      if (okc) xnb = xm;
    }
    __syncwarp();
    // ---- the block's rows back to their owner lanes ----
    if (kseg < 0) s.scale(kseg);
    s.y[CUR][0] = wslab[(1 + 2 * t) * 8 + team];
    s.y[CUR][1] = wslab[(2 + 2 * t) * 8 + team];
    if (st && t == 3) s.y[PRV][1] = wslab[team];
    __syncwarp();
    int eu = 0;
    if (blk > 0) {
      // ---- update of all rows above the block by DMMA (Alg. 3 on the in-tile panel) ----
      const double2 tv = sm.tau[blk];
      const double tt = __dadd_rn(__dmul_rn(beta, tv.x), __dmul_rn(ab, tv.y));
      // ProtectUpdate: while the running bound of the pending rows keeps every column of the
      // task below 2^1020 nothing scales; otherwise the exact maximum of the pending rows
      // replaces the bound of every column (rows above this warp's range: asked from the warps
      // that hold them, after the block's in-block scaling, which they apply first)
      double nb = fma(tt, xnb, bound);
      const bool need = !(nb <= 0x1p1020);
      if (__any_sync(0xffffffffu, need)) {
        double mx = range_max<G, PAIR>(s, rot, t, rlo, s0);
        if (W > 1 && w > 0) {
          Pub& pk = pub[blk];
          if (t == 0) pk.kseg[team] = kseg;
          __syncwarp();
          if (lane == 0) pub_release(&pk.flag, 2 * tm.gen - 1);
          while (ld_relaxed(&pk.cnt) != w) {
          }
          asm volatile("fence.acq_rel.cta;" ::: "memory");
          for (int v = 0; v < w; ++v) mx = dmaxd(mx, tm.red2[v * 8 + team]);
          __syncwarp();
          if (lane == 0) pk.cnt = 0;
        }
        bound = mx;   // every column of the task (as one warp would)
        eu = protect_update(bound, tt, xnb);
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
      ZZ_TR(256 + blk * 8 + 3);
      dmma_block<G>(s, blk, blk, gmin, st, sm, nt, t, team, aS, aT);
      ZZ_TR(256 + blk * 8 + 4);
      if (st && t == 3) s.y[PRV][1] = keep;
    }
    ZZ_TR(blk * 8 + 3);
    if (W > 1) {
      // ---- publish the block: its rows at the segment's new scale, the scalings, the chain
      // state (slot r of column `team` rescaled by lane r & 3: after the __syncwarp above) ----
      if (eu < 0)
        for (int r = t; r < 9; r += 4) wslab[r * 8 + team] = scale2k(wslab[r * 8 + team], eu);
      Pub& pk = pub[blk];
      if (t == 0) {
        pk.kseg[team] = kseg;
        pk.eu[team] = eu;
        pk.ex[team] = ex;
        pk.bound[team] = bound;
      }
      __syncwarp();
      if (lane == 0) pub_release(&pk.flag, 2 * tm.gen);
    }
    ZZ_TR(blk * 8 + 4);
    s.rotate();
    ++rot;
  }
  // ---- the scalings of the blocks above this warp's range: one exponent per segment ----
  if (W > 1) {
    for (int k = lo - 1; k >= 0; --k) {
      const Pub& pk = pub[k];
      pub_wait(&pk.flag, 2 * tm.gen, lane);
      const int k1 = pk.kseg[team], k2 = pk.eu[team];
      if (k1 < 0) s.scale(k1);
      if (k2 < 0) s.scale(k2);
    }
    if (!(lo == 0 && hi > 0)) ex = pub[0].ex[team];   // (block 0's publication was awaited above)
  }
  // ---- segment norms, exponent and the scaling decision of the next update (a5) ----
  double lm = 0.0, lh = 0.0;
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int g = (q - rot % G + G) % G;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = 8 * g + 2 * t + i;
      const double v = s.y[q][i];
      const double o = PAIR ? __shfl_xor_sync(0xffffffffu, v, 4) : 0.0;
      if (r >= rlo && r < rhi) {
        lm = fmax(lm, fabs(v));
        lh = fmax(lh, PAIR ? __dadd_rn(__dmul_rn(0.5, fabs(v)), __dmul_rn(0.5, fabs(o))) : __dmul_rn(0.5, fabs(v)));
      }
    }
  }
  lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, 1));
  lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, 2));
  lh = fmax(lh, __shfl_xor_sync(0xffffffffu, lh, 1));
  lh = fmax(lh, __shfl_xor_sync(0xffffffffu, lh, 2));
  if (PAIR) lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, 4));
  if (W > 1) {   // over the team (exact, order-independent)
    if (t == 0) {
      tm.red1[(w * 8 + team) * 2] = lm;
      tm.red1[(w * 8 + team) * 2 + 1] = lh;
    }
    team_sync(tm);
    lm = 0.0;
    lh = 0.0;
    for (int v = 0; v < W; ++v) {
      lm = fmax(lm, tm.red1[(v * 8 + team) * 2]);
      lh = fmax(lh, tm.red1[(v * 8 + team) * 2 + 1]);
    }
  }
  const bool w0 = (w == 0);   // the team's warp 0 writes the per-column state
  ZZ_TR(140 + w);
  const int es = ep + ex;
  int sx = 0;
  if (valid) {
    const long long so = (long long)p.I * p.n_sel + c;
    if (t == 0 && w0) {
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
        // (lookahead: the previous group's recorded bound of these rows, at the exponent e_p
        // it was recorded at, instead of the maximum the bulk update is still measuring)
        nyv = p.use_bound ? P.nYb[(long long)p.bnd_in * p.n_sel + c0] : __longlong_as_double((long long)nyi[c0]);
        if (PAIR) nyv = dmaxd(nyv, p.use_bound ? P.nYb[(long long)p.bnd_in * p.n_sel + c0 + 1] : __longlong_as_double((long long)nyi[c0 + 1]));
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
      if (t == 0 && w0) {
        // lookahead: this maximum covers the rows the band and bulk updates measured, which
        // can differ from the plain schedule's; a decision that scales is recomputed without
        // lookahead (as for a group's first decision)
        if ((p.record_bound || p.use_bound) && ef < g0) atomicOr(&P.status[6], 1);
        P.sY[c] = ef - e_p;
        P.e_pend[c] = ef;
        P.nY[(long long)(1 - p.nY_in) * p.n_sel + c] = 0ull;
        // lookahead: an upper bound of |pending| after this group's update, at exponent ef
        // (2^(ef-g) (y^ + tau x^), with a margin for the rounding of the sum and the update)
        if (p.record_bound)
          P.nYb[(long long)(1 - p.bnd_in) * p.n_sel + c] = scale2k(__dmul_rn(__dadd_rn(yh, __dmul_rn(tau, xh)), 1.0 + 0x1p-40), ef - g0);
      }
      // each earlier W of this column brought to ef (rare), or zero where the column was not
      // active at that step (stale entries)
#pragma unroll
      for (int k = 0; k < kMaxGroup - 1; ++k) {
        if (k < p.n_prev && w0) {
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
        nyv = p.use_bound ? P.nYb[(long long)p.bnd_in * p.n_sel + c0] : __longlong_as_double((long long)nyi[c0]);
        if (PAIR) nyv = dmaxd(nyv, p.use_bound ? P.nYb[(long long)p.bnd_in * p.n_sel + c0 + 1] : __longlong_as_double((long long)nyi[c0 + 1]));
      }
      const int g0 = min(ep, es);
      const double yh = scale2k(nyv, g0 - ep), xh = scale2k(lm, g0 - es);
      const double tau = __dadd_rn(__dmul_rn(beta, P.cS[p.I]), __dmul_rn(ab, P.cT[p.I]));
      const int en = g0 + protect_update(yh, tau, xh);
      sx = en - es;
      if (t == 0 && w0) {
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
      if (valid && r >= rlo && r < rhi) {
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
  if (valid && p.do_update && w0) {
    for (int r = nt + t; r < p.nks * kBK; r += 4) {
      const long long off = (long long)(r / kBK) * (kBN * kBK) + (long long)((r % kBK) >> 2) * (kBN * 4) + (r & 3);
      Wc[off] = 0.0;
      Wc[off + half] = 0.0;
    }
  }
  // W is read next by bulk copies (the async proxy): order the generic writes before them
  asm volatile("fence.proxy.async.global;" ::: "memory");
  ZZ_TR(160 + w);
}

// NW warps per CTA: W3<G>::n (12 or 16) in general; 8 with G producers (one or two tasks per
// CTA, up to 255 registers per thread: no spills in the solving warp)
template <int G, bool TEAMS, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_diag3(Diag2Params p) {
  constexpr int kW3 = NW;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int nt = p.nt;
  ZZ_TR0();
  const int W = TEAMS ? p.team_w : 1, nteams = kW3 / W;
  const int nblk = (nt + 7) / 8;
  const size_t tb = a16(team_bytes(W, nblk));
  Sm3 sm = carve3(smraw, nt, nteams, tb, kW3);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tix = warp / W;
  Team tm;
  tm.W = W;
  tm.w = warp % W;
  tm.bar = 1 + tix;
  tm.pub = reinterpret_cast<Pub*>(sm.teams + tb * tix);
  const int nslot = (W == 1) ? 1 : nblk;
  tm.pslab = sm.ptab + 576 * warp;
  tm.red0 = reinterpret_cast<double*>(tm.pub + nslot);
  tm.red1 = tm.red0 + 8 * W;
  tm.red2 = tm.red1 + 16 * W;
  GRing ring;
  ring.slot = nullptr;
  ring.ns = kGSlots;
  ring.ready = reinterpret_cast<int*>(sm.gring + kGSlots * kGSlotBytes);
  ring.done = ring.ready + kGSlots;
  if (!TEAMS && threadIdx.x < 2 * kGSlots) ring.ready[threadIdx.x] = 0;   // (ready and done)
  for (int i = tm.w * 32 + lane; i < nslot; i += 32 * W) {
    tm.pub[i].flag = 0;
    tm.pub[i].cnt = 0;
  }
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
  if (threadIdx.x <= nblk) {
    const int b = threadIdx.x;
    int v = 8 * b;
    if (v >= nt) v = nt;
    else if (b > 0 && sm.fl[v] == kRowBot2) v -= 1;
    sm.bs[b] = v;
  }
#ifdef ZZ_VARIANT_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) g_trace[181] = clock64();
#endif
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
    // ||S_bb||_inf, ||T_bb||_inf of the block's diagonal sub-block (gsolve_block's condition
    // check): lane i < e0 - s0 sums row s0 + i over the block's columns
    double bs_ = 0.0, bt_ = 0.0;
    if (lane < e0 - s0) {
      const int i = s0 + lane;
      for (int l = max(s0, i - 1); l < e0; ++l) {
        const double2 v = sm.ST[poff3(l) + i];
        bs_ += fabs(v.x);
        bt_ += fabs(v.y);
      }
    }
    for (int o = 16; o; o >>= 1) {
      bs_ = fmax(bs_, __shfl_xor_sync(0xffffffffu, bs_, o));
      bt_ = fmax(bt_, __shfl_xor_sync(0xffffffffu, bt_, o));
    }
    if (lane == 0) sm.bn[b] = make_double2(bs_, bt_);
  }
  __syncthreads();
#ifdef ZZ_VARIANT_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) g_trace[182] = clock64();
#endif
  // ---- tasks (4 complex pairs or 8 real columns), one per team of W warps ----
  const int npt = (p.n_pair + p.cpt / 2 - 1) / (p.cpt / 2), nrt = (p.n_real + p.cpt - 1) / p.cpt;
  // CTA-fastest assignment: with few tasks every SM gets one before any SM gets two
  // (measured: contiguous per-CTA task ranges were slower, pair tasks being heavier)
  if (!TEAMS && p.gprod && npt + nrt <= 2 * (int)gridDim.x) {
    // one or two tasks per CTA: a task's first warp solves it, its other warps form its rows
    // of G ahead of it (tasks CTA-fastest, as below)
    const int tpc = (npt + nrt <= (int)gridDim.x) ? 1 : 2, wpt = kW3 / tpc;
    const int ti = warp / wpt, role = warp % wpt;
    const int task = ti * gridDim.x + blockIdx.x;
    if (task >= npt + nrt) return;
    ring.ns = kGSlots / tpc;
    ring.slot = reinterpret_cast<double*>(sm.gring) + ti * ring.ns * (kGVals * 32);
    ring.ready += ti * ring.ns;
    ring.done += ti * ring.ns;
    tm.gen = task + 1;
    if (role == 0) {
      if (task < npt) solve_task<G, true, TEAMS>(p, sm, nblk, task, lane, tm, ring);
      else solve_task<G, false, TEAMS>(p, sm, nblk, task - npt, lane, tm, ring);
    } else {
      if (task < npt) gproduce_task<true>(p, sm, nblk, task, lane, role - 1, wpt - 1, sm.ptab + 576 * warp, ring);
      else gproduce_task<false>(p, sm, nblk, task - npt, lane, role - 1, wpt - 1, sm.ptab + 576 * warp, ring);
    }
    return;
  }
  for (int task = tix * gridDim.x + blockIdx.x; task < npt + nrt; task += gridDim.x * nteams) {
    tm.gen = task + 1;
    if (task < npt) solve_task<G, true, TEAMS>(p, sm, nblk, task, lane, tm, ring);
    else solve_task<G, false, TEAMS>(p, sm, nblk, task - npt, lane, tm, ring);
  }
}

int g_sms3 = 0;

}  // namespace

size_t diag3_smem_bytes(int nt) {
  const int nblk = (nt + 7) / 8;
  return smem3(nt, 12, a16(team_bytes(1, nblk)), 12);
}

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
  const int nblk = (p.nt + 7) / 8;
  const bool small = p.nt <= 64;
  const int nw = small ? W3<8>::n : W3<16>::n;
  // team size W (a divisor of the CTA's warps): as many warps per task as keep every task in
  // one wave over the SMs -- the chain of a task then runs on W warps (results do not
  // depend on W, see solve_task); limited by the shared memory of the teams
  // Automatic: one warp per task.  Measured (C2, tools/time_team.py): teams are slower --
  // the hand-off of a block between warps costs about as much as the DMMA updates it spreads
  // (DESIGN.md s.6 "Teams"); zz_set_diag_team(W) selects them explicitly.
  int W = 1;
  if (p.team_w > 0) {
    W = p.team_w;
    if (nw % W || smem3(p.nt, nw / W, a16(team_bytes(W, nblk)), nw) > 227 * 1024) W = 1;
  } else if (p.team_w < 0 && !p.pack) {
    const int cand[5] = {small ? 16 : 12, small ? 8 : 6, 4, small ? 2 : 3, 1};
    for (int i = 0; i < 5; ++i) {
      const int Wc = cand[i];
      if ((long long)tasks * Wc > (long long)g_sms3 * nw) continue;
      if (smem3(p.nt, nw / Wc, a16(team_bytes(Wc, nblk)), nw) > 227 * 1024) continue;
      W = Wc;
      break;
    }
  }
  p.team_w = W;
  // default (team_w 0): with one task per CTA the idle warps produce the rows of G
  p.gprod = (pin.team_w == 0 && W == 1 && tasks <= 2 * g_sms3) ? 1 : 0;
#ifdef ZZ_VARIANT_NW8
  const int nwl = 8;
#else
  const int nwl = p.gprod ? 8 : nw;   // warps per CTA of this launch
#endif
  const int per_cta = nwl / W;        // tasks per CTA at a time
  const size_t smem = smem3(p.nt, per_cta, a16(team_bytes(W, nblk)), nwl);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e;
  // pack: as few CTAs as the tasks need (one task per team), leaving the other SMs to a
  // concurrent update (lookahead); otherwise one task per CTA first (lowest latency alone)
  int grid = p.pack ? std::min(g_sms3, (tasks + per_cta - 1) / per_cta) : (tasks < g_sms3 ? tasks : g_sms3);
  if (p.gprod && p.pack) grid = (tasks + 1) / 2;   // lookahead: two tasks (and their producers) per CTA
#define ZZ_LAUNCH3(GG, TT, NN)                                                                           \
  do {                                                                                                  \
    e = cudaFuncSetAttribute(k_diag3<GG, TT, NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024); \
    if (e != cudaSuccess) return e;                                                                     \
    k_diag3<GG, TT, NN><<<grid, NN * 32, smem, st>>>(p);                                                \
  } while (0)
  if (small) {
    if (W > 1) ZZ_LAUNCH3(8, true, W3<8>::n);
    else if (p.gprod || nwl == 8) ZZ_LAUNCH3(8, false, 8);
    else ZZ_LAUNCH3(8, false, W3<8>::n);
  } else {
    if (W > 1) ZZ_LAUNCH3(16, true, W3<16>::n);
    else if (p.gprod || nwl == 8) ZZ_LAUNCH3(16, false, 8);
    else ZZ_LAUNCH3(16, false, W3<16>::n);
  }
#undef ZZ_LAUNCH3
  return cudaGetLastError();
}

}  // namespace zz

#ifdef ZZ_VARIANT_TRACE
extern "C" int zz_trace_get(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, zz::g_trace, sizeof(long long) * 512);
}
#endif
