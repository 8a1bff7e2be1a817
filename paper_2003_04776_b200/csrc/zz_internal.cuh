// zz_internal.cuh -- internal declarations of the B200 (sm_100a) robust eigenvector path.
// Product code: never includes or links anything under oracle/.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include <nccl.h>

namespace zz {

// ------------------------------------------------------------------------------------
// Constants (readings R1, R8): Omega = 2^1023, u = 2^-53, smlnum = 2^-969.
// ------------------------------------------------------------------------------------
constexpr double kOmega = 0x1p1023;
constexpr double kU = 0x1p-53;
constexpr double kSmlnum = 0x1p-969;

// GEMM (robust update) tiling, shared by the update kernel and the W writer of the
// diagonal solve (W is stored in the update kernel's shared-memory stage order).
constexpr int kBM = 128;   // rows of X per CTA tile
constexpr int kBN = 64;    // eigenvector columns per CTA tile
constexpr int kBK = 16;    // K chunk (columns of S or T per pipeline stage)
constexpr int kMaxMB = 160;

// column kinds
enum : int { kReal = 0, kPairFirst = 1, kPairSecond = 2, kIndefinite = 3 };
// row flags inside the diagonal structure
enum : int { kRow1x1 = 0, kRowTop2 = 1, kRowBot2 = 2 };

// ------------------------------------------------------------------------------------
// Overflow protection.  Definitions of DESIGN.md R4/R5; written with
// explicit round-to-nearest intrinsics so that no contraction changes the decision.
// ------------------------------------------------------------------------------------
// ProtectUpdate(y, t, x) -> e with 2^e (y + t x) <= Omega
__device__ __forceinline__ int protect_update(double y, double t, double x) {
  double s = __dadd_rn(__dmul_rn(y, 0x1p-1023), __dmul_rn(__dmul_rn(t, 0x1p-512), __dmul_rn(x, 0x1p-511)));
  if (s <= 0.5) return 0;
  int k;
  double f = frexp(s, &k);
  int c = (f == 0.5) ? k - 1 : k;
  return -c - 1;
}
// ProtectDivision(b, t) -> e with 2^e b <= t Omega
__device__ __forceinline__ int protect_division(double b, double t) {
  if (t >= 1.0 || b <= __dmul_rn(t, kOmega)) return 0;
  double r = __ddiv_rn(__dmul_rn(t, kOmega), b);
  int k;
  frexp(r, &k);
  return k - 2;
}

// ------------------------------------------------------------------------------------
// Host-side plan of one call (built by zz_api.cu, copied to the device).
// ------------------------------------------------------------------------------------
struct DevPlan {
  // per output column c (n_sel)
  double* col_a;
  double* col_b;
  double* col_beta;
  double* logmax;     // L_c = log2(max measure of the stored column before normalisation) - e_c
  int* col_kind;
  int* col_r;         // last row of the column's diagonal block
  int* col_tile;      // tile index of that block
  // per item (selected block) t
  int* item_col;      // first output column
  int* real_items;    // columns of the selected real eigenvalues (ascending)
  int* pair_items;    // first columns of the selected complex pairs (ascending)
  // per tile
  int* tile_start;    // M+1
  // per row
  signed char* row_flag;
  int* row_tile;
  // per block (all blocks) for the pair kernel
  int* blk_start;
  int* blk_size;
  int* blk_col;       // first output column or -1
  // robustness state
  int* e_pend;        // per column: exponent of the pending (not yet solved) rows
  int* sY;            // per column: exponent shift of the pending rows at this step
  int* e_prev;        // per column: pending exponent before a group's first decision
  int* e_grp;         // (kMaxGroup - 1) x n_sel: exponent of each earlier step's W in a group
  double* nYb;        // per column: upper bound of |pending| after a group's update (lookahead)
  unsigned long long* nY;   // kMaxGroup x n_sel: max |pending| (double bits), 2 alternating + band buffers
  int* e_seg;         // M x n_sel: exponent of each solved segment
  double* nrm_seg;    // M x n_sel: max(|Re|,|Im|) of the segment
  double* nrmh_seg;   // M x n_sel: max(|x|/2 + |y|/2) (pair) or |x|/2 (real)
  double* cS;         // M: infinity norm of the S panel above tile I
  double* cT;
  double* W;          // update B operand, blocked [ntile][kc][BK/4][BN][4]
  int* status;        // [0]: first bad 2x2 row (1-based) or 0; [1]: nonfinite flag;
                      // [2]: indefinite count; [3]: maxabs bits lo; ...
  unsigned long long* maxabs;  // [0] S, [1] T (double bits)
};

struct DiagParams {
  int I, t0, nt;
  int item_begin, n_items;
  int tip_col_end;   // columns < tip_col_end (and >= first active) are tips
  int do_update;
  int nks;           // K chunks per part (S or T) in W for this step
  int n_sel;
  const double* S; long long lds;
  const double* T; long long ldt;
  double* X; long long ldx;
  DevPlan P;
  int nY_in;         // which nY buffer holds the pending max of this step
};

// steps per group of the wavefront (zz_set_fusion): one update per group of this many steps
constexpr int kMaxGroup = 6;

struct UpdParams {
  int rows;          // ts_I: rows [0, rows) are updated
  int max_row;       // ts_{I-1}: rows [0, max_row) form the next pending region
  int t0;            // first column of tile I in S and T
  int nks;           // K chunks per part
  int c_begin;       // first active column (cs_I)
  int first_end;     // columns < first_end start from C = 0 (cs_{I+1})
  int n_sel;
  int ntile0;        // first N tile index (c_begin / BN)
  int ntile_end;     // one past the last 64-column N tile (set by the launcher)
  double* X; long long ldx;
  const double* W;
  const int* sY;
  unsigned long long* nY_out;
  int vec;           // 16-byte aligned X access possible
  int row_lo;        // rows [row_lo, rows) are updated (0, or a tile start for the thin update)
  // further K segments of a step group's update (MODE 1): S/T columns of tile xt0[e]
  // (xnks[e] chunks per part) against xW[e], in this order after (t0, nks, W)
  int nxs;
  int xt0[kMaxGroup - 1], xnks[kMaxGroup - 1];
  const double* xW[kMaxGroup - 1];
};

// Diagonal solve with 8 columns per warp (zz_diag3.cu): tiles of at most kDiag2MaxNT rows.
constexpr int kDiag2MaxNT = 128;

struct Diag2Params {
  int I, t0, nt;
  int n_real, n_pair;      // active real columns / complex pairs at this step
  const int* real_items;   // their columns (ascending), already offset to the active suffix
  const int* pair_items;   // first columns of the active pairs
  int tip_col_end;         // columns < tip_col_end have their eigenvalue block in tile I
  int do_update;
  int nks;
  int n_sel;
  const double* S; long long lds;
  const double* T; long long ldt;
  double* X; long long ldx;
  DevPlan P;
  int nY_in;
  int bnd_in;        // lookahead: the set of recorded bounds (nYb) this step reads; a group's last
                     // decision writes the other set
  int cpt;                 // columns per warp task (set by launch_diag3)
  double* Wout;            // where this step's B operand W goes
  // second step of a fused pair (I, J = I - 1): the update of the rows above tile J is done
  // once with both tiles; tile I's step left its W in Wprev (nks_prev chunks per part)
  // role in a step group (I, I-1, ..., L) whose rows above tile L get one update with all
  // the group's tiles: fused = 0 a single step or the group's first (grp_slot = 0, it zeroes
  // n_band_reset band buffers nY[2..]); 2 a middle step (a band decision for the group's rows
  // below it, band maximum in nY[band_in], exponent to e_grp[grp_slot]); 3 the last step L
  // (the decision for the rows above L with the n_prev earlier steps' terms)
  int fused;
  int grp_slot;            // -1: not recorded
  int n_band_reset;
  int band_in;
  int n_prev;
  int prev_I[kMaxGroup - 1], prev_cs[kMaxGroup - 1], prev_nks[kMaxGroup - 1];
  double* prev_W[kMaxGroup - 1];
  int zero_pend_end;       // columns < zero_pend_end (tips of the group) have no pending rows
  // lookahead: a group's first step takes the pending bound nYb recorded by the previous
  // group's last step (use_bound) instead of the measured maximum; the last step records it
  int use_bound, record_bound;
  int pack;                // launch as few CTAs as the tasks need (lookahead)
  int team_w;              // warps per task (0: chosen by launch_diag3; results do not depend on it)
  int gprod;               // one task per CTA: the idle warps form the rows of G (set by launch_diag3)
};

// launchers (zz_kernels.cu / zz_update.cu / zz_diag.cu)
cudaError_t launch_diag3(const Diag2Params& p, cudaStream_t st);
size_t diag3_smem_bytes(int nt);
cudaError_t launch_subdiag(const double* S, long long lds, int m, double* sub, cudaStream_t st);
cudaError_t launch_pairs(const double* S, long long lds, const double* T, long long ldt, int p0, int nblk,
                         const DevPlan& P, cudaStream_t st);
cudaError_t launch_maxabs(const double* S, long long lds, const double* T, long long ldt, int m,
                          unsigned long long* out, cudaStream_t st);
cudaError_t launch_rowsum_max(const double* A, long long lda, int m, unsigned long long* out,
                              cudaStream_t st);
cudaError_t launch_scale_copy(const double* A, long long lda, int m, int k, double* B, long long ldb,
                              cudaStream_t st);
cudaError_t launch_panel_norms(const double* S, long long lds, const double* T, long long ldt, int M,
                               const int* tile_start_host, const DevPlan& P, cudaStream_t st, int J0, int nJ);
cudaError_t launch_diag(const DiagParams& p, cudaStream_t st);
cudaError_t launch_normalize(int m, int n_sel, int M, double* X, long long ldx, int* col_scale_exp,
                             const DevPlan& P, int* exp_tmp, double* rec_tmp, cudaStream_t st);
cudaError_t launch_update(const CUtensorMap* tmS, const CUtensorMap* tmT, const UpdParams& p,
                          int n_mtiles, int n_ntiles, cudaStream_t st);
size_t diag_smem_bytes(int nt);
// zz_back.cu: LAPACK normalisation of the back-transformed columns (xTGEVC HOWMNY='B')
cudaError_t launch_back_gemm(const CUtensorMap* tmV, const double* X, long long ldx, int m, int n_sel,
                             const int* nkc, const long long* woff, int max_nkc, double* Xp, double* W,
                             long long ldw, unsigned long long* colmax, cudaStream_t st);
cudaError_t launch_back_norm(double* W, long long ldw, int m, int n_sel, const int* col_kind,
                             const unsigned long long* colmax, cudaStream_t st);
// zz_left.cu: left eigenvectors through the flipped pencil S' = J S^T J, T' = J T^T J
cudaError_t launch_flip_transpose(const double* A, long long lda, double* B, long long ldb, int m, cudaStream_t st);
cudaError_t launch_left_gather(const double* Xf, long long ldxf, double* Y, long long ldy, int m, int n_sel,
                               const int* kind_f, const int* ef, int* ey, cudaStream_t st);

// zz_comm.cu: NCCL (dlopen'ed at first use; nullptr if unavailable) and the gather kernels
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*);
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*commDestroy)(ncclComm_t);
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*groupStart)();
  ncclResult_t (*groupEnd)();
};
const NcclApi* nccl_api();
// eigenvalue blocks are owned in groups of kShardNB rows, cyclically over the ranks
// (block of first row j -> shard (j / kShardNB) mod P)
constexpr int kShardNB = 64;
cudaError_t launch_shard_pack(const double* X, long long ldx, const int* cse, int n, const long long* off,
                              const int* h, double* buf, int* ebuf, cudaStream_t st);
cudaError_t launch_shard_unpack(const unsigned char* buf, int ne, const long long* boff, const long long* beoff,
                                const int* h, const int* g, int m, double* X, long long ldx, int* cse,
                                cudaStream_t st);

}  // namespace zz
