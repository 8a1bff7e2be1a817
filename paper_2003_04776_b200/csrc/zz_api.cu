// zz_api.cu -- host runtime and C ABI (include/zz.h) of the B200 robust eigenvector path.
//
// The runtime owns a per-thread context (device, stream, tile size, workspace), builds the
// plan of one call on the host (block structure, tile partition, selection, column and
// item maps -- PAPER.md:128-132, 268-273), and drives the bottom-up wavefront over tile
// rows (Algorithm 1): for I = M-1..0, the robust diagonal solve of tile
// row I for every active eigenvector (tips for the blocks inside tile I), then one fused
// robust update of all rows above it.  Two host synchronisations happen before the
// wavefront (structure, then pair/norm status); none inside it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "../../include/zz.h"
#include "zz_internal.cuh"

using namespace zz;

namespace {

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = bytes + bytes / 8 + 256;
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) { p = nullptr; return e; }
    cap = want;
    return cudaSuccess;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Context {
  int device = -1;
  cudaStream_t stream = nullptr;
  int mb = 0;
  int timing = 0;
  // step groups of the wavefront: k consecutive steps share one update (zz_set_fusion)
  int fusion = 4;
  bool fusion_explicit = false;   // zz_set_fusion was called (zz_ztgevc's default depends on m)
  Buf zw;                         // zz_ztgevc's workspace (kept between calls)
  // CUDA graph of the wavefront (zz_set_graphs): the last captured plan and its replayable exec
  int graphs = 1;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap = nullptr;   // capture stream
  uint64_t gkey = 0;
  int g_nupd = 0, g_nfused = 0, g_launches = 0;
  // lookahead (zz_set_lookahead): the chain of solves runs on a high-priority stream beside
  // the bulk of the previous group's update (DESIGN.md s.6 "Lookahead"); 1 = automatic
  int lookahead = 1;
  // warps per diagonal-solve task (zz_set_diag_team): 0 = automatic
  int diag_team = 0;
  cudaStream_t hi = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::vector<cudaEvent_t> ev_la;
  zz_info_t info;
  EncodeTiledFn encode = nullptr;
  // workspace
  Buf sub, colf, coli, items, tiles, rows, blks, state, seg, norms, W, status, tmp, Sc, Tc, Xi, egrp;
  Buf Wx[kMaxGroup - 1];   // the W operands of a step group's later steps
  Buf Wy[kMaxGroup];       // second set (lookahead: groups alternate between the sets)
  Buf sYb, nYb;            // second sY set; per-column bound of the pending rows (lookahead)
  Buf hS, hT, hX, hE;  // device staging of zz_tgevc_host
  Buf Xb;              // X of zz_tgevc_back / the flipped solve of zz_tgevc_left
  Buf Xp, btab, Vc;    // zz_tgevc_back: tile-packed X, tile tables + column maxima, aligned V
  // communicator (zz_init with an id) and the shard of this rank
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  int shard_p = 0, shard_P = 1;   // zz_set_shard: one-GPU emulation of a rank's share
  Buf Sw, Tw, Xloc, Eloc, bbuf, sendb, recvb, gtab, subd;
  Buf Sl, Tl, El;      // zz_tgevc_left: S' = J S^T J, T' = J T^T J, exponents
  std::vector<int> last_col_r;            // r_c of the last call's columns (host)
  std::vector<cudaEvent_t> ev;
  std::vector<cudaEvent_t> ev_copy;       // per-panel arrival events of zz_tgevc_host
  cudaStream_t copy = nullptr;            // host-to-device copy stream of zz_tgevc_host
  cudaEvent_t e_copy = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr;
  ~Context() {}
  void release() {
    Buf* all[] = {&sub, &colf, &coli, &items, &tiles, &rows, &blks, &state, &seg, &norms, &W,
                  &status, &tmp, &Sc, &Tc, &Xi, &egrp, &hS, &hT, &hX, &hE};
    for (Buf* b : all) b->release();
    zw.release();
    for (Buf& b : Wx) b.release();
    for (Buf& b : Wy) b.release();
    sYb.release();
    nYb.release();
    for (cudaEvent_t e : ev_la) cudaEventDestroy(e);
    ev_la.clear();
    if (ev_in) { cudaEventDestroy(ev_in); cudaEventDestroy(ev_out); }
    ev_in = ev_out = nullptr;
    if (gexec) cudaGraphExecDestroy(gexec);
    gexec = nullptr;
    gkey = 0;
    if (cap) cudaStreamDestroy(cap);
    cap = nullptr;
    if (hi) cudaStreamDestroy(hi);
    hi = nullptr;
    Xb.release();
    Xp.release();
    btab.release();
    Vc.release();
    Buf* cb[] = {&Sw, &Tw, &Xloc, &Eloc, &bbuf, &sendb, &recvb, &gtab, &subd};
    for (Buf* b : cb) b->release();
    if (comm) {
      if (const NcclApi* api = nccl_api()) api->commDestroy(comm);
      comm = nullptr;
    }
    Sl.release();
    Tl.release();
    El.release();
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    ev.clear();
    for (cudaEvent_t e : ev_copy) cudaEventDestroy(e);
    ev_copy.clear();
    if (copy) cudaStreamDestroy(copy);
    copy = nullptr;
    if (e_copy) cudaEventDestroy(e_copy);
    e_copy = nullptr;
    if (e0) { cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2); cudaEventDestroy(e3); }
    e0 = e1 = e2 = e3 = nullptr;
  }
};

thread_local Context* g_ctx = nullptr;

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t _e = (x);                                                         \
    if (_e != cudaSuccess) {                                                      \
      if (getenv("ZZ_DEBUG_SYNC"))                                                \
        fprintf(stderr, "zz: %s (line %d): %s\n", #x, __LINE__, cudaGetErrorString(_e)); \
      return map_err(_e);                                                         \
    }                                                                             \
  } while (0)

// NVTX ranges around the phases of a call (header-only NVTX v3: no library, no cost when
// no tool is attached)
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};

int map_err(cudaError_t e) {
  if (e == cudaErrorMemoryAllocation) return ZZ_ERR_NOMEM;
  return ZZ_ERR_CUDA;
}

int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// Tile partition (reading R12): nominal boundaries every mb
// rows; a boundary that would split a 2x2 block (i.e. fall on the block's second row)
// moves up one row, so that every tile has at most mb rows.
int partition_host(int m, const std::vector<char>& two_bot, int mb, std::vector<int>& ts) {
  ts.clear();
  ts.push_back(0);
  int s = 0;
  while (s < m) {
    int nx = s + mb;
    if (nx >= m) { nx = m; }
    else if (two_bot[nx]) nx -= 1;
    ts.push_back(nx);
    s = nx;
  }
  return (int)ts.size() - 1;
}

// blocks from the subdiagonal: returns nb or -105
int blocks_host(int m, const double* sub, std::vector<int>& bs, std::vector<int>& bz) {
  bs.clear();
  bz.clear();
  int j = 0;
  while (j < m) {
    bool two = (j + 1 < m) && sub[j] != 0.0;
    if (two && j + 2 < m && sub[j + 1] != 0.0) return ZZ_ERR_OVERLAP;
    bs.push_back(j);
    bz.push_back(two ? 2 : 1);
    j += two ? 2 : 1;
  }
  return (int)bs.size();
}

int tile_of(int mb_user) { return mb_user > 0 ? mb_user : 128; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int make_map(Context* c, CUtensorMap* tm, const double* A, long long lda, int m) {
  if (!c->encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return ZZ_ERR_CUDA;
    c->encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)m};
  cuuint64_t strides[1] = {(cuuint64_t)lda * 8};
  cuuint32_t box[2] = {8u, (cuuint32_t)kBK};   // 8 rows x 16 columns per TMA box
  cuuint32_t estr[2] = {1, 1};
  CUresult r = c->encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)A, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : ZZ_ERR_CUDA;
}

// Staged panels: S and T arrive tile column by tile column in the order the wavefront
// consumes them (tile columns M-1 .. 0, upper part and subdiagonal only) on a separate
// stream -- from host memory (zz_tgevc_host) and/or by an NCCL broadcast from rank 0 (the
// collective zz_tgevc); step I waits for panel I only, so the transfers
// overlap the solve.  The pairs and panel norms of panel I are computed when it lands and
// the status checks are deferred to the end of the wavefront.
struct Feed {
  const double* Sh = nullptr;  // host source of S, T (zz_tgevc_host), or null
  long long ldsh = 0;
  const double* Th = nullptr;
  long long ldth = 0;
  const double* sub = nullptr; // host copy of the subdiagonal (m-1 entries), if known
  cudaStream_t copy = nullptr; // stream of the transfers
  std::vector<cudaEvent_t>* ev = nullptr;
  ncclComm_t comm = nullptr;   // NCCL broadcast of the panels from rank 0
  const NcclApi* api = nullptr;
  bool root = true;            // this rank sends (its S, T are complete: Ssrc, Tsrc)
  const double* Ssrc = nullptr;  // root: the device S, T the panels are packed from
  long long ldss = 0;
  const double* Tsrc = nullptr;
  long long ldts = 0;
  double* bbuf = nullptr;      // contiguous staging of one panel pair (comm only)
  bool wait = true;            // the steps wait for the panel events
};

// The solve on device pointers.  S/T are const; X, cse written.
int tgevc_device(Context* c, int m, const double* S, long long lds, const double* T, long long ldt,
                 const int* select, double* X, long long ldx, int* cse, const Feed* hs = nullptr) {
  cudaStream_t st = c->stream;
  // the caller's X: the recomputations below (pre-scale of the host path, lookahead redo)
  // start again from it, not from the aligned internal buffer X may be swapped for
  double* const X_call = X;
  const long long ldx_call = ldx;
  zz_info_t info;
  memset(&info, 0, sizeof(info));
  info.m = m;
  const int mb = tile_of(c->mb);
  info.mb = mb;
  if (!c->e0) {
    cudaEventCreate(&c->e0); cudaEventCreate(&c->e1); cudaEventCreate(&c->e2); cudaEventCreate(&c->e3);
  }
  Range r_call("zz_tgevc");
  CK(cudaEventRecord(c->e0, st));
  int launches = 0;
  // ---- a1: structure scan (one host sync; none when S is on the host) ----
  std::vector<double> sub((size_t)std::max(m - 1, 1), 0.0);
  if (hs && hs->sub) {
    for (int j = 0; j + 1 < m; ++j) sub[j] = hs->sub[j];
  } else if (hs && hs->Sh) {
    for (int j = 0; j + 1 < m; ++j) sub[j] = hs->Sh[(size_t)j * hs->ldsh + j + 1];
  } else {
    CK(c->sub.ensure(sizeof(double) * (size_t)std::max(m, 1)));
    CK(launch_subdiag(S, lds, m, c->sub.as<double>(), st));
    launches += (m > 1);
    if (m > 1) CK(cudaMemcpyAsync(sub.data(), c->sub.p, sizeof(double) * (m - 1), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  std::vector<int> bs, bz;
  int nb = blocks_host(m, sub.data(), bs, bz);
  if (nb < 0) return nb;
  std::vector<char> two_bot((size_t)m + 1, 0);
  std::vector<signed char> row_flag((size_t)m, kRow1x1);
  for (int p = 0; p < nb; ++p)
    if (bz[p] == 2) {
      two_bot[bs[p] + 1] = 1;
      row_flag[bs[p]] = kRowTop2;
      row_flag[bs[p] + 1] = kRowBot2;
    }
  std::vector<int> ts;
  const int M = partition_host(m, two_bot, mb, ts);
  info.n_tiles = M;
  std::vector<int> row_tile((size_t)m);
  for (int I = 0; I < M; ++I)
    for (int i = ts[I]; i < ts[I + 1]; ++i) row_tile[i] = I;
  // selection, packed columns, items (xTGEVC HOWMNY='S')
  std::vector<int> blk_col((size_t)nb, -1), item_col, item_tile, item_two;
  std::vector<int> col_r, col_tile;
  int n_sel = 0;
  for (int p = 0; p < nb; ++p) {
    int j = bs[p];
    bool sel = !select || select[j] || (bz[p] == 2 && select[j + 1]);
    if (!sel) continue;
    blk_col[p] = n_sel;
    item_col.push_back(n_sel);
    item_tile.push_back(row_tile[j]);
    item_two.push_back(bz[p] == 2);
    for (int q = 0; q < bz[p]; ++q) {
      col_r.push_back(j + bz[p] - 1);
      col_tile.push_back(row_tile[j]);
    }
    n_sel += bz[p];
  }
  info.n_sel = n_sel;
  c->last_col_r = col_r;
  const int n_items = (int)item_col.size();
  std::vector<int> tile_item((size_t)M + 1, n_items), cs((size_t)M + 1, n_sel);
  for (int I = M - 1; I >= 0; --I) {
    int t = tile_item[I + 1];
    while (t > 0 && item_tile[t - 1] >= I) --t;
    tile_item[I] = t;
    cs[I] = (t < n_items) ? item_col[t] : n_sel;
  }
  // per-kind item lists (thread-per-eigenvector diagonal solve): ascending columns, and per
  // tile row I the first entry whose eigenvalue block lies in a tile >= I
  std::vector<int> real_list, pair_list, real_tile, pair_tile;
  for (int t = 0; t < n_items; ++t) {
    if (item_two[t]) { pair_list.push_back(item_col[t]); pair_tile.push_back(item_tile[t]); }
    else { real_list.push_back(item_col[t]); real_tile.push_back(item_tile[t]); }
  }
  std::vector<int> rbeg((size_t)M + 1), pbeg((size_t)M + 1);
  for (int I = 0; I <= M; ++I) {
    rbeg[I] = (int)(std::lower_bound(real_tile.begin(), real_tile.end(), I) - real_tile.begin());
    pbeg[I] = (int)(std::lower_bound(pair_tile.begin(), pair_tile.end(), I) - pair_tile.begin());
  }
  // diagonal-solve kernel: k_diag3 (8 columns per warp, DMMA in-tile updates) for tiles of
  // <= 128 rows, k_diag (warp per eigenvector) above
  // ---- workspace ----
  const int n = std::max(n_sel, 1);
  const int nks_max = ceil_div(mb, kBK);
  const int n_ntiles_all = ceil_div(n, kBN);
  CK(c->colf.ensure(sizeof(double) * 4 * (size_t)n));
  CK(c->coli.ensure(sizeof(int) * 9 * (size_t)n));
  CK(c->items.ensure(sizeof(int) * 2 * (size_t)std::max(n_items, 1)));
  CK(c->tiles.ensure(sizeof(int) * (size_t)(M + 1)));
  CK(c->rows.ensure((sizeof(int) + 1) * (size_t)m + 16));
  CK(c->blks.ensure(sizeof(int) * 3 * (size_t)nb));
  CK(c->state.ensure(sizeof(unsigned long long) * kMaxGroup * (size_t)n));
  CK(c->egrp.ensure(sizeof(int) * (kMaxGroup - 1) * (size_t)n));
  CK(c->seg.ensure((sizeof(int) + 2 * sizeof(double)) * (size_t)M * n));
  CK(c->norms.ensure(sizeof(double) * 4 * (size_t)M));
  CK(c->W.ensure(sizeof(double) * (size_t)n_ntiles_all * 2 * nks_max * kBN * kBK));
  CK(c->status.ensure(sizeof(int) * 16 + sizeof(unsigned long long) * 2));
  CK(c->tmp.ensure((sizeof(int) + sizeof(double)) * (size_t)n + 16));
  DevPlan P;
  P.col_a = c->colf.as<double>();
  P.col_b = P.col_a + n;
  P.col_beta = P.col_b + n;
  P.logmax = P.col_beta + n;
  P.col_kind = c->coli.as<int>();
  P.col_r = P.col_kind + n;
  P.col_tile = P.col_r + n;
  P.e_pend = P.col_tile + n;
  P.sY = P.e_pend + n;
  P.e_prev = P.sY + n;
  P.e_grp = c->egrp.as<int>();
  CK(c->nYb.ensure(sizeof(double) * 2 * (size_t)n));   // two sets: read / written by a group's last decision
  P.nYb = c->nYb.as<double>();
  P.item_col = c->items.as<int>();
  P.real_items = P.item_col + n_items;
  P.pair_items = P.real_items + real_list.size();
  P.tile_start = c->tiles.as<int>();
  P.row_tile = c->rows.as<int>();
  P.row_flag = reinterpret_cast<signed char*>(P.row_tile + m);
  P.blk_start = c->blks.as<int>();
  P.blk_size = P.blk_start + nb;
  P.blk_col = P.blk_size + nb;
  P.nY = c->state.as<unsigned long long>();
  {
    // e_seg (int) first, then the two double arrays at an 8-byte aligned offset
    size_t off = (sizeof(int) * (size_t)M * n + 7) / 8 * 8;
    P.e_seg = c->seg.as<int>();
    P.nrm_seg = reinterpret_cast<double*>(c->seg.as<char>() + off);
  }
  P.nrmh_seg = P.nrm_seg + (size_t)M * n;
  P.cS = c->norms.as<double>();
  P.cT = P.cS + M;
  P.W = c->W.as<double>();
  P.status = c->status.as<int>();
  P.maxabs = reinterpret_cast<unsigned long long*>(P.status + 16);
  int* exp_tmp = c->tmp.as<int>();
  double* rec_tmp = reinterpret_cast<double*>(c->tmp.as<char>() + ((sizeof(int) * (size_t)n + 15) / 16 * 16));
  // ---- upload the plan ----
  if (n_sel > 0) {
    CK(cudaMemcpyAsync(P.col_r, col_r.data(), sizeof(int) * n_sel, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(P.col_tile, col_tile.data(), sizeof(int) * n_sel, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(P.item_col, item_col.data(), sizeof(int) * n_items, cudaMemcpyHostToDevice, st));
    if (!real_list.empty())
      CK(cudaMemcpyAsync(P.real_items, real_list.data(), sizeof(int) * real_list.size(), cudaMemcpyHostToDevice, st));
    if (!pair_list.empty())
      CK(cudaMemcpyAsync(P.pair_items, pair_list.data(), sizeof(int) * pair_list.size(), cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemcpyAsync(P.tile_start, ts.data(), sizeof(int) * (M + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(P.row_tile, row_tile.data(), sizeof(int) * m, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(P.row_flag, row_flag.data(), m, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(P.blk_start, bs.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(P.blk_size, bz.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(P.blk_col, blk_col.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st));
  {
    int init[16] = {0x7fffffff, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(P.status, init, sizeof(init), cudaMemcpyHostToDevice, st));
  }
  // block range of every tile (for the per-panel pair kernel of the host-staged path)
  std::vector<int> tile_blk((size_t)M + 1, nb);
  for (int p = nb - 1; p >= 0; --p) tile_blk[row_tile[bs[p]]] = p;
  for (int I = M - 1; I >= 0; --I) tile_blk[I] = std::min(tile_blk[I], tile_blk[I + 1]);
  if (hs) {
    if ((int)hs->ev->size() < M) {
      for (cudaEvent_t e : *hs->ev) cudaEventDestroy(e);
      hs->ev->assign((size_t)M, nullptr);
      for (auto& e : *hs->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (int I = M - 1; I >= 0; --I) {
      const int rows = std::min(ts[I + 1] + 1, m), ncol = ts[I + 1] - ts[I];
      double* Sp = (double*)(S + (size_t)ts[I] * lds);
      double* Tp = (double*)(T + (size_t)ts[I] * ldt);
      if (hs->Sh) {
        // host panel -> rank 0's device copy (Ssrc, Tsrc)
        CK(cudaMemcpy2DAsync((void*)(hs->Ssrc + (size_t)ts[I] * hs->ldss), (size_t)hs->ldss * 8,
                             hs->Sh + (size_t)ts[I] * hs->ldsh, (size_t)hs->ldsh * 8, (size_t)rows * 8, ncol,
                             cudaMemcpyHostToDevice, hs->copy));
        CK(cudaMemcpy2DAsync((void*)(hs->Tsrc + (size_t)ts[I] * hs->ldts), (size_t)hs->ldts * 8,
                             hs->Th + (size_t)ts[I] * hs->ldth, (size_t)hs->ldth * 8, (size_t)rows * 8, ncol,
                             cudaMemcpyHostToDevice, hs->copy));
      }
      if (hs->comm) {
        // one contiguous buffer [S panel | T panel] per broadcast (rows x ncol each)
        const size_t half = (size_t)rows * ncol;
        if (hs->root) {
          CK(cudaMemcpy2DAsync(hs->bbuf, (size_t)rows * 8, hs->Ssrc + (size_t)ts[I] * hs->ldss,
                               (size_t)hs->ldss * 8, (size_t)rows * 8, ncol, cudaMemcpyDeviceToDevice, hs->copy));
          CK(cudaMemcpy2DAsync(hs->bbuf + half, (size_t)rows * 8, hs->Tsrc + (size_t)ts[I] * hs->ldts,
                               (size_t)hs->ldts * 8, (size_t)rows * 8, ncol, cudaMemcpyDeviceToDevice, hs->copy));
        }
        if (hs->api->broadcast(hs->bbuf, hs->bbuf, 2 * half, ncclFloat64, 0, hs->comm, hs->copy) != ncclSuccess)
          return ZZ_ERR_NCCL;
        if (!hs->root || Sp != hs->Ssrc + (size_t)ts[I] * hs->ldss) {
          CK(cudaMemcpy2DAsync(Sp, (size_t)lds * 8, hs->bbuf, (size_t)rows * 8, (size_t)rows * 8, ncol,
                               cudaMemcpyDeviceToDevice, hs->copy));
          CK(cudaMemcpy2DAsync(Tp, (size_t)ldt * 8, hs->bbuf + half, (size_t)rows * 8, (size_t)rows * 8, ncol,
                               cudaMemcpyDeviceToDevice, hs->copy));
        }
      }
      CK(cudaEventRecord((*hs->ev)[I], hs->copy));
    }
  }
  // TMA needs 16-byte aligned bases and even leading dimensions; otherwise repack
  const double* Su = S;
  const double* Tu = T;
  long long ldsu = lds, ldtu = ldt;
  auto repack = [&](Buf& b, const double* A, long long lda, int k, const double*& out, long long& ldo) -> int {
    long long ld2 = (m + 1) / 2 * 2;
    cudaError_t e = b.ensure(sizeof(double) * (size_t)ld2 * m);
    if (e != cudaSuccess) return map_err(e);
    e = launch_scale_copy(A, lda, m, k, b.as<double>(), ld2, st);
    if (e != cudaSuccess) return map_err(e);
    out = b.as<double>();
    ldo = ld2;
    launches++;
    return 0;
  };
  if ((lds & 1) || !aligned16(S)) { int r = repack(c->Sc, S, lds, 0, Su, ldsu); if (r) return r; }
  if ((ldt & 1) || !aligned16(T)) { int r = repack(c->Tc, T, ldt, 0, Tu, ldtu); if (r) return r; }
  // ---- a2 pairs, a3 norms (second host sync: status + pre-scale test) ----
  // (host-staged path: per panel inside the wavefront, checked after it)
  if (hs) CK(cudaMemsetAsync(P.cS, 0, sizeof(double) * 4 * M, st));
  double panel_max = 0.0;   // largest panel norm (the lookahead heuristic below)
  for (int pass = 0; pass < 2 && !hs; ++pass) {
    CK(cudaMemsetAsync(P.cS, 0, sizeof(double) * 4 * M, st));
    CK(launch_pairs(Su, ldsu, Tu, ldtu, 0, nb, P, st));
    CK(launch_panel_norms(Su, ldsu, Tu, ldtu, M, ts.data(), P, st, 0, M));
    launches += 2 + (M > 1);
    std::vector<double> nrm(4 * (size_t)M);
    int stat[16];
    CK(cudaMemcpyAsync(stat, P.status, sizeof(stat), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(nrm.data(), P.cS, sizeof(double) * 4 * M, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (stat[0] != 0x7fffffff) {
      int p = stat[0] >> 2, kind = stat[0] & 3;
      return kind == 1 ? ZZ_ERR_NONFINITE : bs[p] + 1;
    }
    info.n_indefinite = stat[2];
    for (int I = 0; I < M; ++I) panel_max = std::max(panel_max, std::max(nrm[I], nrm[M + I]));
    if (pass == 1) break;
    // pre-scale test (reading R6): every row sum of |S| is <= sum_J cS[J] + max_J dS[J]
    double bS = 0, bT = 0, mdS = 0, mdT = 0;
    for (int I = 0; I < M; ++I) {
      bS += nrm[I]; bT += nrm[M + I];
      mdS = std::max(mdS, nrm[2 * M + I]); mdT = std::max(mdT, nrm[3 * M + I]);
    }
    bS += mdS;
    bT += mdT;
    const double lim = 0x1p1020;  // Omega / 8
    if (bS <= lim && bT <= lim) break;
    // rare path: scale S and/or T by 2^-k (exact), so that m * maxabs <= Omega / 8
    CK(cudaMemsetAsync(P.maxabs, 0, 16, st));
    CK(launch_maxabs(Su, ldsu, Tu, ldtu, m, P.maxabs, st));
    unsigned long long mx[2];
    CK(cudaMemcpyAsync(mx, P.maxabs, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int w = 0; w < 2; ++w) {
      double bound = w ? bT : bS;
      if (bound <= lim) continue;
      double amax;
      memcpy(&amax, &mx[w], 8);
      int ea;
      frexp(amax, &ea);  // amax < 2^ea
      int em = (int)ceil(log2((double)std::max(m, 2)));
      int k = ea + em - 1020 + 1;
      if (k < 0) k = 0;
      int r = w ? repack(c->Tc, Tu, ldtu, k, Tu, ldtu) : repack(c->Sc, Su, ldsu, k, Su, ldsu);
      if (r) return r;
    }
    info.prescaled = 1;
    int init[16] = {0x7fffffff, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(P.status, init, sizeof(init), cudaMemcpyHostToDevice, st));
  }
  if (n_sel == 0 && !hs) {
    c->info = info;
    return 0;
  }
  CUtensorMap tmS, tmT;
  if (M > 1) {
    int r = make_map(c, &tmS, Su, ldsu, m);
    if (!r) r = make_map(c, &tmT, Tu, ldtu, m);
    if (r) return r;
  }
  CK(cudaMemsetAsync(P.e_pend, 0, sizeof(int) * n, st));
  CK(cudaMemsetAsync(P.nY, 0, sizeof(unsigned long long) * kMaxGroup * n, st));
  CK(cudaEventRecord(c->e1, st));
  // ---- the wavefront (Algorithm 1 over tile rows, bottom-up) ----
  // X with an odd leading dimension or a base that is not 16-byte aligned: solve into an
  // aligned internal buffer and copy out once (below), so that every X runs the same kernels
  // in the same order -- results are bitwise independent of ldx
  double* Xout = nullptr;
  long long ldxo = 0;
  if (n_sel > 0 && (((ldx & 1) != 0) || !aligned16(X))) {
    const long long ldi = (m + 1) & ~1LL;
    CK(c->Xi.ensure(sizeof(double) * (size_t)ldi * n_sel));
    Xout = X;
    ldxo = ldx;
    X = c->Xi.as<double>();
    ldx = ldi;
  }
  const int vec = ((ldx & 1) == 0) && aligned16(X);
  if (c->timing && (int)c->ev.size() < 4 * M) {
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    c->ev.assign(4 * (size_t)M, nullptr);
    for (auto& e : c->ev) cudaEventCreate(&e);
  }
  int n_upd = 0, n_fused = 0;
  // Two-step fusion (ZZ_FUSE, default on with the k_diag3 / k_update_t path): for a pair of
  // steps (I, J = I - 1) the rows of tile J get step I's update first (a thin update, one
  // 128-row band), tile J is solved, and the rows above tile J get both steps' updates in one
  // contraction with K = [tile J | tile I] (twice the K of a single step: half the C-tile
  // traffic and prologue/epilogue per flop).
  const int fusion = std::max(1, std::min(kMaxGroup, c->fusion));
  const bool can_fuse = fusion > 1 && vec && mb <= kDiag2MaxNT;
  for (int k = 0; k + 1 < fusion; ++k) CK(c->Wx[k].ensure(c->W.cap));
  // Lookahead: the chain of solves and band updates runs on a high-priority stream `ms`; the
  // bulk of each group's update (the rows above the next group's band) runs on the caller's
  // stream `st` beside the next group's solves.  W and sY alternate between two sets by
  // group; the next group's first decision uses the recorded bound nYb instead of the
  // maximum the bulk update is still computing.
  // (lookahead = 1, the default, is automatic: on for m >= 1024 unless a panel norm exceeds
  // 2^64 -- then the first decisions of the groups would likely have to scale on the bound
  // and the call would be recomputed; 2 forces it, 0 disables it)
  const bool la = can_fuse && (c->lookahead == 2 || (c->lookahead == 1 && m >= 1024 && panel_max <= 0x1p64));
  cudaStream_t ms = st;
  int* sY_set[2] = {P.sY, P.sY};
  if (la) {
    if (!c->hi) {
      int lo_p, hi_p;
      CK(cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p));
      CK(cudaStreamCreateWithPriority(&c->hi, cudaStreamNonBlocking, hi_p));
      CK(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
    }
    if ((int)c->ev_la.size() < 2 * M + 2) {
      for (cudaEvent_t e : c->ev_la) cudaEventDestroy(e);
      c->ev_la.assign(2 * (size_t)M + 2, nullptr);
      for (auto& e : c->ev_la) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (int k = 0; k < fusion; ++k) CK(c->Wy[k].ensure(c->W.cap));
    CK(c->sYb.ensure(sizeof(int) * (size_t)n));
    sY_set[1] = c->sYb.as<int>();
    ms = c->hi;
  }
  int n_la_ev = 0;
  int gpar = 0;                      // W / sY set of the current group (lookahead)
  bool prev_bound = false;           // the previous group recorded nYb (lookahead)
  cudaEvent_t ev_rest = nullptr;     // the bulk update of the previous group (lookahead)
  int nyb = (M - 1) & 1;   // nY buffer holding the pending max for the next decision
  auto panel_ready = [&](int I) -> int {
    if (!hs) return 0;
    // panel I has arrived: its eigenvalue pairs and column-panel norms
    if (hs->wait) CK(cudaStreamWaitEvent(ms, (*hs->ev)[I], 0));
    CK(launch_pairs(Su, ldsu, Tu, ldtu, tile_blk[I], tile_blk[I + 1] - tile_blk[I], P, ms));
    CK(launch_panel_norms(Su, ldsu, Tu, ldtu, M, ts.data(), P, ms, I, 1));
    launches += 2;
    return 0;
  };
  auto diag = [&](int I, double* Wout, const Diag2Params* fuse_from) -> int {
    DiagParams dp;
    dp.I = I;
    dp.t0 = ts[I];
    dp.nt = ts[I + 1] - ts[I];
    dp.item_begin = tile_item[I];
    dp.n_items = n_items;
    dp.tip_col_end = cs[I + 1];
    dp.do_update = (I > 0);
    dp.nks = ceil_div(dp.nt, kBK);
    dp.n_sel = n_sel;
    dp.S = Su; dp.lds = ldsu; dp.T = Tu; dp.ldt = ldtu;
    dp.X = X; dp.ldx = ldx;
    dp.P = P;
    dp.nY_in = nyb;
    if (dp.nt <= kDiag2MaxNT) {
      Diag2Params d2;
      memset(&d2, 0, sizeof(d2));
      d2.I = I; d2.t0 = dp.t0; d2.nt = dp.nt;
      d2.n_real = (int)real_list.size() - rbeg[I];
      d2.n_pair = (int)pair_list.size() - pbeg[I];
      d2.real_items = P.real_items + rbeg[I];
      d2.pair_items = P.pair_items + pbeg[I];
      d2.tip_col_end = dp.tip_col_end;
      d2.do_update = dp.do_update;
      d2.nks = dp.nks;
      d2.n_sel = n_sel;
      d2.S = Su; d2.lds = ldsu; d2.T = Tu; d2.ldt = ldtu;
      d2.X = X; d2.ldx = ldx;
      d2.P = P;
      d2.P.sY = sY_set[gpar];
      d2.pack = la;
      d2.team_w = c->diag_team;
      d2.nY_in = dp.nY_in;
      d2.bnd_in = nyb;   // the recorded bounds alternate between two sets by group (as nY)
      d2.Wout = Wout;
      d2.grp_slot = -1;
      if (fuse_from) {
        // role in a step group (zz_diag3.cu): first (grp_slot 0), middle (fused 2), last (3)
        d2.fused = fuse_from->fused;
        d2.grp_slot = fuse_from->grp_slot;
        d2.n_band_reset = fuse_from->n_band_reset;
        d2.band_in = fuse_from->band_in;
        d2.n_prev = fuse_from->n_prev;
        for (int k = 0; k < kMaxGroup - 1; ++k) {
          d2.prev_I[k] = fuse_from->prev_I[k];
          d2.prev_cs[k] = fuse_from->prev_cs[k];
          d2.prev_nks[k] = fuse_from->prev_nks[k];
          d2.prev_W[k] = fuse_from->prev_W[k];
        }
        d2.zero_pend_end = fuse_from->zero_pend_end;
        d2.use_bound = fuse_from->use_bound;
        d2.record_bound = fuse_from->record_bound;
        if (d2.fused == 2) d2.nY_in = d2.band_in;
      }
      CK(launch_diag3(d2, ms));
    } else {
      CK(launch_diag(dp, ms));
    }
    launches++;
    return 0;
  };
  auto update = [&](UpdParams up, int n_m, cudaStream_t us) -> int {
    const int n_n = ceil_div(n_sel, kBN) - up.ntile0;
    if (c->timing) CK(cudaEventRecord(c->ev[2 * n_upd], us));
    CK(launch_update(&tmS, &tmT, up, n_m, n_n, us));
    if (c->timing) CK(cudaEventRecord(c->ev[2 * n_upd + 1], us));
    n_upd++;
    launches++;
    return 0;
  };
  auto base_up = [&](int I) {
    UpdParams up;
    memset(&up, 0, sizeof(up));
    up.rows = ts[I];
    up.max_row = (I > 0) ? ts[I - 1] : 0;
    up.t0 = ts[I];
    up.nks = ceil_div(ts[I + 1] - ts[I], kBK);
    up.c_begin = cs[I];
    up.first_end = cs[I + 1];
    up.n_sel = n_sel;
    up.ntile0 = cs[I] / kBN;
    up.X = X; up.ldx = ldx;
    up.W = P.W;
    up.sY = sY_set[gpar];
    up.nY_out = P.nY + (size_t)(1 - nyb) * n;
    up.vec = vec;
    return up;
  };
  // the wavefront proper: a fixed sequence of launches for a given plan (no host decision
  // depends on device data inside it), captured once into a CUDA graph and replayed while
  // the plan and every pointer it uses stay the same
  auto wavefront = [&]() -> int {
    if (la) {   // fork the chain's stream from the caller's (inside a capture: joins the graph)
      CK(cudaEventRecord(c->ev_in, st));
      CK(cudaStreamWaitEvent(ms, c->ev_in, 0));
    }
    int I = M - 1;
    while (I >= 0) {
      int r = panel_ready(I);
      if (r) return r;
      if (tile_item[I] >= n_items) { --I; continue; }
      // Step groups are fixed by the tile index alone (groups of `fusion` consecutive steps
      // counted from M-1), not by which steps have active columns: a step that opens the
      // solve in the middle of its group runs the group's remaining steps, so a column's
      // operations do not depend on the selection (sharding, select).  The last step of a
      // fused group needs rows above it (index >= 1).
      int len = 1;
      if (can_fuse) {
        len = fusion - (M - 1 - I) % fusion;
        while (len > 1 && I - (len - 1) < 1) --len;
      }
      auto nks_of = [&](int t) { return ceil_div(ts[t + 1] - ts[t], kBK); };
      if (len >= 2) {
        // ---- a step group (I, I-1, ..., L = I-len+1): diag of each step, thin updates of the
        // group's own band (the rows of its later tiles) after every step but the last, and one
        // update of all rows above tile L with K = [tile L | ... | tile I] ----
        const int L = I - len + 1;
        double* Wg[kMaxGroup];
        Wg[0] = P.W;
        for (int k = 1; k < len; ++k) Wg[k] = c->Wx[k - 1].as<double>();
        if (la && gpar == 1)
          for (int k = 0; k < len; ++k) Wg[k] = c->Wy[k].as<double>();
        bool rest_waited = false;   // the chain has waited for the previous group's bulk update
        for (int sgi = 0; sgi < len; ++sgi) {
          const int X = I - sgi;
          if (sgi > 0 && (r = panel_ready(X))) return r;
          Diag2Params o;
          memset(&o, 0, sizeof(o));
          if (sgi == 0) {
            o.fused = 0;
            o.grp_slot = 0;
            o.n_band_reset = len - 2;
            o.use_bound = la && prev_bound;
            if (la && !prev_bound && ev_rest) {
              CK(cudaStreamWaitEvent(ms, ev_rest, 0));
              rest_waited = true;
            }
          } else if (sgi < len - 1) {
            o.fused = 2;
            o.grp_slot = sgi;
            o.band_in = 2 + (sgi - 1);
          } else {
            o.fused = 3;
            o.grp_slot = -1;
            o.n_prev = len - 1;
            for (int k = 0; k < len - 1; ++k) {
              o.prev_I[k] = I - k;
              o.prev_cs[k] = cs[I - k];
              o.prev_nks[k] = nks_of(I - k);
              o.prev_W[k] = Wg[k];
            }
            o.zero_pend_end = cs[I + 1];       // tips of the group start from zero pending rows
            o.record_bound = la;
            // Lookahead: the decision takes the previous group's recorded bound of the rows
            // above tile L, as the group's first decision does, so the whole chain of the group
            // runs beside the previous group's bulk update (it used to wait here for that
            // update's measured maximum: 0.2-0.5 ms per group with the machine mostly idle).
            // Without a recorded bound it needs the measured maximum, i.e. that update.
            o.use_bound = la && prev_bound;
            if (la && ev_rest && !o.use_bound) {
              CK(cudaStreamWaitEvent(ms, ev_rest, 0));
              rest_waited = true;
            }
          }
          if ((r = diag(X, Wg[sgi], &o))) return r;
          if (sgi < len - 1) {
            UpdParams th = base_up(X);         // rows of the group's tiles below X with W_X
            th.row_lo = ts[L];
            th.W = Wg[sgi];
            if (sgi + 1 < len - 1) {           // band maximum for the next (middle) step
              th.max_row = ts[X - 1];
              th.nY_out = P.nY + (size_t)(2 + sgi) * n;
            } else {
              th.max_row = 0;
            }
            if ((r = update(th, ceil_div(ts[X] - (ts[L] & ~1), kBM), ms))) return r;
          }
        }
        UpdParams fu = base_up(L);
        fu.W = Wg[len - 1];
        fu.first_end = cs[I + 1];
        fu.nxs = len - 1;
        for (int e = 0; e < len - 1; ++e) {    // tiles L+1, ..., I after tile L
          const int X = L + 1 + e;
          fu.xt0[e] = ts[X];
          fu.xnks[e] = nks_of(X);
          fu.xW[e] = Wg[I - X];
        }
        // the next group's band: its tiles L-1 .. L-len_next (the grouping rule of this loop)
        int len_next = 0;
        if (la && L - 1 >= 1) {
          const int In = L - 1;
          len_next = fusion - (M - 1 - In) % fusion;
          while (len_next > 1 && In - (len_next - 1) < 1) --len_next;
        }
        if (la && len_next >= 1 && ts[L - len_next] > 0) {
          const int rb = ts[L - len_next];        // rows [rb, ts[L]): the next group's band
          UpdParams fb = fu;                    // the band first, on the chain's stream
          fb.row_lo = rb;
          // the band part measures rows [rb, ts[L-1]) and the bulk rows [0, rb) into the same
          // buffer (atomicMax: order-independent), so the next group's last decision reads the
          // maximum over [0, ts[L-1]) exactly as in the plain schedule (base_up(L).max_row)
          fb.max_row = ts[L - 1];
          // the group's W operands and decisions are complete: the bulk may start (after the
          // previous bulk, in stream order), beside the band part (disjoint rows)
          // (from 4096 columns; with fewer the chain is the critical path and a bulk update
          // beside its band part slows it -- C2 2.05 -> 2.14 ms, a 1 % subset of C4 45.6 ->
          // 48.0 ms measured -- so there the bulk starts after the band part)
          const bool early_bulk = n_sel >= 4096;
          cudaEvent_t ev_dec = c->ev_la[n_la_ev++];
          if (early_bulk) CK(cudaEventRecord(ev_dec, ms));
          // the band part updates rows the previous group's bulk update wrote
          if (ev_rest && !rest_waited) CK(cudaStreamWaitEvent(ms, ev_rest, 0));
          if ((r = update(fb, ceil_div(ts[L] - (rb & ~1), kBM), ms))) return r;
          if (!early_bulk) CK(cudaEventRecord(ev_dec, ms));
          CK(cudaStreamWaitEvent(st, ev_dec, 0));
          UpdParams fr = fu;                    // the bulk on the caller's stream
          fr.rows = rb;
          fr.max_row = rb;
          if ((r = update(fr, ceil_div(rb, kBM), st))) return r;
          ev_rest = c->ev_la[n_la_ev++];
          CK(cudaEventRecord(ev_rest, st));
          prev_bound = true;
        } else {
          if (la && ev_rest) CK(cudaStreamWaitEvent(ms, ev_rest, 0));
          if ((r = update(fu, ceil_div(ts[L], kBM), ms))) return r;
          ev_rest = nullptr;
          prev_bound = false;
        }
        nyb = 1 - nyb;
        gpar ^= (la ? 1 : 0);
        ++n_fused;
        I -= len;
        continue;
      }
      if (la && ev_rest) {               // a single step takes the measured maximum
        CK(cudaStreamWaitEvent(ms, ev_rest, 0));
        ev_rest = nullptr;
      }
      prev_bound = false;
      if ((r = diag(I, P.W, nullptr))) return r;
      if (I > 0) {
        UpdParams up = base_up(I);
        if ((r = update(up, ceil_div(ts[I], kBM), ms))) return r;
        nyb = 1 - nyb;
      }
      --I;
    }
    if (la) {                            // join the chain's stream back into the caller's
      CK(cudaEventRecord(c->ev_out, ms));
      CK(cudaStreamWaitEvent(st, c->ev_out, 0));
    }
    return 0;
  };
  // (not with per-launch timing: the roofline pass measures plain stream launches)
  const bool use_graph = c->graphs && !hs && n_sel > 0 && !c->timing;
  nvtxRangePushA(use_graph ? "zz.wavefront (graph)" : "zz.wavefront");
  if (use_graph) {
    // the plan's identity: sizes, modes, every pointer the launches use, and the host tables
    uint64_t key = 1469598103934665603ull;
    auto mix = [&](const void* d, size_t bytes) {
      const unsigned char* q = static_cast<const unsigned char*>(d);
      for (size_t i = 0; i < bytes; ++i) key = (key ^ q[i]) * 1099511628211ull;
    };
    const long long sc[] = {m, mb, n_sel, M, fusion, (long long)la, (long long)c->timing, (long long)vec, ldsu, ldtu,
                            ldx, nb, n_items, (long long)c->diag_team};
    mix(sc, sizeof(sc));
    const void* ptrs[] = {Su, Tu, X, c->colf.p, c->coli.p, c->items.p, c->tiles.p, c->rows.p, c->blks.p,
                          c->state.p, c->seg.p, c->norms.p, c->W.p, c->status.p, c->egrp.p, c->nYb.p, c->sYb.p,
                          c->Wx[0].p, c->Wx[1].p, c->Wx[2].p, c->Wx[3].p, c->Wx[4].p, c->Wy[0].p, c->Wy[1].p,
                          c->Wy[2].p, c->Wy[3].p, c->Wy[4].p, c->Wy[5].p, c->hi};
    mix(ptrs, sizeof(ptrs));
    mix(ts.data(), sizeof(int) * ts.size());
    mix(col_r.data(), sizeof(int) * col_r.size());
    mix(item_col.data(), sizeof(int) * item_col.size());
    mix(real_list.data(), sizeof(int) * real_list.size());
    mix(pair_list.data(), sizeof(int) * pair_list.size());
    if (c->gexec && key == c->gkey) {
      CK(cudaGraphLaunch(c->gexec, st));
      n_upd = c->g_nupd;
      n_fused = c->g_nfused;
      launches += c->g_launches;
    } else {
      const int l0 = launches;
      // captured on a stream of the library's own (the caller's stream may be the legacy
      // default stream, which cannot be captured); the graph is then launched on st
      if (!c->cap) CK(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
      const cudaStream_t st0 = st;
      const bool ms_is_st = ms == st;
      st = c->cap;
      if (ms_is_st) ms = c->cap;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
      const int r = wavefront();
      cudaGraph_t g = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(st, &g);
      st = st0;
      if (ms_is_st) ms = st0;
      if (r) {
        if (g) cudaGraphDestroy(g);
        return r;
      }
      CK(ec);
      if (c->gexec) cudaGraphExecDestroy(c->gexec);
      c->gexec = nullptr;
      // node priorities as captured: the lookahead's chain keeps its high-priority stream's
      // priority inside the graph
      const cudaError_t ei = cudaGraphInstantiateWithFlags(&c->gexec, g, cudaGraphInstantiateFlagUseNodePriority);
      cudaGraphDestroy(g);
      CK(ei);
      c->gkey = key;
      c->g_nupd = n_upd;
      c->g_nfused = n_fused;
      c->g_launches = launches - l0;
      CK(cudaGraphLaunch(c->gexec, st));
    }
  } else {
    if (int r = wavefront()) return r;
  }
  nvtxRangePop();
  CK(cudaEventRecord(c->e2, st));
  // ---- a7 consistency and normalisation ----
  CK(launch_normalize(m, n_sel, M, X, ldx, cse, P, exp_tmp, rec_tmp, st));
  launches += 2;
  if (Xout)
    CK(cudaMemcpy2DAsync(Xout, sizeof(double) * ldxo, X, sizeof(double) * ldx, sizeof(double) * m, n_sel,
                         cudaMemcpyDeviceToDevice, st));
  // every staged transfer (the last one is panel 0) completes before the call returns
  if (hs && M > 0) CK(cudaStreamWaitEvent(st, (*hs->ev)[0], 0));
  CK(cudaEventRecord(c->e3, st));
  int stat[16];
  CK(cudaMemcpyAsync(stat, P.status, sizeof(stat), cudaMemcpyDeviceToHost, st));
  std::vector<double> nrm(hs ? 4 * (size_t)M : 0);
  if (hs) CK(cudaMemcpyAsync(nrm.data(), P.cS, sizeof(double) * 4 * M, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hs) {
    // deferred checks of the host-staged path: pair status, then the pre-scale test (R6);
    // a pencil that needs the pre-scale is solved again on the (now complete) device copy
    if (stat[0] != 0x7fffffff) {
      int p = stat[0] >> 2, kind = stat[0] & 3;
      return kind == 1 ? ZZ_ERR_NONFINITE : bs[p] + 1;
    }
    info.n_indefinite = stat[2];
    double bS = 0, bT = 0, mdS = 0, mdT = 0;
    for (int I = 0; I < M; ++I) {
      bS += nrm[I]; bT += nrm[M + I];
      mdS = std::max(mdS, nrm[2 * M + I]); mdT = std::max(mdT, nrm[3 * M + I]);
    }
    if (bS + mdS > 0x1p1020 || bT + mdT > 0x1p1020)
      return tgevc_device(c, m, S, lds, T, ldt, select, X_call, ldx_call, cse, nullptr);
  }
  if (la && stat[6]) {
    // a group's first decision on the recorded bound would have scaled where the measured
    // maximum may not: recompute without lookahead (bitwise the plain schedule's result)
    const int saved = c->lookahead;
    c->lookahead = 0;
    const int rr = tgevc_device(c, m, S, lds, T, ldt, select, X_call, ldx_call, cse, nullptr);
    c->lookahead = saved;
    c->info.lookahead_redo = 1;
    return rr;
  }
  info.n_scaled = stat[4];
  info.min_exp = stat[5];
  if (n_sel > 0) {
    info.d_logmax = P.logmax;
    info.d_a = P.col_a;
    info.d_b = P.col_b;
    info.d_beta = P.col_beta;
  }
  info.update_launches = n_upd;
  info.fused_pairs = n_fused;
  info.total_launches = launches;
  float el;
  cudaEventElapsedTime(&el, c->e0, c->e1); info.ms_setup = el;
  cudaEventElapsedTime(&el, c->e1, c->e2); info.ms_steps = el;
  cudaEventElapsedTime(&el, c->e2, c->e3); info.ms_normalize = el;
  if (c->timing) {
    double tot = 0;
    for (int u = 0; u < n_upd; ++u) {
      cudaEventElapsedTime(&el, c->ev[2 * u], c->ev[2 * u + 1]);
      tot += el;
    }
    info.ms_update = tot;
  }
  c->info = info;
  return 0;
}

// xTGEVC HOWMNY='B' (reading A1): W = V X as one FP64 tensor-core
// contraction over the triangular K range (columns are in block order, so r_c is
// non-decreasing and X is zero below r_c: tile J of 64 columns needs K_J = 1 + its last
// column's r_c), then LAPACK's normalisation of the back-transformed columns (zz_back.cu).
int tgevc_back_device(Context* c, int m, const double* S, long long lds, const double* T, long long ldt,
                      const int* select, const double* V, long long ldv, double* W, long long ldw, int* cse) {
  cudaStream_t st = c->stream;
  const long long ldxb = (m + 1) & ~1LL;
  CK(c->Xb.ensure(sizeof(double) * (size_t)ldxb * (size_t)std::max(m, 1)));
  double* Xb = c->Xb.as<double>();
  int r = tgevc_device(c, m, S, lds, T, ldt, select, Xb, ldxb, cse);
  if (r) return r;
  const int n_sel = c->info.n_sel;
  if (n_sel == 0) return 0;
  CK(cudaEventRecord(c->e0, st));
  // V by TMA needs a 16-byte aligned base and an even leading dimension; W is stored with
  // 16-byte stores: otherwise through aligned library copies
  const double* Vu = V;
  long long ldvu = ldv;
  if ((ldv & 1) || !aligned16(V)) {
    CK(c->Vc.ensure(sizeof(double) * (size_t)ldxb * m));
    CK(cudaMemcpy2DAsync(c->Vc.p, sizeof(double) * ldxb, V, sizeof(double) * ldv, sizeof(double) * m, m,
                         cudaMemcpyDeviceToDevice, st));
    Vu = c->Vc.as<double>();
    ldvu = ldxb;
  }
  double* Wu = W;
  long long ldwu = ldw;
  if ((ldw & 1) || !aligned16(W)) {
    CK(c->Xi.ensure(sizeof(double) * (size_t)ldxb * n_sel));
    Wu = c->Xi.as<double>();
    ldwu = ldxb;
  }
  const int n_nt = (n_sel + kBN - 1) / kBN;
  std::vector<int> nkc((size_t)n_nt);
  std::vector<long long> woff((size_t)n_nt);
  long long tot = 0;
  int max_nkc = 1;
  for (int J = 0; J < n_nt; ++J) {
    const int last = std::min(n_sel - 1, J * kBN + kBN - 1);
    nkc[J] = ceil_div(c->last_col_r[last] + 1, kBK);
    max_nkc = std::max(max_nkc, nkc[J]);
    woff[J] = tot;
    tot += (long long)nkc[J] * (kBN * kBK);
  }
  CK(c->Xp.ensure(sizeof(double) * (size_t)tot));
  CK(c->btab.ensure((sizeof(int) + sizeof(long long)) * (size_t)n_nt + sizeof(unsigned long long) * (size_t)n_sel + 64));
  long long* d_woff = c->btab.as<long long>();
  int* d_nkc = reinterpret_cast<int*>(d_woff + n_nt);
  unsigned long long* d_cmax = reinterpret_cast<unsigned long long*>(d_woff + n_nt + (n_nt + 1) / 2 + 1);
  CK(cudaMemcpyAsync(d_woff, woff.data(), sizeof(long long) * n_nt, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_nkc, nkc.data(), sizeof(int) * n_nt, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(d_cmax, 0, sizeof(unsigned long long) * n_sel, st));
  CUtensorMap tmV;
  if (int e = make_map(c, &tmV, Vu, ldvu, m)) return e;
  CK(launch_back_gemm(&tmV, Xb, ldxb, m, n_sel, d_nkc, d_woff, max_nkc, c->Xp.as<double>(), Wu, ldwu, d_cmax, st));
  // the column kinds of the last call are still in the workspace (DevPlan.col_kind)
  CK(launch_back_norm(Wu, ldwu, m, n_sel, c->coli.as<int>(), d_cmax, st));
  if (Wu != W)
    CK(cudaMemcpy2DAsync(W, sizeof(double) * ldw, Wu, sizeof(double) * ldwu, sizeof(double) * m, n_sel,
                         cudaMemcpyDeviceToDevice, st));
  CK(cudaEventRecord(c->e1, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->e0, c->e1);
  c->info.ms_back = ms;
  c->info.total_launches += 3;
  return 0;
}

// Left eigenvectors (LAPACK xTGEVC SIDE='L'): y^H (beta S - alpha T) = 0
// is (beta S^T - conj(alpha) T^T) y = 0, and with the reversal J, (S', T') = (J S^T J, J T^T J) is
// a real Schur pencil with the same eigenvalues whose right eigenvector for lambda is
// conj(J y) (csrc/zz_left.cu).  The robust blocked right solve runs on (S', T'); the result
// is mapped back: rows reversed, a pair's imaginary column negated, columns in S's block order.
int tgevc_left_device(Context* c, int m, const double* S, long long lds, const double* T, long long ldt,
                      const int* select, double* Y, long long ldy, int* cse) {
  cudaStream_t st = c->stream;
  const long long ldf = (m + 1) & ~1LL;
  const size_t mat = sizeof(double) * (size_t)ldf * (size_t)m;
  CK(c->Sl.ensure(mat));
  CK(c->Tl.ensure(mat));
  CK(c->Xb.ensure(mat));
  CK(c->El.ensure(sizeof(int) * (size_t)m));
  double* Sf = c->Sl.as<double>();
  double* Tf = c->Tl.as<double>();
  CK(launch_flip_transpose(S, lds, Sf, ldf, m, st));
  CK(launch_flip_transpose(T, ldt, Tf, ldf, m, st));
  std::vector<int> self;
  if (select) {
    self.resize(m);
    for (int j = 0; j < m; ++j) self[m - 1 - j] = select[j];
  }
  int r = tgevc_device(c, m, Sf, ldf, Tf, ldf, select ? self.data() : nullptr, c->Xb.as<double>(), ldf,
                       c->El.as<int>());
  if (r > 0) return m - r;          // the 2x2 block at rows (r-1, r) of S' is rows (m-r-1, m-r) of S
  if (r) return r;
  const int n_sel = c->info.n_sel;
  CK(launch_left_gather(c->Xb.as<double>(), ldf, Y, ldy, m, n_sel, c->coli.as<int>(), c->El.as<int>(), cse, st));
  CK(cudaStreamSynchronize(st));
  c->info.total_launches += 3;
  // the device views describe the flipped pencil's columns: not exported for left vectors
  c->info.d_logmax = c->info.d_a = c->info.d_b = c->info.d_beta = nullptr;
  return 0;
}

// ---- the sharded / collective solve ----
// The eigenvalue blocks are owned in groups of kShardNB rows, cyclically over P shards (block
// with first row j -> shard (j / kShardNB) mod P: triangular load balance).  Every shard runs
// the full bottom-up wavefront over its own columns only -- the task graph is the disjoint
// union of per-column-block subgraphs, and a column's arithmetic does not depend
// on which other columns are computed, so X is bitwise independent of P.  With a communicator,
// S and T come from rank 0 by NCCL broadcast panel by panel in consumption order (I = M-1 .. 0,
// upper part and subdiagonal only; step I waits for panel I), and the finished columns -- their
// upper parts only, rows 0 .. r_c -- are gathered on rank 0 and written into the caller's X
// (zeros below).  Without one (zz_set_shard on a single GPU) the shard's columns are written
// into their global positions of X and the others are left untouched.
struct ShardCol { int g, r; };

// Owner of every selected eigenvalue block (first row j -> shard (j / kShardNB) mod P): the
// global output columns (block order) and last rows of each shard, and shard p's select mask.
void shard_owners(int m, const std::vector<int>& bs, const std::vector<int>& bz, const int* select, int P, int p,
                  std::vector<std::vector<ShardCol>>& cols, std::vector<int>& sel_loc) {
  cols.assign((size_t)P, {});
  sel_loc.assign((size_t)m, 0);
  int n_glob = 0;
  for (size_t q = 0; q < bs.size(); ++q) {
    const int j = bs[q];
    const bool sel = !select || select[j] || (bz[q] == 2 && select[j + 1]);
    if (!sel) continue;
    const int own = (j / kShardNB) % P;
    for (int k = 0; k < bz[q]; ++k) cols[own].push_back(ShardCol{n_glob + k, j + bz[q] - 1});
    if (own == p)
      for (int k = 0; k < bz[q]; ++k) sel_loc[j + k] = 1;
    n_glob += bz[q];
  }
}

int tgevc_sharded(Context* c, int m, const double* S, long long lds, const double* T, long long ldt,
                  const int* select, double* X, long long ldx, int* cse, const double* Sh = nullptr,
                  long long ldsh = 0, const double* Th = nullptr, long long ldth = 0) {
  cudaStream_t st = c->stream;
  Range r_call("zz_tgevc (sharded)");
  const NcclApi* api = c->comm ? nccl_api() : nullptr;
  if (c->comm && !api) return ZZ_ERR_NCCL;
  const int P = (c->nranks > 1) ? c->nranks : c->shard_P;
  const int p = (c->nranks > 1) ? c->rank : c->shard_p;
  const bool root = c->rank == 0;               // communication role
  const bool recv_role = c->comm && (!root || p != 0);   // computes from the broadcast copy
  // ---- a1 on rank 0, the subdiagonal to every rank ----
  std::vector<double> sub((size_t)std::max(m - 1, 1), 0.0);
  if (m > 1) {
    CK(c->subd.ensure(sizeof(double) * (size_t)m));
    double* sd = c->subd.as<double>();
    if (root) {
      if (Sh) {
        for (int j = 0; j + 1 < m; ++j) sub[j] = Sh[(size_t)j * ldsh + j + 1];
        CK(cudaMemcpyAsync(sd, sub.data(), sizeof(double) * (m - 1), cudaMemcpyHostToDevice, st));
      } else {
        CK(launch_subdiag(S, lds, m, sd, st));
      }
    }
    if (c->comm && api->broadcast(sd, sd, (size_t)(m - 1), ncclFloat64, 0, c->comm, st) != ncclSuccess)
      return ZZ_ERR_NCCL;
    CK(cudaMemcpyAsync(sub.data(), sd, sizeof(double) * (m - 1), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  std::vector<int> bs, bz;
  const int nb = blocks_host(m, sub.data(), bs, bz);
  if (nb < 0) return nb;
  // ---- ownership: global columns of every shard (block order), the local select ----
  std::vector<std::vector<ShardCol>> cols;
  std::vector<int> sel_loc;
  shard_owners(m, bs, bz, select, P, p, cols, sel_loc);
  const int n_loc = (int)cols[p].size();
  // ---- the local solve: all of S, T's panels stream in; own columns only ----
  const long long ldl = (m + 1) & ~1LL;
  CK(c->Xloc.ensure(sizeof(double) * (size_t)ldl * std::max(n_loc, 1)));
  CK(c->Eloc.ensure(sizeof(int) * (size_t)std::max(n_loc, 1)));
  const double* Sc = S;
  const double* Tc = T;
  long long ldsc = lds, ldtc = ldt;
  if (recv_role) {
    CK(c->Sw.ensure(sizeof(double) * (size_t)ldl * m));
    CK(c->Tw.ensure(sizeof(double) * (size_t)ldl * m));
    Sc = c->Sw.as<double>();
    Tc = c->Tw.as<double>();
    ldsc = ldtc = ldl;
  }
  int r;
  if (c->comm || Sh) {
    size_t pan = 0;   // largest panel pair: 2 x (rows up to the subdiagonal) x mb
    const int mbt = tile_of(c->mb);
    pan = 2 * (size_t)(m + 1) * (size_t)std::min(mbt, m);
    if (c->comm) CK(c->bbuf.ensure(sizeof(double) * pan));
    if (!c->copy) CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    if (!c->e_copy) CK(cudaEventCreateWithFlags(&c->e_copy, cudaEventDisableTiming));
    CK(cudaEventRecord(c->e_copy, st));
    CK(cudaStreamWaitEvent(c->copy, c->e_copy, 0));
    Feed fd;
    fd.Sh = Sh; fd.ldsh = ldsh; fd.Th = Th; fd.ldth = ldth;
    fd.sub = sub.data();
    fd.copy = c->copy;
    fd.ev = &c->ev_copy;
    fd.comm = c->comm;
    fd.api = api;
    fd.root = root;
    fd.Ssrc = S; fd.ldss = lds; fd.Tsrc = T; fd.ldts = ldt;
    fd.bbuf = c->bbuf.as<double>();
    fd.wait = recv_role || Sh != nullptr;
    r = tgevc_device(c, m, Sc, ldsc, Tc, ldtc, sel_loc.data(), c->Xloc.as<double>(), ldl, c->Eloc.as<int>(), &fd);
  } else {
    r = tgevc_device(c, m, Sc, ldsc, Tc, ldtc, sel_loc.data(), c->Xloc.as<double>(), ldl, c->Eloc.as<int>());
  }
  if (r) return r;
  // ---- gather: pack the upper parts (rows 0 .. r_c) of the local columns ----
  Range r_gather("zz.gather");
  auto region = [&](int q, std::vector<long long>* off) -> long long {   // bytes of shard q's buffer
    long long o = 0;
    if (off) off->resize(cols[q].size());
    for (size_t l = 0; l < cols[q].size(); ++l) {
      if (off) (*off)[l] = o;
      o += cols[q][l].r + 1;
    }
    return ((8 * o + 4 * (long long)cols[q].size()) + 15) / 16 * 16;
  };
  // rank 0 unpacks every shard (nranks > 1) or the emulated shard p (one GPU)
  auto unpacked = [&](int q) { return root && (c->nranks > 1 || q == p); };
  std::vector<long long> rbase((size_t)P + 1, 0);
  for (int q = 0; q < P; ++q) rbase[q + 1] = rbase[q] + (unpacked(q) ? region(q, nullptr) : 0);
  std::vector<long long> loff;
  const long long my_bytes = region(p, &loff);
  long long dsum = 0;
  for (int l = 0; l < n_loc; ++l) dsum += cols[p][l].r + 1;
  // pack destination: rank 0's own shard goes straight into its receive region
  const bool self_pack = root && !(c->comm && p != 0);
  CK(c->recvb.ensure((size_t)std::max(rbase[P], (long long)16)));
  if (!self_pack) CK(c->sendb.ensure((size_t)std::max(my_bytes, (long long)16)));
  unsigned char* pk = self_pack ? c->recvb.as<unsigned char>() + rbase[p] : c->sendb.as<unsigned char>();
  {
    // tables: [off (int64) | h (int32)]
    std::vector<long long> tb((size_t)n_loc * 2);
    for (int l = 0; l < n_loc; ++l) { tb[l] = loff[l]; reinterpret_cast<int*>(tb.data() + n_loc)[l] = cols[p][l].r + 1; }
    CK(c->gtab.ensure(sizeof(long long) * 2 * (size_t)std::max(n_loc, 1) + 16));
    if (n_loc > 0) CK(cudaMemcpyAsync(c->gtab.p, tb.data(), sizeof(long long) * 2 * n_loc, cudaMemcpyHostToDevice, st));
    CK(launch_shard_pack(c->Xloc.as<double>(), ldl, c->Eloc.as<int>(), n_loc, c->gtab.as<long long>(),
                         reinterpret_cast<const int*>(c->gtab.as<long long>() + n_loc),
                         reinterpret_cast<double*>(pk), reinterpret_cast<int*>(pk + 8 * dsum), st));
    CK(cudaStreamSynchronize(st));   // the tables are host vectors
  }
  if (c->comm) {
    if (api->groupStart() != ncclSuccess) return ZZ_ERR_NCCL;
    bool ok = true;
    if (!self_pack) ok &= api->send(pk, (size_t)my_bytes, ncclUint8, 0, c->comm, st) == ncclSuccess;
    if (root) {
      for (int q = 0; q < P; ++q) {
        if (!unpacked(q) || (q == p && self_pack)) continue;
        const int src = (c->nranks > 1) ? q : 0;
        ok &= api->recv(c->recvb.as<unsigned char>() + rbase[q], (size_t)(rbase[q + 1] - rbase[q]), ncclUint8, src,
                        c->comm, st) == ncclSuccess;
      }
    }
    if (api->groupEnd() != ncclSuccess || !ok) return ZZ_ERR_NCCL;
  }
  // ---- rank 0: every received column into its global position of X ----
  if (root) {
    std::vector<long long> bo, beo;
    std::vector<int> hh, gg;
    for (int q = 0; q < P; ++q) {
      if (!unpacked(q)) continue;
      std::vector<long long> off;
      region(q, &off);
      long long ds = 0;
      for (const ShardCol& sc : cols[q]) ds += sc.r + 1;
      for (size_t l = 0; l < cols[q].size(); ++l) {
        bo.push_back(rbase[q] + 8 * off[l]);
        beo.push_back(rbase[q] + 8 * ds + 4 * (long long)l);
        hh.push_back(cols[q][l].r + 1);
        gg.push_back(cols[q][l].g);
      }
    }
    const int ne = (int)gg.size();
    CK(c->gtab.ensure((sizeof(long long) * 2 + sizeof(int) * 2) * (size_t)std::max(ne, 1) + 16));
    long long* tb = c->gtab.as<long long>();
    if (ne > 0) {
      CK(cudaMemcpyAsync(tb, bo.data(), sizeof(long long) * ne, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(tb + ne, beo.data(), sizeof(long long) * ne, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(tb + 2 * ne, hh.data(), sizeof(int) * ne, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(reinterpret_cast<int*>(tb + 2 * ne) + ne, gg.data(), sizeof(int) * ne, cudaMemcpyHostToDevice, st));
    }
    CK(launch_shard_unpack(c->recvb.as<unsigned char>(), ne, tb, tb + ne, reinterpret_cast<const int*>(tb + 2 * ne),
                           reinterpret_cast<const int*>(tb + 2 * ne) + ne, m, X, ldx, cse, st));
    CK(cudaStreamSynchronize(st));
  } else {
    CK(cudaStreamSynchronize(st));
  }
  c->info.n_sel = n_loc;
  c->info.d_logmax = c->info.d_a = c->info.d_b = c->info.d_beta = nullptr;   // local columns only
  return 0;
}

int check_args(int m, const double* S, int lds, const double* T, int ldt, double* X, int ldx) {
  if (m < 0) return -1;
  if (m > 0 && !S) return -2;
  if (lds < std::max(1, m)) return -3;
  if (m > 0 && !T) return -4;
  if (ldt < std::max(1, m)) return -5;
  if (m > 0 && !X) return -7;
  if (ldx < std::max(1, m)) return -8;
  return 0;
}

}  // namespace

// Context access for the complex-pencil path (zz_complex.cu): binds the device and hands out
// the stream, tile and info record.
int ctx_acquire(cudaStream_t* st, int* mb, int* lookahead, zz_info_t** info) {
  Context* c = g_ctx;
  if (!c) return ZZ_ERR_NOCTX;
  if (cudaSetDevice(c->device) != cudaSuccess) return ZZ_ERR_CUDA;
  *st = c->stream;
  *mb = c->mb;
  *lookahead = c->lookahead;
  *info = &c->info;
  return 0;
}

int ctx_fusion() { return g_ctx ? g_ctx->fusion : 1; }
int ctx_fusion_explicit() { return g_ctx && g_ctx->fusion_explicit; }
// zz_ztgevc's workspace, kept by the context between calls (nullptr: out of memory)
void* ctx_zwork(size_t bytes) { return (g_ctx && g_ctx->zw.ensure(bytes) == cudaSuccess) ? g_ctx->zw.p : nullptr; }

extern "C" {

int zz_get_unique_id(unsigned char* id) {
  if (!id) return -1;
  const NcclApi* api = nccl_api();
  if (!api) return ZZ_ERR_NCCL;
  ncclUniqueId u;
  if (api->getUniqueId(&u) != ncclSuccess) return ZZ_ERR_NCCL;
  memcpy(id, u.internal, sizeof(u.internal));
  return 0;
}

int zz_init(int device, int nranks, int rank, const unsigned char* id) {
  if (nranks < 1) return -2;
  if (rank < 0 || rank >= nranks) return -3;
  if (nranks > 1 && !id) return -4;
  int nd = 0;
  if (cudaGetDeviceCount(&nd) != cudaSuccess || device < 0 || device >= nd) return ZZ_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return ZZ_ERR_CUDA;
  if (g_ctx && (g_ctx->device != device || g_ctx->comm || id)) {
    g_ctx->release();
    delete g_ctx;
    g_ctx = nullptr;
  }
  if (!g_ctx) {
    g_ctx = new Context();
    memset(&g_ctx->info, 0, sizeof(g_ctx->info));
  }
  g_ctx->device = device;
  g_ctx->nranks = nranks;
  g_ctx->rank = rank;
  g_ctx->shard_p = 0;
  g_ctx->shard_P = 1;
  if (id) {
    const NcclApi* api = nccl_api();
    if (!api) return ZZ_ERR_NCCL;
    ncclUniqueId u;
    memcpy(u.internal, id, sizeof(u.internal));
    if (api->commInitRank(&g_ctx->comm, nranks, u, rank) != ncclSuccess) {
      g_ctx->comm = nullptr;
      return ZZ_ERR_NCCL;
    }
  }
  return 0;
}

int zz_set_shard(int p, int P) {
  if (!g_ctx) return ZZ_ERR_NOCTX;
  if (P < 1 || P > 4096) return -2;
  if (p < 0 || p >= P) return -1;
  if (g_ctx->nranks > 1) return ZZ_ERR_SHARD;
  g_ctx->shard_p = p;
  g_ctx->shard_P = P;
  return 0;
}

int zz_set_stream(void* stream) {
  if (!g_ctx) return ZZ_ERR_NOCTX;
  g_ctx->stream = reinterpret_cast<cudaStream_t>(stream);
  return 0;
}

int zz_set_tile(int mb) {
  if (!g_ctx) return ZZ_ERR_NOCTX;
  if (mb != 0 && (mb < 32 || mb > kMaxMB || (mb % 16) != 0)) return ZZ_ERR_TILE;
  g_ctx->mb = mb;
  return 0;
}

int zz_set_fusion(int k) {
  if (!g_ctx) return ZZ_ERR_NOCTX;
  if (k < 0 || k > kMaxGroup) return -1;
  g_ctx->fusion = k ? k : 4;          // 0: the library defaults
  g_ctx->fusion_explicit = k != 0;
  return 0;
}

int zz_set_lookahead(int mode) {
  if (!g_ctx) return ZZ_ERR_NOCTX;
  if (mode < 0 || mode > 2) return -1;
  g_ctx->lookahead = mode;
  return 0;
}

int zz_set_diag_team(int w) {
  if (!g_ctx) return ZZ_ERR_NOCTX;
  if (!(w == -1 || w == 0 || w == 1 || w == 2 || w == 3 || w == 4 || w == 6 || w == 8 || w == 12 || w == 16)) return -1;
  g_ctx->diag_team = w;
  return 0;
}

int zz_set_graphs(int on) {
  if (!g_ctx) return ZZ_ERR_NOCTX;
  g_ctx->graphs = on ? 1 : 0;
  if (!on && g_ctx->gexec) {
    cudaGraphExecDestroy(g_ctx->gexec);
    g_ctx->gexec = nullptr;
    g_ctx->gkey = 0;
  }
  return 0;
}

int zz_set_timing(int on) {
  if (!g_ctx) return ZZ_ERR_NOCTX;
  g_ctx->timing = on ? 1 : 0;
  return 0;
}

int zz_tgevc(int m, const double* S, int lds, const double* T, int ldt, const int* select, double* X,
             int ldx, int* col_scale_exp) {
  Context* c = g_ctx;
  // collective call: only rank 0 passes S, T, X (the other ranks' pointers are ignored)
  const bool nonroot = c && c->nranks > 1 && c->rank != 0;
  int a = nonroot ? (m < 0 ? -1 : 0) : check_args(m, S, lds, T, ldt, X, ldx);
  if (a) return a;
  if (!c) return ZZ_ERR_NOCTX;
  if (cudaSetDevice(c->device) != cudaSuccess) return ZZ_ERR_CUDA;
  if (m == 0) {
    memset(&c->info, 0, sizeof(c->info));
    return 0;
  }
  if (c->nranks > 1 || c->shard_P > 1 || c->comm)
    return tgevc_sharded(c, m, S, lds, T, ldt, select, X, ldx, col_scale_exp);
  return tgevc_device(c, m, S, lds, T, ldt, select, X, ldx, col_scale_exp);
}

int zz_tgevc_back(int m, const double* S, int lds, const double* T, int ldt, const int* select,
                  const double* V, int ldv, double* W, int ldw, int* col_scale_exp) {
  int a = check_args(m, S, lds, T, ldt, W, ldw);
  if (a == -7 || a == -8) a -= 2;     // W, ldw are arguments 9 and 10
  if (a) return a;
  if (m > 0 && !V) return -7;
  if (ldv < std::max(1, m)) return -8;
  if (!g_ctx) return ZZ_ERR_NOCTX;
  if (cudaSetDevice(g_ctx->device) != cudaSuccess) return ZZ_ERR_CUDA;
  if (m == 0) {
    memset(&g_ctx->info, 0, sizeof(g_ctx->info));
    return 0;
  }
  return tgevc_back_device(g_ctx, m, S, lds, T, ldt, select, V, ldv, W, ldw, col_scale_exp);
}

int zz_tgevc_left(int m, const double* S, int lds, const double* T, int ldt, const int* select, double* Y,
                  int ldy, int* col_scale_exp) {
  int a = check_args(m, S, lds, T, ldt, Y, ldy);
  if (a) return a;
  if (!g_ctx) return ZZ_ERR_NOCTX;
  if (cudaSetDevice(g_ctx->device) != cudaSuccess) return ZZ_ERR_CUDA;
  if (m == 0) {
    memset(&g_ctx->info, 0, sizeof(g_ctx->info));
    return 0;
  }
  return tgevc_left_device(g_ctx, m, S, lds, T, ldt, select, Y, ldy, col_scale_exp);
}

int zz_tgevc_host(int m, const double* S, int lds, const double* T, int ldt, const int* select, double* X,
                  int ldx, int* col_scale_exp) {
  Context* c = g_ctx;
  const bool nonroot = c && c->nranks > 1 && c->rank != 0;
  int a = nonroot ? (m < 0 ? -1 : 0) : check_args(m, S, lds, T, ldt, X, ldx);
  if (a) return a;
  if (!c) return ZZ_ERR_NOCTX;
  if (cudaSetDevice(c->device) != cudaSuccess) return ZZ_ERR_CUDA;
  if (m == 0) return 0;
  const bool coll = c->nranks > 1 || c->comm;
  if (c->shard_P > 1) return ZZ_ERR_SHARD;     // the one-GPU shard emulation is device-only
  if (nonroot) return tgevc_sharded(c, m, nullptr, 0, nullptr, 0, select, nullptr, 0, nullptr);
  int n_sel = zz_count_columns(m, S, lds, select);
  if (n_sel < 0) return n_sel;
  cudaStream_t st = c->stream;
  long long ld = (m + 1) / 2 * 2;
  CK(c->hS.ensure(sizeof(double) * (size_t)ld * m));
  CK(c->hT.ensure(sizeof(double) * (size_t)ld * m));
  CK(c->hX.ensure(sizeof(double) * (size_t)ld * std::max(n_sel, 1)));
  CK(c->hE.ensure(sizeof(int) * (size_t)std::max(n_sel, 1)));
  if (!c->copy) CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
  // the copy stream starts after everything already queued on the context's stream
  if (!c->e_copy) CK(cudaEventCreateWithFlags(&c->e_copy, cudaEventDisableTiming));
  CK(cudaEventRecord(c->e_copy, st));
  CK(cudaStreamWaitEvent(c->copy, c->e_copy, 0));
  Feed hs;
  hs.Sh = S; hs.ldsh = lds; hs.Th = T; hs.ldth = ldt; hs.copy = c->copy; hs.ev = &c->ev_copy;
  hs.Ssrc = c->hS.as<double>(); hs.ldss = ld; hs.Tsrc = c->hT.as<double>(); hs.ldts = ld;
  // X is block-upper-triangular: column c is zero below its last row r_c.  Only the upper
  // part travels back over PCIe (one 2D copy per 64-column block, rows 0 .. the block's
  // largest r_c); the zeros below are written by host threads while the GPU solves (the
  // regions are disjoint, and the device never touches X before the download).
  std::vector<int> rmax;   // per 64-column block
  {
    int col = 0, j = 0;
    rmax.assign((size_t)(n_sel + 63) / 64, -1);
    while (j < m) {
      const bool two = j + 1 < m && S[(size_t)j * lds + j + 1] != 0.0;
      const int sz = two ? 2 : 1;
      if (!select || select[j] || (two && select[j + 1]))
        for (int q = 0; q < sz; ++q, ++col) rmax[col / 64] = j + sz - 1;
      j += sz;
    }
  }
  const int nthr = std::max(1, std::min(8, (int)std::thread::hardware_concurrency() / 2));
  std::vector<std::thread> zt;
  for (int w = 0; w < nthr && n_sel > 0; ++w)
    zt.emplace_back([=, &rmax]() {
      for (int cb = w; cb < (int)rmax.size(); cb += nthr) {
        const int r0 = rmax[cb] + 1;
        if (r0 >= m) continue;
        for (int cc = cb * 64; cc < std::min(n_sel, cb * 64 + 64); ++cc)
          memset(X + (size_t)cc * ldx + r0, 0, sizeof(double) * (size_t)(m - r0));
      }
    });
  int r = coll ? tgevc_sharded(c, m, c->hS.as<double>(), ld, c->hT.as<double>(), ld, select, c->hX.as<double>(), ld,
                               c->hE.as<int>(), S, lds, T, ldt)
               : tgevc_device(c, m, c->hS.as<double>(), ld, c->hT.as<double>(), ld, select, c->hX.as<double>(), ld,
                              c->hE.as<int>(), &hs);
  for (auto& th : zt) th.join();
  if (r) return r;
  if (n_sel > 0) {
    for (int cb = 0; cb < (int)rmax.size(); ++cb) {
      const int c0 = cb * 64, nc = std::min(64, n_sel - c0);
      CK(cudaMemcpy2DAsync(X + (size_t)c0 * ldx, (size_t)ldx * 8, c->hX.as<double>() + (size_t)c0 * ld, ld * 8,
                           (size_t)(rmax[cb] + 1) * 8, nc, cudaMemcpyDeviceToHost, st));
    }
    if (col_scale_exp)
      CK(cudaMemcpyAsync(col_scale_exp, c->hE.p, sizeof(int) * n_sel, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return 0;
}

int zz_count_columns(int m, const double* S_host, int lds, const int* select) {
  if (m < 0) return -1;
  if (m > 0 && !S_host) return -2;
  if (lds < std::max(1, m)) return -3;
  int n = 0, j = 0;
  while (j < m) {
    bool two = (j + 1 < m) && S_host[(size_t)j * lds + j + 1] != 0.0;
    if (two && j + 2 < m && S_host[(size_t)(j + 1) * lds + j + 2] != 0.0) return ZZ_ERR_OVERLAP;
    int sz = two ? 2 : 1;
    if (!select || select[j] || (two && select[j + 1])) n += sz;
    j += sz;
  }
  return n;
}

int zz_partition(int m, const double* sub, int mb, int* tile_start) {
  if (m < 0) return -1;
  if (mb < 2) return ZZ_ERR_TILE;
  std::vector<double> s((size_t)std::max(m, 1), 0.0);
  if (m > 1) memcpy(s.data(), sub, sizeof(double) * (m - 1));
  std::vector<int> bs, bz;
  int nb = blocks_host(m, s.data(), bs, bz);
  if (nb < 0) return nb;
  std::vector<char> two_bot((size_t)m + 1, 0);
  for (int p = 0; p < nb; ++p)
    if (bz[p] == 2) two_bot[bs[p] + 1] = 1;
  std::vector<int> ts;
  int M = partition_host(m, two_bot, mb, ts);
  for (int I = 0; I <= M; ++I) tile_start[I] = ts[I];
  return M;
}

int zz_shard_columns(int m, const double* sub, const int* select, int P, int p, int* cols) {
  if (m < 0) return -1;
  if (P < 1) return -4;
  if (p < 0 || p >= P) return -5;
  std::vector<double> s((size_t)std::max(m, 1), 0.0);
  if (m > 1) {
    if (!sub) return -2;
    memcpy(s.data(), sub, sizeof(double) * (m - 1));
  }
  std::vector<int> bs, bz;
  const int nb = blocks_host(m, s.data(), bs, bz);
  if (nb < 0) return nb;
  std::vector<std::vector<ShardCol>> own;
  std::vector<int> sel_loc;
  shard_owners(m, bs, bz, select, P, p, own, sel_loc);
  if (cols)
    for (size_t l = 0; l < own[p].size(); ++l) cols[l] = own[p][l].g;
  return (int)own[p].size();
}

int zz_last_info(zz_info_t* out) {
  if (!g_ctx) return ZZ_ERR_NOCTX;
  if (out) *out = g_ctx->info;
  return 0;
}

int zz_finalize(void) {
  if (g_ctx) {
    g_ctx->release();
    delete g_ctx;
    g_ctx = nullptr;
  }
  return 0;
}

const char* zz_status_string(int s) {
  if (s == 0) return "success";
  if (s > 0) return "a 2x2 diagonal block has real eigenvalues (assumption 2 violated)";
  switch (s) {
    case ZZ_ERR_CUDA: return "CUDA error (or no CUDA device)";
    case ZZ_ERR_NOMEM: return "out of device memory";
    case ZZ_ERR_NOCTX: return "no context: call zz_init first";
    case ZZ_ERR_NONFINITE: return "non-finite entry in a diagonal block of S or T";
    case ZZ_ERR_OVERLAP: return "overlapping 2x2 blocks (two consecutive nonzero subdiagonals)";
    case ZZ_ERR_TILE: return "unsupported tile size";
    case ZZ_ERR_CPLXDIAG: return "a diagonal entry of T is not real (zz_ztgevc)";
    case ZZ_ERR_NCCL: return "NCCL error (or NCCL not available)";
    case ZZ_ERR_SHARD: return "zz_set_shard: not with a multi-rank context / not for this call";
    default: return (s >= -9) ? "invalid argument" : "unknown status";
  }
}

}  // extern "C"
