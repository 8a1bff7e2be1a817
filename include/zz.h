/*
 * include/zz.h -- C ABI of the B200-native robust generalized-eigenvector solver.
 *
 * Operation.  For a real pencil (S,T) in generalized real Schur form (PAPER.md:56-61:
 * S quasi-upper-triangular with 1x1 and 2x2 diagonal blocks, T upper triangular) compute
 * the right generalized eigenvectors, i.e. the columns of V in the homogeneous matrix
 * equation  S V D - T V B = 0, D diagonal and B block diagonal
 * as in PAPER.md:83-99, by the robust blocked back-substitution of Algorithm 1
 * with augmented matrices and int32 power-of-two scaling exponents
 * (PAPER.md:202-268).  All matrices are FP64, column-major (LAPACK convention).
 *
 * Conventions (those of LAPACK xTGEVC, verified as a black box in
 * tests/test_oracle_vectors.py):
 *  - a real eigenvalue gives one column; a complex pair gives two columns [Re z, Im z] of
 *    the eigenvector z for the eigenvalue with positive imaginary part;
 *  - columns are normalised so that max_i |x_i| = 1 (real) or max_i (|x_i| + |y_i|) = 1
 *    (pair); rows below the eigenvalue's diagonal block are exactly 0;
 *  - an indefinite 1x1 block (alpha = beta = 0) gives the unit vector e_j.
 *
 * Status codes (int return value, LAPACK INFO style):
 *     0   success
 *    -i   argument i of zz_tgevc / zz_tgevc_host is invalid (1-based)
 *    +j   the 2x2 diagonal block S(j:j+1, j:j+1) (1-based) has real eigenvalues
 *         (assumption 2 of PAPER.md:69 violated); zz_tgevc does not write X.  zz_tgevc_host
 *         learns the status only after the wavefront: it may already have written the zeros
 *         below each column's block into the caller's host X (the same holds for -104)
 *  -100   CUDA error      -102 out of device memory      -103 no context (zz_init missing)
 *  -104   non-finite entry in a diagonal block of S or T
 *  -105   overlapping 2x2 blocks (two consecutive nonzero subdiagonal entries of S)
 *  -106   unsupported tile size
 *  -107   zz_ztgevc: a diagonal entry of T is not real
 * There is no CPU fallback: without a CUDA device every call returns -100 or -103.
 *
 * Threading and multi-GPU.  One context per host thread (thread-local), bound to one device.
 * Calls on a context are not reentrant.  Multi-GPU (one process per GPU):
 * zz_get_unique_id on rank 0, the 128 bytes shipped to the other ranks by the caller (e.g.
 * torch.distributed), zz_init(device, nranks, rank, id) on every rank; zz_tgevc and
 * zz_tgevc_host are then collective.  The task graph of the method is the disjoint union of
 * per-column-block subgraphs: eigenvalue blocks are owned in groups of 64 rows
 * cyclically over the ranks, every rank runs the whole bottom-up wavefront over its own
 * columns, S and T are broadcast from rank 0 (NCCL, panel by panel in the order the wavefront
 * consumes them, upper part only, overlapped with the solve), and the finished columns (rows
 * 0 .. r_c) are gathered on rank 0.  X is bitwise independent of the number of ranks.
 */
#ifndef ZZ_H
#define ZZ_H

#ifdef __cplusplus
extern "C" {
#endif

#define ZZ_OK 0
#define ZZ_ERR_CUDA (-100)
#define ZZ_ERR_NCCL (-101)
#define ZZ_ERR_NOMEM (-102)
#define ZZ_ERR_NOCTX (-103)
#define ZZ_ERR_NONFINITE (-104)
#define ZZ_ERR_OVERLAP (-105)
#define ZZ_ERR_TILE (-106)
#define ZZ_ERR_CPLXDIAG (-107)
#define ZZ_ERR_SHARD (-108)

/* Statistics of the last zz_tgevc call of this thread's context. */
typedef struct zz_info {
  int m;              /* order of the pencil */
  int n_sel;          /* number of output columns */
  int mb;             /* tile size used */
  int n_tiles;        /* M, number of tile rows (steps of the wavefront) */
  int n_scaled;       /* columns with col_scale_exp < 0 */
  int min_exp;        /* min col_scale_exp (0 if none scaled) */
  int n_indefinite;   /* indefinite eigenvalues among the selected ones */
  int prescaled;      /* 1 if S or T was pre-scaled by a power of two (reading R6) */
  int update_launches;     /* robust-update kernel launches */
  int total_launches;      /* all kernel launches of the call */
  int fused_pairs;         /* step groups whose updates ran as one multi-tile contraction */
  int lookahead_redo;      /* 1 if the lookahead schedule had to be recomputed without it */
  double ms_setup;         /* structure scan, pairs, norms */
  double ms_steps;         /* the wavefront (diagonal solves + updates) */
  double ms_normalize;     /* consistency and normalisation */
  double ms_update;        /* summed device time of the robust-update kernels (if timed) */
  double ms_back;          /* zz_tgevc_back: back-transformation GEMMs + normalisation */
  /* DEVICE views into the library workspace, n_sel doubles each in output
   * column order; valid until the next call on this context; NULL when n_sel == 0 and after
   * zz_tgevc_left / zz_ztgevc.  Read-only for the caller.
   *   logmax   L_c = log2(max_i measure of the stored column before normalisation) - e_c,
   *            i.e. log2 of the max measure of the tip-normalised eigenvector (x_r = 1,
   *            PAPER.md:152; Definition 1); measure |x_i| (real) or
   *            |x_i| + |y_i| (pair); -inf for an all-zero column (never produced)
   *   a, b, beta  the power-of-two normalised eigenvalue pair (alpha = a + i b, PAPER.md:72,
   *            79-99) the pivots beta S_ii - alpha T_ii were formed with; both columns of a
   *            pair carry the same values (b > 0); real columns have b = 0 */
  const double* d_logmax;
  const double* d_a;
  const double* d_b;
  const double* d_beta;
} zz_info_t;

/* 128-byte NCCL unique id for zz_init (call on rank 0, ship the bytes to every rank).
 * Returns 0, -1 (id NULL) or -101 (NCCL not available: it is loaded at run time). */
int zz_get_unique_id(unsigned char* id);

/* Create (or re-bind) this thread's context on CUDA device `device` as rank `rank` of
 * `nranks` processes (one per GPU).  id: the 128 bytes of zz_get_unique_id, or NULL iff
 * nranks == 1 (no communicator).  With an id the call is collective (ncclCommInitRank):
 * every rank blocks until all have joined.  nranks = 1 with an id creates a one-rank
 * communicator: zz_tgevc then runs its collective code path on one GPU (broadcast and
 * gather to itself; used by the tests).  Returns 0, -2 (nranks < 1), -3 (bad rank),
 * -4 (id NULL with nranks > 1), -100 (no such device) or -101 (NCCL). */
int zz_init(int device, int nranks, int rank, const unsigned char* id);

/* One-GPU emulation of a rank's share (single-rank contexts only): subsequent zz_tgevc calls
 * compute only the columns that rank p of P would own (eigenvalue blocks with first row j
 * such that (j / 64) mod P == p) and write them into their global positions of X (the
 * columns of X that belong to other shards are not written; col_scale_exp likewise).
 * Running p = 0 .. P-1 into one X assembles, bit for bit, the X of a plain call.  With a
 * one-rank communicator, p != 0 also takes the non-root data path (S, T from the broadcast
 * copy, columns through NCCL send/recv).  zz_set_shard(0, 1) restores the plain call.
 * zz_tgevc_host rejects an emulated shard (-108).  Returns 0, -1 / -2 (bad p / P), -103,
 * or -108 (the context has nranks > 1). */
int zz_set_shard(int p, int P);

/* Stream for subsequent calls (a cudaStream_t passed as void*; NULL = legacy default
 * stream).  The stream is borrowed, never destroyed.  Returns 0 or -103. */
int zz_set_stream(void* stream);

/* Tile size mb (rows of the diagonal tiles): 0 = automatic (128), or a
 * multiple of 16 in [32, 160].  A tile boundary that would split a 2x2 block moves up one
 * row (reading R12).  Returns 0, -103 or -106. */
int zz_set_tile(int mb);

/* CUDA graph of the wavefront: 1 (default) captures the launch sequence
 * of a call's wavefront once and replays it while the plan (sizes, block structure,
 * selection, tile, step groups, lookahead) and every pointer it uses are unchanged -- the
 * same kernels in the same order, so results are bitwise those of 0 (plain stream launches).
 * Not used by the host-staged or collective paths.  Returns 0 or -103. */
int zz_set_graphs(int on);

/* Warps per diagonal-solve task (DESIGN.md s.6 "Teams"): the tile's 8-row blocks of a task's
 * columns are split into W contiguous ranges, one per warp; the chain of blocks runs through
 * the warps and every warp applies each solved block to its own rows with the same
 * instructions, so results are bitwise independent of W.  0 (default) = one warp per task
 * (measured fastest); -1 = as many warps per task as keep the step's tasks in one wave over
 * the SMs; W in {1, 2, 3, 4, 6, 8, 12, 16} forces W where it divides the kernel's warps per
 * CTA and the shared memory allows (otherwise 1).  Returns 0, -1 or -103. */
int zz_set_diag_team(int w);

/* Per-kernel timing of the robust update with CUDA events (0 off, 1 on): fills
 * zz_info_t.ms_update.  Adds an event pair per step; used by bench.py for the roofline. */
int zz_set_timing(int on);

/* Step grouping of the wavefront for this thread's context: k consecutive steps share one
 * update of the rows above them with K = k tiles (1 = the paper's one update per step; 2 =
 * pairs; 3 = triples; 4 = the default; up to 6).  Results differ only by summation order and by
 * how conservative the scaling bounds are (DESIGN.md s.6); groups are fixed by the tile
 * index, so results never depend on `select`.  Tiles of more than 128 rows always run
 * ungrouped.  zz_ztgevc groups min(k, 4) steps (its decisions use the pending bound, so
 * they are those of the ungrouped schedule; results differ by summation order only); until
 * zz_set_fusion is called it picks 1..4 from the number of tile rows (m / tile + 16) / 32.
 * k = 0 restores the defaults (4; zz_ztgevc by the number of tile rows).
 * Returns 0, -1 (k not in 0..6) or -103. */
int zz_set_fusion(int k);

/* Lookahead schedule: the chain of diagonal solves of a step group runs on a high-priority
 * stream beside the bulk of the previous group's update (DESIGN.md s.6 "Lookahead").  The
 * first and the last decision of a group then use a recorded upper bound of the pending rows
 * instead of their measured maximum; where that bound would make one scale, the call is recomputed
 * without lookahead (zz_info_t.lookahead_redo), so results are always those of the plain
 * schedule, bit for bit.  mode 0 = off, 1 = automatic (default: on for m >= 1024 unless a
 * panel norm exceeds 2^64), 2 = on whenever step groups are used.  Returns 0, -1 or -103. */
int zz_set_lookahead(int mode);

/*
 * zz_tgevc: selected right eigenvectors on the device.
 *   m              order of S and T (m >= 0)                                   [arg 1]
 *   S, lds         DEVICE, m x m column-major, lds >= max(1,m); never written  [args 2,3]
 *   T, ldt         DEVICE, m x m column-major, ldt >= max(1,m); never written  [args 4,5]
 *   select         HOST int[m] or NULL (all eigenvectors).  select[j] != 0 picks
 *                  eigenvalue j; a complex pair (j, j+1) is computed if either flag is
 *                  set.  Output columns are packed in block order.           [arg 6]
 *   X, ldx         DEVICE, m x n_sel column-major, ldx >= max(1,m); written
 *                  completely (including the zeros below each column's block).
 *                  An odd ldx or a base not 16-byte aligned is solved in an internal
 *                  aligned m x n_sel workspace and copied out: results are bitwise
 *                  independent of ldx.                                          [args 7,8]
 *   col_scale_exp  DEVICE int32[n_sel] or NULL: e_c <= 0 such that the tip-normalised
 *                  eigenvector (x_r = 1) is 2^-e_c times the column before
 *                  normalisation (Definition 1).  Both columns of a
 *                  pair carry the same e_c.  Values are implementation-defined.  [arg 9]
 * The strictly lower parts of S (outside the 2x2 blocks) and of T are never read.
 * Work runs on the context's stream; the call returns after the stream has completed.
 * Ownership: S, T, X, col_scale_exp are caller-owned; the library owns a workspace grown
 * on demand and freed by zz_finalize.
 * Multi-rank context (zz_init with nranks > 1): collective; every rank passes the same m and
 * select; rank 0 passes S, T, X, col_scale_exp, the other ranks' pointer and leading-
 * dimension arguments are ignored (pass NULL / 0).  On return rank 0 holds the full X.  The
 * non-root ranks keep a library copy of S and T (2 m^2 doubles) and of their own columns.
 * Status -101 for an NCCL failure.  zz_last_info describes the rank's own columns (n_sel =
 * local columns, device views NULL).
 */
int zz_tgevc(int m, const double* S, int lds, const double* T, int ldt, const int* select,
             double* X, int ldx, int* col_scale_exp);

/* zz_tgevc_host: the same operation with HOST S, T, X, col_scale_exp (pinned memory
 * recommended).  The library stages S and T into device memory, solves, and copies X and
 * col_scale_exp back, all on the context's stream (end-to-end path of bench.py).
 * Arguments and status codes as zz_tgevc; collective on a multi-rank context (rank 0's host
 * panels go up and out by broadcast as they arrive).  On a nonzero status the rows of X
 * below each selected column's diagonal block may already have been set to zero (they are
 * written by host threads while the device solves); nothing else of X is written. */
int zz_tgevc_host(int m, const double* S, int lds, const double* T, int ldt, const int* select,
                  double* X, int ldx, int* col_scale_exp);

/* zz_tgevc_back: back-transformed eigenvectors, the xTGEVC HOWMNY='B' mode (PAPER.md:28-32:
 * with S = U^T A V and T = U^T B V from the QZ step, S z = lambda T z implies
 * A (V z) = lambda B (V z); the back-transform uses V, not U).
 *   m, S, lds, T, ldt, select   as zz_tgevc                                 [args 1-6]
 *   V, ldv         DEVICE, m x m column-major, ldv >= max(1,m); never written
 *                  (the right Schur vectors; any real matrix is accepted)     [args 7,8]
 *   W, ldw         DEVICE, m x n_sel column-major, ldw >= max(1,m); written
 *                  completely: W(:,c) = V(:, 0:r_c) X(0:r_c, c) with X the
 *                  zz_tgevc result of column c (r_c its last row), then
 *                  normalised as LAPACK does after its back-transform:
 *                  max_i |w_i| = 1 (real), max_i (|Re w_i| + |Im w_i|) = 1 (pair).
 *                  W must not overlap V, S or T.                              [args 9,10]
 *   col_scale_exp  DEVICE int32[n_sel] or NULL: as zz_tgevc (the exponents of the
 *                  (S,T) eigenvectors before their normalisation)             [arg 11]
 * The product is one FP64 tensor-core contraction (DMMA) of this library over tiles of 64
 * columns with K = 1 + the tile's largest r_c (X is block-upper-triangular, so the work is
 * ~ m^3 flop for all eigenvectors instead of 2 m^3); the column maxima come from its epilogue
 * and the normalisation is one pass over W.  The library keeps an m x n_sel workspace for X
 * and a tile-packed copy of its upper part.  V may have any leading dimension (an odd one
 * or a misaligned base is copied to an aligned workspace).  Status codes as zz_tgevc.
 */
int zz_tgevc_back(int m, const double* S, int lds, const double* T, int ldt, const int* select,
                  const double* V, int ldv, double* W, int ldw, int* col_scale_exp);

/* zz_tgevc_left: selected LEFT eigenvectors y, y^H S = lambda y^H T (PAPER.md:330 names them
 * as the next step; LAPACK xTGEVC SIDE='L' conventions).  Arguments as zz_tgevc, with
 *   Y, ldy         DEVICE, m x n_sel column-major; written completely.  Column order, pair
 *                  layout (Re y, Im y for the eigenvalue with positive imaginary part) and
 *                  normalisation (max |y| = 1, pairs max |Re|+|Im| = 1) as zz_tgevc; y_i = 0
 *                  exactly above the eigenvalue's block (rows < its first row).  [args 7,8]
 *   col_scale_exp  as zz_tgevc, for the left vectors before normalisation.       [arg 9]
 * Method: (beta S^T - conj(alpha) T^T) y = 0; with the reversal J, (J S^T J, J T^T J) is a real
 * Schur pencil with the same eigenvalues, and J conj(y) is its right eigenvector, which the
 * robust blocked path computes (csrc/zz_left.cu: one tiled flip-transpose of each matrix
 * into a library workspace of 2 m^2 doubles, the solve, one gather back).  A status +j
 * refers to rows of S.  Ownership and errors as zz_tgevc. */
int zz_tgevc_left(int m, const double* S, int lds, const double* T, int ldt, const int* select,
                  double* Y, int ldy, int* col_scale_exp);

/* zz_ztgevc: selected right eigenvectors of a COMPLEX pencil in generalized complex Schur
 * form (the ZTGEVC analogue; PAPER.md:333 names complex pencils as the next step): S and T
 * upper triangular, T with a real diagonal.  For (alpha, beta) = (S_jj, T_jj) the eigenvector
 * z solves (beta S - alpha T) z = 0 with z_i = 0 for i > j (Lemma 1, all
 * blocks 1x1), computed by the robust blocked substitution (Algorithms 1-3)
 * with complex entries (readings R18-R21).
 *   m              order (m >= 0)                                                [arg 1]
 *   S, lds         DEVICE, m x m complex column-major, INTERLEAVED (re, im) doubles
 *                  (LAPACK COMPLEX*16 layout), base 16-byte aligned (else -2); lds in
 *                  complex elements; never written.  The strictly lower part is never
 *                  read.                                                        [args 2,3]
 *   T, ldt         DEVICE, as S (16-byte aligned, else -4); Im T_jj must be 0 (else -107)
 *                                                                                [args 4,5]
 *   select         HOST int[m] or NULL (all); select[j] != 0 picks eigenvalue j; output
 *                  columns in increasing j.                                      [arg 6]
 *   X, ldx         DEVICE, m x n_sel complex interleaved, ldx (complex elements) >= m,
 *                  base 16-byte aligned (else -7); written completely: z_i = 0 for i > j, normalised as ZTGEVC does,
 *                  max_i (|Re z_i| + |Im z_i|) = 1, from a real positive z_j before
 *                  normalisation; alpha = beta = 0 gives e_j.                  [args 7,8]
 *   col_scale_exp  DEVICE int32[n_sel] or NULL: exponents as zz_tgevc.            [arg 9]
 * Tiles of zz_set_tile() rows when it is 32, 48 or 64, else 64 (fastest,
 * profiles/r01o_complex_tile_sweep.txt).  The update of a step group (zz_set_fusion, at
 * most 4 steps) is one complex contraction of K = 2 x tile per step (this library's DMMA
 * kernel, Gauss's three-multiplication form, R23) over fragment-ordered copies of
 * the S and T panels; zz_set_lookahead(0) runs the chain of diagonal solves in line instead
 * of on a high-priority stream (bitwise the same result).  The
 * workspace is kept by the context between calls; the call returns after the stream has
 * completed.  Status codes as zz_tgevc (-104 non-finite diagonal entry, -107). */
int zz_ztgevc(int m, const double* S, int lds, const double* T, int ldt, const int* select,
              double* X, int ldx, int* col_scale_exp);

/* Number of output columns zz_tgevc would produce for (S, select) with S on the HOST
 * (pairs count 2).  Returns n_sel >= 0, -105, or -i for a bad argument.  Host-only. */
int zz_count_columns(int m, const double* S_host, int lds, const int* select);

/* Host-only tile partition (reading R12): given the m-1
 * subdiagonal entries sub[j] = S(j+1,j) (HOST) and mb, writes tile_start[0..M] (M+1
 * entries, tile_start[M] = m) and returns M, or -105 / -106.  tile_start must hold
 * m/(mb-1)+2 ints. */
int zz_partition(int m, const double* sub, int mb, int* tile_start);

/* Host-only ownership rule of the multi-GPU path: given the m-1
 * subdiagonal entries sub[j] = S(j+1,j) (HOST), the HOST select (or NULL) and P shards,
 * writes the global output column indices owned by shard p (ascending; eigenvalue blocks with
 * first row j such that (j / 64) mod P == p; a pair's two columns stay together) to cols (may
 * be NULL) and returns their number, or -105 / a negative argument index. */
int zz_shard_columns(int m, const double* sub, const int* select, int P, int p, int* cols);

/* Statistics of the last call.  Returns 0 or -103. */
int zz_last_info(zz_info_t* out);

/* Free the workspace and the context of this thread.  Returns 0. */
int zz_finalize(void);

/* Static description of a status code. */
const char* zz_status_string(int status);

#ifdef __cplusplus
}
#endif
#endif /* ZZ_H */
