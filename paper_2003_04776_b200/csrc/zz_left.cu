// zz_left.cu -- left eigenvectors through the right
// eigenvector path.  y^H (beta S - alpha T) = 0 is (beta S^T - conj(alpha) T^T) y = 0; with J
// the row/column reversal, S' = J S^T J and T' = J T^T J are again a real Schur pencil (upper
// quasi-triangular S' with the mirrored 2x2 blocks, upper triangular T', the same
// eigenvalues), and J y is the right eigenvector of (S', T') for conj(lambda), i.e. the
// complex conjugate of the one the right path computes for lambda.  So: flip the pencil,
// run the robust blocked right solve on it, and map back (reverse the rows, negate the
// imaginary column of a pair, restore the block order of S).
#include "zz_internal.cuh"

namespace zz {

namespace {

constexpr int kFT = 32;   // transpose tile

// A'(i, j) = A(m-1-j, m-1-i) for i <= j + 1 (the upper part and the subdiagonal, all the
// solve reads); the rest of A' is left as is.  32 x 32 tiles through shared memory so both
// the reads (columns of A) and the writes (columns of A') are coalesced.
__global__ void __launch_bounds__(kFT * 8) k_flip_transpose(const double* __restrict__ A, long long lda,
                                                            double* __restrict__ B, long long ldb, int m) {
  __shared__ double tile[kFT][kFT + 1];
  const int bi = blockIdx.x * kFT, bj = blockIdx.y * kFT;   // output tile rows i, columns j
  if (bi > bj + kFT) return;                                // strictly below the band: unused
  // source rows m-1-j, source columns m-1-i
  const int tx = threadIdx.x & (kFT - 1), ty = threadIdx.x / kFT;
#pragma unroll
  for (int k = ty; k < kFT; k += 8) {
    const int i = bi + k;                 // output row    -> source column m-1-i
    const int j = bj + tx;                // output column -> source row m-1-j (lanes: a column run)
    double v = 0.0;
    if (i < m && j < m) v = A[(long long)(m - 1 - i) * lda + (m - 1 - j)];
    tile[k][tx] = v;                      // tile[i - bi][j - bj]
  }
  __syncthreads();
#pragma unroll
  for (int k = ty; k < kFT; k += 8) {
    const int j = bj + k, i = bi + tx;
    if (i < m && j < m && i <= j + 1) B[(long long)j * ldb + i] = tile[tx][k];
  }
}

// Y(i, c) = sign * X'(m-1-i, src(c)), e(c) = e'(src(c)): output columns in the block order of
// S; a pair's (Re, Im) come from the flipped solve's (Re, -Im).
__global__ void __launch_bounds__(256) k_left_gather(const double* __restrict__ Xf, long long ldxf, double* __restrict__ Y,
                                                     long long ldy, int m, int n_sel, const int* __restrict__ kind_f,
                                                     const int* __restrict__ ef, int* __restrict__ ey) {
  const int c = blockIdx.y;
  const int cc = n_sel - 1 - c;
  const int k = kind_f[cc];
  const int src = (k == kPairSecond) ? cc - 1 : (k == kPairFirst) ? cc + 1 : cc;
  const double sg = (k == kPairFirst) ? -1.0 : 1.0;
  const double* x = Xf + (long long)src * ldxf;
  double* y = Y + (long long)c * ldy;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) y[i] = sg * x[m - 1 - i];
  if (ey && blockIdx.x == 0 && threadIdx.x == 0) ey[c] = ef[src];
}

}  // namespace

cudaError_t launch_flip_transpose(const double* A, long long lda, double* B, long long ldb, int m, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  dim3 g((m + kFT - 1) / kFT, (m + kFT - 1) / kFT);
  k_flip_transpose<<<g, kFT * 8, 0, st>>>(A, lda, B, ldb, m);
  return cudaGetLastError();
}

cudaError_t launch_left_gather(const double* Xf, long long ldxf, double* Y, long long ldy, int m, int n_sel,
                               const int* kind_f, const int* ef, int* ey, cudaStream_t st) {
  if (m <= 0 || n_sel <= 0) return cudaSuccess;
  dim3 g(std::min((m + 255) / 256, 8), n_sel);
  k_left_gather<<<g, 256, 0, st>>>(Xf, ldxf, Y, ldy, m, n_sel, kind_f, ef, ey);
  return cudaGetLastError();
}

}  // namespace zz
