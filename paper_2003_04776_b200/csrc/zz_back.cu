// zz_back.cu -- normalisation after the back-transformation W = V X (xTGEVC HOWMNY='B',
// PAPER.md:28-32 with SURVEY.md reading A1).  The product itself is a plain DGEMM per
// column block (cuBLAS, zz_api.cu); this kernel applies LAPACK's normalisation of the
// back-transformed vectors: max_i |w_i| = 1 for a real column, max_i (|Re w_i| + |Im w_i|)
// = 1 for a complex pair, by one multiply with the reciprocal of the maximum.
#include "zz_internal.cuh"

namespace zz {

namespace {

constexpr int kNormThreads = 256;

// one CTA per output column; the CTA of a pair's second column returns at once and the
// first column's CTA scales both
__global__ void __launch_bounds__(kNormThreads) k_back_norm(double* __restrict__ W, long long ldw, int m,
                                                            const int* __restrict__ col_kind) {
  const int c = blockIdx.x;
  const int kind = col_kind[c];
  if (kind == kPairSecond) return;
  const bool pair = kind == kPairFirst;
  double* w0 = W + (long long)c * ldw;
  double* w1 = pair ? w0 + ldw : w0;
  double mx = 0.0;
  for (int i = threadIdx.x; i < m; i += kNormThreads) {
    const double v = pair ? fabs(w0[i]) + fabs(w1[i]) : fabs(w0[i]);
    mx = fmax(mx, v);
  }
  __shared__ double red[kNormThreads / 32];
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
  if (!(mx > 0.0)) return;           // a zero column (V singular) stays zero
  const double r = 1.0 / mx;
  for (int i = threadIdx.x; i < m; i += kNormThreads) {
    w0[i] *= r;
    if (pair) w1[i] *= r;
  }
}

}  // namespace

cudaError_t launch_back_norm(double* W, long long ldw, int m, int n_sel, const int* col_kind, cudaStream_t st) {
  if (n_sel <= 0 || m <= 0) return cudaSuccess;
  k_back_norm<<<n_sel, kNormThreads, 0, st>>>(W, ldw, m, col_kind);
  return cudaGetLastError();
}

}  // namespace zz
