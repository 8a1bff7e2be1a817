// Development: latency of a dependent chain of mma.m8n8k4.f64 (DMMA.8x8x4) in one warp, and the
// issue interval of N independent chains; also DFMA and __drcp_rn dependent latencies.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NC>
__global__ void k(double* out, long long* cyc, int iters) {
  double d[NC][2];
  for (int c = 0; c < NC; ++c) { d[c][0] = threadIdx.x * 1e-3 + c; d[c][1] = 1.0; }
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < NC; ++c) dmma(d[c][0], d[c][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < NC; ++c) s += d[c][0] + d[c][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void kfma(double* out, long long* cyc, int iters) {
  double x = threadIdx.x * 1e-3, y = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, 1e-9);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void krcp(double* out, long long* cyc, int iters) {
  double x = 1.5 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __drcp_rn(x) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
  const int it = 4096;
#define RUN(NC) k<NC><<<1, 32>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); \
  printf("DMMA %2d independent chains: %.1f cycles per DMMA per chain step, %.1f cycles per DMMA issued\n", NC, (double)h / it, (double)h / it / NC);
  RUN(1) RUN(2) RUN(4) RUN(8) RUN(16)
  kfma<<<1, 32>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("DFMA dependent: %.1f cycles\n", (double)h / it);
  krcp<<<1, 32>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("drcp_rn + add dependent: %.1f cycles\n", (double)h / it);
  return 0;
}
