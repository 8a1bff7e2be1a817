// Microbenchmark: FP64 FMA-pipe (DFMA) vs FP64 tensor (DMMA.8x8x4) throughput on sm_100a.
// Used once to fix the FP64 roofline denominator (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double s) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, s); a1 = fma(a1, m, s); a2 = fma(a2, m, s); a3 = fma(a3, m, s);
      a4 = fma(a4, m, s); a5 = fma(a5, m, s); a6 = fma(a6, m, s); a7 = fma(a7, m, s);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double c[NACC][2];
#pragma unroll
  for (int j = 0; j < NACC; ++j) { c[j][0] = 0; c[j][1] = 0; }
  double a = 1e-3 * threadIdx.x, b = 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  printf("{\"gpu\":\"%s\",\"sms\":%d", p.name, sms);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 64 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bpsm : {4, 8}) {
    int blocks = sms * bpsm, threads = 256, iters = 4096;
    dfma_loop<<<blocks, threads>>>(out, 64, 1e-7);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf(",\"dfma_bpsm%d_tflops\":%.3f", bpsm, flop / ms * 1e-9);
  }
  for (int wpsm : {4, 8, 16, 32}) {
    int threads = 128, blocks = sms * wpsm / 4, iters = 8192;
    dmma_loop<8><<<blocks, threads>>>(out, 64);
    cudaEventRecord(e0);
    dmma_loop<8><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 256 * 8 * (double)iters * blocks * threads / 32;
    printf(",\"dmma_wpsm%d_tflops\":%.3f", wpsm, flop / ms * 1e-9);
  }
  {
    int threads = 128, blocks = sms * 4, iters = 8192;
    dmma_loop<16><<<blocks, threads>>>(out, 64);
    cudaEventRecord(e0);
    dmma_loop<16><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 256 * 16 * (double)iters * blocks * threads / 32;
    printf(",\"dmma16acc_wpsm16_tflops\":%.3f", flop / ms * 1e-9);
  }
  printf(",\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
