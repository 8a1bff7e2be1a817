// Feasibility probe for a lookahead schedule: can a high-priority "diagonal solve"-shaped
// kernel (1 CTA/SM, 220 KB smem) get SMs while a low-priority "update"-shaped kernel
// (2 CTAs/SM, 99 KB smem each, many short CTAs) is running?  Prints the time from the
// high-priority launch to its completion, with and without the background kernel.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void spin_kernel(long long cycles, int* sink) {
  extern __shared__ char sm[];
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
  (void)sm;
  if (threadIdx.x == 0 && cycles < 0) atomicAdd(sink, 1);
}

int main() {
  int lo, hi;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t sl, sh;
  cudaStreamCreateWithPriority(&sl, cudaStreamNonBlocking, lo);
  cudaStreamCreateWithPriority(&sh, cudaStreamNonBlocking, hi);
  int* sink;
  cudaMalloc(&sink, 4);
  const int smem_upd = 99 * 1024, smem_diag = 220 * 1024;
  cudaError_t e0 = cudaFuncSetAttribute(spin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_diag);
  printf("attr: %s\n", cudaGetErrorString(e0));
  cudaEvent_t a, b, c0, c1;
  cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c0); cudaEventCreate(&c1);
  const long long cyc_upd = 2000LL * 70;     // ~70 us per update CTA at ~2 GHz
  const long long cyc_diag = 2000LL * 170;   // ~170 us per diag CTA
  for (int bg = 0; bg < 2; ++bg) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(c0, sl);
      if (bg) spin_kernel<<<296 * 60, 160, smem_upd, sl>>>(cyc_upd, sink);   // ~4 ms of background
      cudaEventRecord(c1, sl);
      // let the background fill the GPU, then launch the high-priority kernel
      spin_kernel<<<1, 32, 0, sh>>>(2000LL * 500, sink);   // 0.5 ms delay on the high stream
      cudaEventRecord(a, sh);
      spin_kernel<<<148, 384, smem_diag, sh>>>(cyc_diag, sink);
      cudaEventRecord(b, sh);
      cudaError_t err = cudaDeviceSynchronize();
      if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(err)); return 1; }
      float ms, msb;
      cudaEventElapsedTime(&ms, a, b);
      cudaEventElapsedTime(&msb, c0, c1);
      printf("background %d rep %d: high-priority kernel %.3f ms after launch (background %.3f ms)\n", bg, rep, ms, msb);
    }
  }
  return 0;
}
