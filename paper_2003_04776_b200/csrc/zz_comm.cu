// zz_comm.cu -- multi-GPU plumbing of the library ("the task
// graph is the disjoint union of p task-graphs, one for each block column"
// distributed memory as the next step): NCCL, loaded at run time, for the broadcast of the
// S/T panels from rank 0 and the gather of the finished eigenvector columns; and the two
// kernels of the gather, which move exactly the upper part of every column (rows 0 .. r_c,
// X is zero below) between the column-major X and a packed buffer.
//
// NCCL is opened with dlopen("libnccl.so.2") when a communicator is first requested, so the
// library itself loads without it (a process that imported torch gets torch's NCCL: the
// dynamic loader matches the soname of the already-loaded copy).  The environment variable
// ZZ_NCCL_LIB may name another library with the same entry points (the tests' in-process
// multi-rank transport, tests/mock_nccl).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdlib.h>

#include "zz_internal.cuh"

namespace zz {

namespace {
NcclApi g_api;
int g_api_state = 0;   // 0 untried, 1 loaded, -1 unavailable
}  // namespace

const NcclApi* nccl_api() {
  if (g_api_state == 0) {
    // ZZ_NCCL_LIB: another library with NCCL's entry points (tests/mock_nccl: an in-process
    // transport that lets several ranks share one GPU in the tests; read once, at first use)
    const char* names[] = {getenv("ZZ_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* n : names)
      if (n && (h = dlopen(n, RTLD_NOW | RTLD_LOCAL))) break;
    g_api_state = -1;
    if (h) {
      g_api.getUniqueId = reinterpret_cast<decltype(g_api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      g_api.commInitRank = reinterpret_cast<decltype(g_api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
      g_api.commDestroy = reinterpret_cast<decltype(g_api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
      g_api.broadcast = reinterpret_cast<decltype(g_api.broadcast)>(dlsym(h, "ncclBroadcast"));
      g_api.send = reinterpret_cast<decltype(g_api.send)>(dlsym(h, "ncclSend"));
      g_api.recv = reinterpret_cast<decltype(g_api.recv)>(dlsym(h, "ncclRecv"));
      g_api.groupStart = reinterpret_cast<decltype(g_api.groupStart)>(dlsym(h, "ncclGroupStart"));
      g_api.groupEnd = reinterpret_cast<decltype(g_api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
      if (g_api.getUniqueId && g_api.commInitRank && g_api.commDestroy && g_api.broadcast && g_api.send &&
          g_api.recv && g_api.groupStart && g_api.groupEnd)
        g_api_state = 1;
    }
  }
  return g_api_state == 1 ? &g_api : nullptr;
}

// ------------------------------------------------------------------------------------
// Gather kernels.  The send buffer of a rank holds its local columns l in order, column l
// as rows 0 .. h_l - 1 (h_l = r_l + 1: the upper part) at double offset off[l], followed by
// the int32 exponents.  One CTA per column, coalesced along the rows.
// ------------------------------------------------------------------------------------
__global__ void k_shard_pack(const double* __restrict__ X, long long ldx, const int* __restrict__ cse,
                             int n, const long long* __restrict__ off, const int* __restrict__ h,
                             double* __restrict__ buf, int* __restrict__ ebuf) {
  const int l = blockIdx.x;
  if (l >= n) return;
  const double* src = X + (long long)l * ldx;
  double* dst = buf + off[l];
  const int hl = h[l];
  for (int i = threadIdx.x; i < hl; i += blockDim.x) dst[i] = src[i];
  if (threadIdx.x == 0) ebuf[l] = cse[l];
}

// Writes column g[e] of X completely: rows 0 .. h-1 from the packed buffer (byte offset
// boff[e]), the rows below exactly 0; col_scale_exp[g[e]] from byte offset beoff[e].
__global__ void k_shard_unpack(const unsigned char* __restrict__ buf, int ne, const long long* __restrict__ boff,
                               const long long* __restrict__ beoff, const int* __restrict__ h,
                               const int* __restrict__ g, int m, double* __restrict__ X, long long ldx,
                               int* __restrict__ cse) {
  const int e = blockIdx.x;
  if (e >= ne) return;
  const double* src = reinterpret_cast<const double*>(buf + boff[e]);
  double* dst = X + (long long)g[e] * ldx;
  const int he = h[e];
  for (int i = threadIdx.x; i < m; i += blockDim.x) dst[i] = (i < he) ? src[i] : 0.0;
  if (threadIdx.x == 0 && cse) cse[g[e]] = *reinterpret_cast<const int*>(buf + beoff[e]);
}

cudaError_t launch_shard_pack(const double* X, long long ldx, const int* cse, int n, const long long* off,
                              const int* h, double* buf, int* ebuf, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_shard_pack<<<n, 256, 0, st>>>(X, ldx, cse, n, off, h, buf, ebuf);
  return cudaGetLastError();
}

cudaError_t launch_shard_unpack(const unsigned char* buf, int ne, const long long* boff, const long long* beoff,
                                const int* h, const int* g, int m, double* X, long long ldx, int* cse,
                                cudaStream_t st) {
  if (ne <= 0) return cudaSuccess;
  k_shard_unpack<<<ne, 256, 0, st>>>(buf, ne, boff, beoff, h, g, m, X, ldx, cse);
  return cudaGetLastError();
}

}  // namespace zz
