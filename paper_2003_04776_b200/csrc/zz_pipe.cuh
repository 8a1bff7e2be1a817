// zz_pipe.cuh -- PTX building blocks of the FP64 tensor-core contractions (sm_100a): mbarrier
// pipeline, TMA (cp.async.bulk.tensor) and bulk copies into shared memory, the FP64 tensor
// instruction DMMA.8x8x4 (mma.sync.m8n8k4.f64: sm_100a has no FP64 tcgen05 kind), L2
// eviction-priority policies and predicated 16-byte global accesses.  Shared by the robust
// update (zz_update.cu), the back-transformation GEMM (zz_back.cu) and the complex update
// (zz_complex.cu).
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace zz {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// L2 eviction priority (createpolicy): streamed C tiles evict_first, re-read B operands
// evict_last
__device__ __forceinline__ uint64_t l2_policy(bool last) {
  uint64_t pol;
  if (last)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// predicated accesses (no branch around a load: all C loads of a lane issue before the
// first one is consumed)
__device__ __forceinline__ void ld2h(double& x, double& y, const double* p, bool pr, uint64_t pol) {
  asm("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %4;\n}"
      : "+d"(x), "+d"(y) : "l"(p), "r"((int)pr), "l"(pol));
}
__device__ __forceinline__ void st2h(double* p, double x, double y, bool pr, uint64_t pol) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %4;\n}"
               ::"l"(p), "d"(x), "d"(y), "r"((int)pr), "l"(pol) : "memory");
}
__device__ __forceinline__ void st1h(double* p, double x, bool pr, uint64_t pol) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global.L2::cache_hint.f64 [%0], %1, %3;\n}"
               ::"l"(p), "d"(x), "r"((int)pr), "l"(pol) : "memory");
}
__device__ __forceinline__ void ld1p_i(int& x, const int* p, bool pr) {
  asm("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q ld.global.b32 %0, [%1];\n}" : "+r"(x) : "l"(p), "r"((int)pr));
}
__device__ __forceinline__ void bulk_load_h(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

}  // namespace zz
