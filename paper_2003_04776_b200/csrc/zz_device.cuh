// zz_device.cuh -- small device helpers shared by the sm_100a kernels: exact max/min,
// complex values carried as (re, im) pairs and the complex operations of the micro-solves
// (reading R9: Smith's division).  Every operation is an explicit round-to-nearest
// intrinsic, so no contraction changes a pivot or a scaling decision (reading R17).
#pragma once
#include "zz_internal.cuh"

namespace zz {

__device__ __forceinline__ double dmaxd(double x, double y) { return x > y ? x : y; }
__device__ __forceinline__ double dmind(double x, double y) { return x < y ? x : y; }

struct cpx { double re, im; };
__device__ __forceinline__ cpx mkc(double r, double i) { cpx z; z.re = r; z.im = i; return z; }
__device__ __forceinline__ double n1(cpx z) { return __dadd_rn(fabs(z.re), fabs(z.im)); }
__device__ __forceinline__ double nmax(cpx z) { return dmaxd(fabs(z.re), fabs(z.im)); }
__device__ __forceinline__ cpx cmulx(cpx x, cpx y) {
  return mkc(__dsub_rn(__dmul_rn(x.re, y.re), __dmul_rn(x.im, y.im)),
             __dadd_rn(__dmul_rn(x.re, y.im), __dmul_rn(x.im, y.re)));
}
__device__ __forceinline__ cpx csubx(cpx x, cpx y) { return mkc(__dsub_rn(x.re, y.re), __dsub_rn(x.im, y.im)); }
// Smith's division (reading R9)
__device__ __forceinline__ cpx cdivx(cpx x, cpx y) {
  if (fabs(y.re) >= fabs(y.im)) {
    double r = __ddiv_rn(y.im, y.re), den = __dadd_rn(y.re, __dmul_rn(y.im, r));
    return mkc(__ddiv_rn(__dadd_rn(x.re, __dmul_rn(x.im, r)), den),
               __ddiv_rn(__dsub_rn(x.im, __dmul_rn(x.re, r)), den));
  } else {
    double r = __ddiv_rn(y.re, y.im), den = __dadd_rn(y.im, __dmul_rn(y.re, r));
    return mkc(__ddiv_rn(__dadd_rn(__dmul_rn(x.re, r), x.im), den),
               __ddiv_rn(__dsub_rn(__dmul_rn(x.im, r), x.re), den));
  }
}

}  // namespace zz
