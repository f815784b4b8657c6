// p*log(p) on the device, bit-identical to the host table entry
// (double)w / m * log((double)w / m) that the reference computes with glibc
// (mutual_info.hpp:24-27).  libm_log replays the host libm's double log --
// the variant glibc's ifunc picks on an FMA host -- operation for operation
// (explicit __fma_rn / __dmul_rn / __dadd_rn, no contraction: the TU is built
// with -fmad=false).  Its coefficients and its 128-entry (1/c, log c) table
// are read from the host's libm at build time (_build.gen_logdata_header), and
// the engine compares every entry of the host-built table with this function
// before using it (k_check_plog); on any difference, or without the libm
// data, the span terms keep their table gathers.
#pragma once

#include "device_common.cuh"
#include "mine_logdata.h"

namespace mb200 {

#if MB_HAVE_LOGDATA
__constant__ unsigned long long kPlogHdr[18] = MB_LOGDATA_HDR;  // ln2hi, ln2lo, A[5], B[11]
__device__ const unsigned long long kPlogTab[256] = MB_LOGDATA_TAB;  // (invc, logc) x 128

__device__ __forceinline__ double plog_c(int i) { return __longlong_as_double((long long)kPlogHdr[i]); }

// log(x) for a normal x > 0 (x = w / m in (0, 1] here).
__device__ __forceinline__ double libm_log(double x) {
  const unsigned long long ix = (unsigned long long)__double_as_longlong(x);
  if (ix == 0x3ff0000000000000ull) return 0.0;
  if (0x308ffffffffffull >= ix + 0xc012000000000000ull) {  // |x - 1| small: the B polynomial
    const double r = __dsub_rn(x, 1.0);
    const double B0 = plog_c(7);
    double x2 = __fma_rn(r, plog_c(9), plog_c(8));
    double x3 = __fma_rn(r, plog_c(12), plog_c(11));
    const double r2 = __dmul_rn(r, r);
    const double x5 = __fma_rn(r, plog_c(15), plog_c(14));
    x2 = __fma_rn(r2, plog_c(10), x2);
    x3 = __fma_rn(r2, plog_c(13), x3);
    const double r3 = __dmul_rn(r, r2);
    double x1 = __fma_rn(r2, plog_c(16), x5);
    x1 = __fma_rn(r3, plog_c(17), x1);
    x1 = __fma_rn(x1, r3, x3);
    x1 = __fma_rn(x1, r3, x2);
    const double t = __fma_rn(r, 0x1p27, r);
    const double rhi = __fma_rn(-0x1p27, r, t);
    const double rhi2 = __dmul_rn(rhi, rhi);
    const double rlo = __dsub_rn(r, rhi);
    const double hi = __fma_rn(rhi2, B0, r);
    const double lo = __fma_rn(rhi2, B0, __dsub_rn(r, hi));
    const double lo2 = __fma_rn(__dmul_rn(B0, rlo), __dadd_rn(r, rhi), lo);
    x1 = __fma_rn(x1, r3, lo2);
    return __dadd_rn(hi, x1);
  }
  const unsigned long long tmp = ix + 0xc01a000000000000ull;  // ix - 0x3fe6000000000000
  const int i = (int)((tmp >> 45) & 0x7f);
  const long long k = (long long)tmp >> 52;
  const double z = __longlong_as_double((long long)(ix - (tmp & 0xfff0000000000000ull)));
  const double kd = __int2double_rn((int)k);
  const double invc = __longlong_as_double((long long)__ldg(kPlogTab + 2 * i));
  const double logc = __longlong_as_double((long long)__ldg(kPlogTab + 2 * i + 1));
  const double w = __fma_rn(kd, plog_c(0), logc);
  const double r = __fma_rn(z, invc, -1.0);
  const double t1 = __fma_rn(r, plog_c(4), plog_c(3));
  const double hi = __dadd_rn(r, w);
  const double r2 = __dmul_rn(r, r);
  const double lo = __fma_rn(kd, plog_c(1), __dadd_rn(__dsub_rn(w, hi), r));
  const double r3 = __dmul_rn(r, r2);
  const double t2 = __fma_rn(r, plog_c(6), plog_c(5));
  const double t3 = __fma_rn(r2, plog_c(2), lo);
  const double t4 = __fma_rn(t2, r2, t1);
  return __dadd_rn(__fma_rn(r3, t4, t3), hi);
}

// p*log(p), p = w / m (IEEE quotient from rm = __drcp_rn(m), int_quot), the
// table's entry for 0 <= w <= m: 0 at w = 0.
__device__ __forceinline__ double plog_dev(unsigned w, unsigned m, double rm) {
  if (w == 0) return 0.0;
  const double p = int_quot((double)w, (double)m, rm);
  return __dmul_rn(p, libm_log(p));
}
#endif

}  // namespace mb200
