// Device helpers shared by the kernel translation units (mine_kernels.cu,
// mine_general.cu).  Everything here must round exactly like the reference:
// the TUs are compiled with -fmad=false.
#pragma once

#include <cfloat>
#include <cstdint>

#include "mine_kernels.h"

// Bounds-checked build (MB_BOUNDS_CHECK, _build.build(checked=True) ->
// libmine_b200_checked.so): device asserts on the scratch / slot / layout
// indexing of the general tier, the substitute for compute-sanitizer (closed
// on this GPU pool).  A failed check traps the kernel and the call fails.
#ifdef MB_BOUNDS_CHECK
#include <cassert>
#define MB_CHECK(cond) assert(cond)
#else
#define MB_CHECK(cond) ((void)0)
#endif

namespace mb200 {

constexpr double kLowest = -DBL_MAX;  // std::numeric_limits<double>::lowest()

__device__ __forceinline__ unsigned tri(unsigned m) { return m * (m + 1u) / 2u; }
// start of row m of the half table H2 (rows of floor(m/2) + 1 entries)
__host__ __device__ __forceinline__ unsigned h2_off(unsigned m) {
  const unsigned q = m >> 1;
  return (m & 1u) ? (q + 1u) * (q + 1u) : q * (q + 1u);
}
// H2(m, w) = pl(m, w) + pl(m, m - w): a two-row span's entropy sum, one gather
__device__ __forceinline__ double h2_at(const double* h2, unsigned m, unsigned w) {
  return __ldg(h2 + (h2_off(m) + min(w, m - w)));  // one 32-bit index: IMAD.WIDE.U32
}

// std::max / std::min argument order (libstdc++): max(a,b) = a < b ? b : a.
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_min_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// In-place inclusive scan of a[0..n) in shared memory; each thread owns a
// contiguous chunk.  tmp: >= 33 ints of shared scratch.  Returns the total.
__device__ inline int block_incl_scan(int* a, int n, int* tmp) {
  const int nt = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = (nt + 31) >> 5;
  const int per = (n + nt - 1) / nt;
  const int beg = min(tid * per, n), end = min(beg + per, n);
  int s = 0;
  for (int i = beg; i < end; ++i) s += a[i];
  const int incl = warp_incl_scan(s);
  if (lane == 31) tmp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int x = lane < nw ? tmp[lane] : 0;
    x = warp_incl_scan(x);
    if (lane < nw) tmp[lane] = x;
  }
  __syncthreads();
  int run = incl - s + (warp ? tmp[warp - 1] : 0);
  for (int i = beg; i < end; ++i) {
    run += a[i];
    a[i] = run;
  }
  const int total = tmp[nw - 1];
  __syncthreads();
  return total;
}

// PairSequence::at (analysis.cpp:66-81), 0-based.
__device__ inline void pair_at(long long p, long long w, int& i, int& j) {
  const long long total = p * (p - 1) / 2;
  const long long r = total - w;
  long long m = (long long)((sqrt(8.0 * (double)r + 1.0) - 1.0) / 2.0);
  while (m * (m + 1) / 2 < r) ++m;
  while (m >= 1 && (m - 1) * m / 2 >= r) --m;
  const long long ii = p - m;
  const long long row_start = total - m * (m + 1) / 2;
  i = (int)(ii - 1);
  j = (int)(ii + (w - row_start));
}

// Variables (x, y) of work item w: x is the column variable of orientation 0.
__device__ __forceinline__ void pair_vars(const PairSpace& ps, long long w, int& vx, int& vy) {
  if (ps.kind == kPairwise) {
    pair_at(ps.p, w, vx, vy);
  } else if (ps.kind == kCross) {
    vx = (int)(w / ps.py);
    vy = ps.px + (int)(w % ps.py);
  } else {
    vx = ps.xi[w];
    vy = ps.yi[w];
  }
}

// The work item after (vx, vy) in pair_vars order (pairwise / cross only).
__device__ __forceinline__ void pair_next(const PairSpace& ps, int& vx, int& vy) {
  if (ps.kind == kPairwise) {
    if (++vy == ps.p) {
      ++vx;
      vy = vx + 1;
    }
  } else if (++vy == ps.px + ps.py) {
    ++vx;
    vy = ps.px;
  }
}

// Realised algorithmic work of one exact subproblem (rows R, k clumps): the
// FP64 operations the reference arithmetic itself requires (mutual_info.cpp:
// 47-66 with every 0.0 + x start elided), its p*log(p) lookups, DP candidates
// and span entries, and the partition's point visits (n per subproblem,
// SURVEY 8d N_pv).  Used only when counters are requested.
__device__ inline void subproblem_work(int R, int k, int x_max, int n, unsigned long long* w,
                                bool gathers_as_reference = true) {
  w[kCntPoints] += n;
  if (k < 2) return;
  const long long l_max = min(x_max, k), K = k;
  const long long f2 = l_max >= 3 ? K * (K - 1) / 2 : K - 1;  // F(t,2) candidates
  long long spans = 0, cand = 0;
  if (l_max >= 3) {
    spans = K - 2;                                             // t = k
    if (l_max >= 4) spans += (K - 3) * (K - 2) / 2;            // t = 3 .. k-1
    for (long long l = 3; l <= l_max; ++l) {
      cand += K - l + 1;                                       // t = k
      if (l <= l_max - 1) cand += (K - l) * (K - l + 1) / 2;   // t = l .. k-1
    }
  }
  w[kCntFp64] += f2 * (2 * R + 2) + spans * (R + 2) + cand * 3;
  w[kCntLookups] += f2 * (2 * R + 2) + spans * R;
  if (gathers_as_reference) w[kCntGathers] += f2 * (2 * R + 2) + spans * R;
  w[kCntCand] += cand;
  w[kCntF2] += f2;
  w[kCntSpanLookups] += spans * R;
  w[kCntSpans] += spans;
  w[kCntSub] += 1;
}

// Instrumented runs only (untimed): plain per-thread atomics, safe from any
// divergent call site.
__device__ inline void flush_work(const unsigned long long* w, unsigned long long* counters) {
#pragma unroll
  for (int i = 0; i < kNumCounters; ++i)
    if (w[i]) atomicAdd(counters + i, w[i]);
}

// char_matrix.cpp:57-64: normalise by min(log l, log yhat); clamp at 1 and
// keep the max with the zero-initialised slot (update_max :28-35).
__device__ __forceinline__ double norm_cell(double I, double logl, double logy) {
  const double norm = dmin(logl, logy);
  double v = norm > 0.0 ? __ddiv_rn(I, norm) : 0.0;
  if (v > 1.0) v = 1.0;
  return 0.0 < v ? v : 0.0;
}

// Correctly rounded a / b for integers 0 <= a <= b <= 65535 (the span-term
// quotients c_s/c_t and (c_t - c_s)/c_t, mutual_info.cpp:62) from
// rcp = __drcp_rn(b), computed once per b: q0 = a*rcp, r = a - q0*b (exact
// with one FMA), q = q0 + r*rcp (Markstein's correction).  Bitwise equal to
// __ddiv_rn(a, b), i.e. to the reference's IEEE division, on the whole domain:
// checked exhaustively (all 2.1e9 pairs) by probes.cu
// mine_b200_check_quotients (tests/test_gpu_parity.py).  Three FP64 ops
// instead of a DDIV sequence.
__device__ __forceinline__ double int_quot(double a, double b, double rcp) {
  const double q0 = __dmul_rn(a, rcp);
  const double r = __fma_rn(-q0, b, a);
  return __fma_rn(r, rcp, q0);
}

}  // namespace mb200
