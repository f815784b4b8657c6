// B200 (sm_100a) kernels of the MINE score engine.
//
// Compiled with -fmad=false: the reference's x86-64 build never contracts
// a*b+c into an FMA, and every FP64 op below must round exactly like it does
// (SURVEY App. B).  Division uses IEEE __ddiv_rn (CUDA's default for double).
// All logarithms come from host-built glibc tables (Tables), so entropies are
// bit-identical to mutual_info.hpp:16-52.
//
// Pipeline of one call:
//   K1 k_sort_vars      per variable: stable rank, tie-run structure       (partition.cpp:13-38)
//   K2 k_equipartition  per (variable, y): greedy row map Q, yhat, H(Q)      (partition.cpp:42-67, A1)
//   memo tier  k_memo_pairs   n <= 31, B <= 7 (c1): one thread per pair, tabulated F(t,2) candidates
//   tiny tier  k_tiny_pairs   n <= 32, B <= 7: one thread per pair, all stages in registers
//   general    mine_general.cu: k_part_f2 + k_dp per y, then k_reduce here
//              (max-merge + MIC/MAS/MEV/MCN/MIC_e/TIC, statistics.cpp:10-37)
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>


#include "device_common.cuh"
#include "mine_kernels.h"

namespace mb200 {

namespace {


// ---------------------------------------------------------------------------
__global__ void k_check_finite(const double* __restrict__ v, long long count, int* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    if (!isfinite(v[i])) *flag = 1;
}

// K1: per-variable stable ranking (CTA per variable).  pos = #smaller +
// #equal-with-lower-index gives the stable sorted position; tie runs are the
// groups of equal values (C++ ==, so -0.0 and +0.0 share a run,
// partition.cpp:20,24,52,124).  The order inside a tie run is irrelevant to
// every result, so a per-variable sort replaces the reference's
// four per-pair stable sorts.
__global__ void k_sort_vars(VarSet vs) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = vs.n;
  double* v = reinterpret_cast<double*>(smem);
  int* rs = reinterpret_cast<int*>(v + n);
  int* tmp = rs + n;
  const int var = blockIdx.x;
  const double* src = vs.vals + (size_t)var * n;
  // NaN would break the total order and leave holes in perm; such inputs are
  // rejected after the call (k_check_finite), but the pipeline must stay
  // memory-safe until then, so NaN sorts as +inf here.
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = src[i];
    v[i] = isnan(x) ? HUGE_VAL : x;
  }
  __syncthreads();
  int* perm = vs.perm + (size_t)var * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = v[i];
    int less = 0, eqb = 0;
    for (int j = 0; j < n; ++j) {
      const double b = v[j];
      less += b < a;
      eqb += (b == a) & (j < i);
    }
    perm[less + eqb] = i;
    rs[less + eqb] = eqb == 0;
  }
  __syncthreads();
  const int runs = block_incl_scan(rs, n, tmp);
  int* runid = vs.runid + (size_t)var * n;
  int* rstart = vs.runstart + (size_t)var * (n + 1);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int r = rs[i] - 1;
    runid[i] = r;
    if (i == 0 || rs[i - 1] != rs[i]) rstart[r] = i;
  }
  if (threadIdx.x == 0) {
    rstart[runs] = n;
    vs.nruns[var] = runs;
  }
}

// K1 for 64 < n <= kBitonicMaxN: a bitonic sort of (order key, sample index)
// pairs in shared memory -- O(n log^2 n) compare-exchanges instead of
// k_sort_vars' O(n^2) ranking (c0's 512 variables of n = 1000: 8% of the call).
// Sorting by (key, index) is the stable order of the ranking (ties by sample
// index); keys map -0.0 to +0.0 and NaN to +inf exactly as k_sort_vars
// compares (order_key below).  Padding keys (all ones) sort last.
__device__ __forceinline__ unsigned long long order_key(double x);
constexpr int kBitonicMaxN = 8192;
__global__ void k_sort_bitonic(VarSet vs, int N) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = vs.n, tid = threadIdx.x;
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem);
  uint16_t* idx = reinterpret_cast<uint16_t*>(key + N);
  int* rs = reinterpret_cast<int*>(smem + 8 * (size_t)N + ((2 * (size_t)N + 15) & ~size_t(15)));
  int* tmp = rs + n;
  const int var = blockIdx.x;
  const double* src = vs.vals + (size_t)var * n;
  for (int i = tid; i < N; i += blockDim.x) {
    key[i] = i < n ? order_key(src[i]) : ~0ull;
    idx[i] = (uint16_t)(i < n ? i : 0xffff);
  }
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = tid; i < (N >> 1); i += blockDim.x) {
        const int a = 2 * i - (i & (stride - 1)), b = a + stride;
        const unsigned long long ka = key[a], kb = key[b];
        const uint16_t ia = idx[a], ib = idx[b];
        const bool gt = ka > kb || (ka == kb && ia > ib);
        if (gt == ((a & size) == 0)) {
          key[a] = kb;
          key[b] = ka;
          idx[a] = ib;
          idx[b] = ia;
        }
      }
    }
  }
  __syncthreads();
  int* perm = vs.perm + (size_t)var * n;
  for (int i = tid; i < n; i += blockDim.x) {
    perm[i] = idx[i];
    rs[i] = i == 0 || key[i] != key[i - 1];
  }
  __syncthreads();
  const int runs = block_incl_scan(rs, n, tmp);
  int* runid = vs.runid + (size_t)var * n;
  int* rstart = vs.runstart + (size_t)var * (n + 1);
  for (int i = tid; i < n; i += blockDim.x) {
    const int r = rs[i] - 1;
    runid[i] = r;
    if (i == 0 || rs[i - 1] != rs[i]) rstart[r] = i;
  }
  if (tid == 0) {
    rstart[runs] = n;
    vs.nruns[var] = runs;
  }
}

// K1 for large n (the 12n-byte working set of k_sort_vars no longer fits on
// chip, or the O(n^2) ranking costs more than a sort): k_sort_big, the same
// bitonic network over (order key, sample index) with the array in an HBM
// scratch slot per variable -- compare-exchange distances below kBigChunk
// run on 8192-element chunks staged in shared memory, the few longer ones
// in place through L2 -- then the tie-run scan (k_sorted_runs).
// -0.0 is keyed as +0.0 (C++ ==), NaN as +inf, as in k_sort_vars.
__device__ __forceinline__ unsigned long long order_key(double x) {
  if (isnan(x)) x = HUGE_VAL;
  if (x == 0.0) x = 0.0;
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

constexpr int kBigChunk = 8192;  // elements per shared-memory chunk (80 KB: keys + 16-bit indices)

// One CTA per variable; N = the power of two >= n (<= 65536).  gkey / gidx:
// this variable's N-element scratch arrays; skeys: the n sorted keys, packed
// per variable for k_sorted_runs.  Element a of a size-`size` bitonic stage
// sorts ascending iff (a & size) == 0, with a the index in the whole array.
__global__ void __launch_bounds__(1024) k_sort_big(VarSet vs, int N, unsigned long long* gkeys,
                                                   uint16_t* gidxs, unsigned long long* skeys) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = vs.n, tid = threadIdx.x, var = blockIdx.x;
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem);
  uint16_t* idx = reinterpret_cast<uint16_t*>(key + kBigChunk);
  unsigned long long* gkey = gkeys + (size_t)var * N;
  uint16_t* gidx = gidxs + (size_t)var * N;
  const double* src = vs.vals + (size_t)var * n;
  const int C = min(N, kBigChunk);
  // compare-exchange distances stride_hi, stride_hi / 2, .. 1 of stage `size`
  // on the staged chunk whose first element is `c0` in the whole array
  auto chunk_strides = [&](int c0, int size, int stride_hi) {
    for (int stride = stride_hi; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = tid; i < (C >> 1); i += blockDim.x) {
        const int a = 2 * i - (i & (stride - 1)), b = a + stride;
        const unsigned long long ka = key[a], kb = key[b];
        const uint16_t ia = idx[a], ib = idx[b];
        const bool gt = ka > kb || (ka == kb && ia > ib);
        if (gt == (((c0 + a) & size) == 0)) {
          key[a] = kb;
          key[b] = ka;
          idx[a] = ib;
          idx[b] = ia;
        }
      }
    }
    __syncthreads();
  };
  // phase A: every chunk fully sorted (stages 2 .. C), direction by its place
  for (int c0 = 0; c0 < N; c0 += C) {
    for (int i = tid; i < C; i += blockDim.x) {
      const int g = c0 + i;
      key[i] = g < n ? order_key(src[g]) : ~0ull;
      idx[i] = (uint16_t)(g < n ? g : 0xffff);
    }
    for (int size = 2; size <= C; size <<= 1) chunk_strides(c0, size, size >> 1);
    for (int i = tid; i < C; i += blockDim.x) {
      __stcg(gkey + c0 + i, key[i]);
      __stcg(gidx + c0 + i, idx[i]);
    }
    __syncthreads();
  }
  // phase B: stages 2 C .. N; distances >= C in place (L2), the rest per chunk
  for (int size = 2 * C; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride >= C; stride >>= 1) {
      for (int i = tid; i < (N >> 1); i += blockDim.x) {
        const int a = 2 * i - (i & (stride - 1)), b = a + stride;
        const unsigned long long ka = __ldcg(gkey + a), kb = __ldcg(gkey + b);
        const uint16_t ia = __ldcg(gidx + a), ib = __ldcg(gidx + b);
        const bool gt = ka > kb || (ka == kb && ia > ib);
        if (gt == ((a & size) == 0)) {
          __stcg(gkey + a, kb);
          __stcg(gkey + b, ka);
          __stcg(gidx + a, ib);
          __stcg(gidx + b, ia);
        }
      }
      __syncthreads();
    }
    for (int c0 = 0; c0 < N; c0 += C) {
      for (int i = tid; i < C; i += blockDim.x) {
        key[i] = __ldcg(gkey + c0 + i);
        idx[i] = __ldcg(gidx + c0 + i);
      }
      chunk_strides(c0, size, C >> 1);
      for (int i = tid; i < C; i += blockDim.x) {
        __stcg(gkey + c0 + i, key[i]);
        __stcg(gidx + c0 + i, idx[i]);
      }
      __syncthreads();
    }
  }
  int* perm = vs.perm + (size_t)var * n;
  unsigned long long* sk = skeys + (size_t)var * n;
  for (int i = tid; i < n; i += blockDim.x) {
    perm[i] = __ldcg(gidx + i);
    sk[i] = __ldcg(gkey + i);
  }
}

__global__ void k_sorted_runs(VarSet vs, const unsigned long long* skeys) {
  __shared__ int tmp[32];
  const int n = vs.n, var = blockIdx.x;
  const unsigned long long* k = skeys + (size_t)var * n;
  int* runid = vs.runid + (size_t)var * n;
  int* rstart = vs.runstart + (size_t)var * (n + 1);
  for (int i = threadIdx.x; i < n; i += blockDim.x) runid[i] = i == 0 || k[i] != k[i - 1];
  __syncthreads();
  const int runs = block_incl_scan(runid, n, tmp);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int r = runid[i] - 1;  // each thread touches only its own entries
    runid[i] = r;
    if (i == 0 || k[i] != k[i - 1]) rstart[r] = i;
  }
  if (threadIdx.x == 0) {
    rstart[runs] = n;
    vs.nruns[var] = runs;
  }
}

// K2: EquipartitionYAxis per (variable, y) -- one thread runs the greedy scan
// of equipartition_runs (partition.cpp:42-67) over the variable's tie runs.
// The row map depends only on the row variable, so it is computed
// once per variable instead of twice per pair.  H(Q) is accumulated with the
// reference's sequential p*log(p) over rows (mutual_info.cpp:33).
// One warp per (variable, y).  The greedy scan of equipartition_runs closes
// the current row before run j iff |in_row + run_j - desired| >=
// |in_row - desired|, with in_row = rs[j] - rs[row start] growing in j: the
// test is false ... false, true ... true (also in FP64: exact integers,
// monotone rounding), so the warp tests 32 runs per step and takes the first
// true one (ballot) -- the same rows as the sequential scan.  Each closed row
// is labelled by the whole warp; H(Q) adds the row sizes in row order.
__global__ void k_equipartition(VarSet vs, Tables tb) {
  const long long idx = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (idx >= (long long)vs.V * vs.ny) return;
  const int var = (int)(idx / vs.ny), yi = (int)(idx % vs.ny), y = yi + 2, n = vs.n;
  const int* rs = vs.runstart + (size_t)var * (n + 1);
  const int* perm = vs.perm + (size_t)var * n;
  const int runs = vs.nruns[var];
  uint16_t* q = vs.q + ((size_t)var * vs.ny + yi) * n;
  const double* pln = tb.pl + tri(n);
  double desired = (double)n / (double)y;
  int curr = 1, r0 = 0, j = 1;  // current row starts at run r0; next run to test j
  double acc = 0.0;
  auto label = [&](int r_end) {  // runs [r0, r_end) get label curr
    for (int t = rs[r0] + lane; t < rs[r_end]; t += 32) q[perm[t]] = (uint16_t)curr;
  };
  while (j < runs) {
    const int jj = j + lane;
    bool close = false;
    if (jj < runs) {
      const int in_row = rs[jj] - rs[r0], run = rs[jj + 1] - rs[jj];
      close = fabs((double)(in_row + run) - desired) >= fabs((double)in_row - desired);
    }
    const unsigned m = __ballot_sync(0xffffffffu, close);
    if (!m) {
      j += 32;
      continue;
    }
    const int jc = j + __ffs(m) - 1;  // the next row starts at run jc
    label(jc);
    acc = __dadd_rn(acc, pln[rs[jc] - rs[r0]]);
    ++curr;
    desired = (double)(n - rs[jc]) / (double)(y - curr + 1);
    r0 = jc;
    j = jc + 1;
  }
  label(runs);
  acc = __dadd_rn(acc, pln[n - rs[r0]]);
  if (lane == 0) {
    vs.yhat[idx] = curr;
    vs.hq[idx] = -acc;
  }
}

// Row-map equality of consecutive row targets, as the canonical row target:
// qsame[v][yi] = the smallest yi' whose row map equals yi's label for label
// (ties make the greedy scan saturate, e.g. a Poisson variable with 5
// distinct values has the same rows for every y >= 5; only consecutive y's
// are compared).  Subproblems whose row map equals a smaller y's need no
// partition or DP when their raw clumps do not superclump (k_part_f2 /
// k_part_warp: the cells are the smaller y's).  One warp per
// variable walks its y's; the label compare runs only when the row counts
// agree.
__global__ void k_row_same(VarSet vs) {
  const long long var = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (var >= vs.V) return;
  const int n = vs.n;
  const size_t row0 = (size_t)var * vs.ny;
  int canon = 0;
  for (int yi = 0; yi < vs.ny; ++yi) {
    bool same = yi > 0 && vs.yhat[row0 + yi] == vs.yhat[row0 + yi - 1];
    if (same) {
      const uint16_t* a = vs.q + (row0 + yi) * n;
      const uint16_t* b = a - n;
      bool diff = false;
      for (int t = lane; t < n; t += 32) diff |= a[t] != b[t];
      same = !__any_sync(0xffffffffu, diff);
    }
    if (!same) canon = yi;
    if (lane == 0) vs.qsame[row0 + yi] = (uint16_t)canon;
  }
}

// Tiny-tier packing: per sample the labels of y=2 and y=3 in one byte, and the
// run-start bitmask over sorted positions.
__global__ void k_pack_tiny(VarSet vs) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int n = vs.n;
  if (idx >= (long long)vs.V * n) return;
  const int var = (int)(idx / n), s = (int)(idx % n);
  const uint16_t* q = vs.q + (size_t)var * vs.ny * n;
  uint8_t l = (uint8_t)(q[s] & 3);
  if (vs.ny > 1) l |= (uint8_t)((q[n + s] & 3) << 2);
  vs.lw[idx] = l;
  if (s == 0) {
    uint32_t m = 0;
    const int* rid = vs.runid + (size_t)var * n;
    for (int t = 0; t < n; ++t)
      if (t == 0 || rid[t] != rid[t - 1]) m |= 1u << t;
    vs.rsmask[var] = m;
  }
}

// ---------------------------------------------------------------------------
// Tiny tier.  Positions fit one 32-bit word, so row maps become bitmasks in
// x-sorted order and every cumulative count is a popcount of a prefix mask.
struct TinyCtx {
  const double* pl;  // shared copy
  int n;
  uint32_t valid;
};

__device__ __forceinline__ uint32_t prefix(int pos) { return pos >= 32 ? 0xffffffffu : ((1u << pos) - 1u); }
__device__ __forceinline__ double PLs(const TinyCtx& c, int m, int w) { return c.pl[tri(m) + w]; }

// F(t,2) candidate (mutual_info.cpp:51-52): H(P) - H(P,Q) for the split at s.
__device__ __forceinline__ double tiny_cand2(const TinyCtx& c, const uint32_t* m, int rows, int cs,
                                             int ct) {
  double acc2 = PLs(c, ct, cs);
  acc2 = __dadd_rn(acc2, PLs(c, ct, ct - cs));
  const uint32_t ps = prefix(cs), pt = prefix(ct);
  int a[3];
  double accj = 0.0;
#pragma unroll
  for (int r = 0; r < 3; ++r)
    if (r < rows) {
      a[r] = __popc(m[r] & ps);
      accj = __dadd_rn(accj, PLs(c, ct, a[r]));
    }
#pragma unroll
  for (int r = 0; r < 3; ++r)
    if (r < rows) accj = __dadd_rn(accj, PLs(c, ct, __popc(m[r] & pt) - a[r]));
  return __dsub_rn(-acc2, -accj);
}

// Clump ends over x-sorted positions packed in one word (n <= 32).  d: label
// changes (bit t: lab[t] != lab[t-1]), rsm: x tie-run starts.  Returns the
// boundary mask (bit t: a clump starts at t >= 1) and k; applies Alg. 2 when
// k > k_hat.
__device__ uint32_t bits_partition(uint32_t d, uint32_t rsm, uint32_t valid, int n, int k_hat,
                                   int& k_out) {
  // Alg. 1 sentinel fusing (partition.cpp:116-133): an x-tie run whose labels
  // change inside it is fused; fused runs never merge with neighbours.
  uint32_t fp = d & ~rsm, fm = 0;
  while (fp) {
    const int t = __ffs(fp) - 1;
    const uint32_t upto = (t >= 31) ? 0xffffffffu : ((2u << t) - 1u);
    const int start = 31 - __clz(rsm & upto);
    const uint32_t after = rsm & ~upto & valid;
    const int end = after ? __ffs(after) - 1 : n;
    const uint32_t run = prefix(end) & ~prefix(start);
    fm |= run;
    fp &= ~run;
  }
  uint32_t bnd = rsm & valid & ~1u & (d | fm | (fm << 1));
  int k = __popc(bnd) + 1;
  if (k > k_hat) {  // Alg. 2 (partition.cpp:148-165): equipartition clump ordinals
    double desired = (double)n / (double)k_hat;
    int curr = 1, in_row = 0, i = 0;
    uint32_t rest = bnd, nb = 0;
    for (;;) {
      const int j = rest ? __ffs(rest) - 1 : n;
      const int run = j - i;
      if (in_row != 0 && fabs((double)(in_row + run) - desired) >= fabs((double)in_row - desired)) {
        ++curr;
        in_row = 0;
        desired = (double)(n - i) / (double)(k_hat - curr + 1);
        nb |= 1u << i;
      }
      in_row += run;
      if (!rest) break;
      rest &= rest - 1;
      i = j;
    }
    bnd = nb;
    k = curr;
  }
  k_out = k;
  return bnd;
}

// One (orientation, y) subproblem; returns I_2 and I_3 (I_3 = I_2 if x_max=2).
__device__ void tiny_subproblem(const TinyCtx& c, const uint32_t* m, int rows, uint32_t rsm,
                                int x_max, int k_hat, double hq, double& i2, double& i3,
                                unsigned long long* work) {
  const int n = c.n;
  uint32_t d = 0;
#pragma unroll
  for (int r = 0; r < 3; ++r)
    if (r < rows) d |= m[r] ^ (m[r] << 1);
  d &= c.valid & ~1u;
  int k;
  const uint32_t bnd = bits_partition(d, rsm, c.valid, n, k_hat, k);
  if (work) subproblem_work(rows, k, x_max, n, work);
  if (k < 2) {
    i2 = 0.0;
    i3 = 0.0;
    return;
  }
  double f2k = kLowest, best3 = kLowest;
  if (x_max <= 2) {
    for (uint32_t s = bnd; s; s &= s - 1) f2k = dmax(f2k, tiny_cand2(c, m, rows, __ffs(s) - 1, n));
  } else {
    // t-outer over clump ends: F(t,2) for every t (mutual_info.cpp:47-56), and
    // the level-3 candidate at t = k (mutual_info.cpp:57-66) as soon as F(s,2)
    // is known, so no F column is stored.
    int j = 0;
    for (uint32_t ts = bnd;; ts &= ts - 1) {
      const int t = ts ? __ffs(ts) - 1 : n;
      ++j;
      if (j >= 2) {
        double f2 = kLowest;
        for (uint32_t s = bnd & prefix(t); s; s &= s - 1)
          f2 = dmax(f2, tiny_cand2(c, m, rows, __ffs(s) - 1, t));
        if (t < n) {
          // h_span(s=t, k): entropy of the rows of (t, n] (mutual_info.cpp:39-41)
          const uint32_t tail = c.valid & ~prefix(t);
          const int mm = n - t;
          double acch = 0.0;
#pragma unroll
          for (int r = 0; r < 3; ++r)
            if (r < rows) acch = __dadd_rn(acch, PLs(c, mm, __popc(m[r] & tail)));
          const double dn = (double)n, rn = __drcp_rn(dn);
          const double r1 = int_quot((double)t, dn, rn);
          const double wv = __dmul_rn(int_quot(__dsub_rn(dn, (double)t), dn, rn), -acch);
          best3 = dmax(best3, __dsub_rn(__dmul_rn(r1, f2), wv));
        } else {
          f2k = f2;
        }
      }
      if (!ts) break;
    }
  }
  i2 = dmax(0.0, __dadd_rn(hq, f2k));
  const int l_max = min(x_max, k);
  i3 = l_max >= 3 ? dmax(0.0, __dadd_rn(hq, best3)) : i2;
}


// Statistics of a B <= 7 matrix (cells 0:(2,2) 1:(3,2) 2:(2,3)) from the two
// orientations' cells -- update_max merge (char_matrix.cpp:28-35), then
// statistics.cpp:10-37 and the MIC_e / TIC extensions.
// kStageStride: doubles per statistic in a memo CTA's staging slot (k_memo_pairs).
constexpr int kStageStride = 8192;

// slot: non-null -> the statistics go to this CTA's staging slot at index oi
// (a sorted position), statistic q at q * kStageStride (k_memo_pairs copies
// them to out in index order); null -> straight to out at oi.
__device__ __forceinline__ void small_stats(const double (&o)[2][3], int ncell, int est,
                                            const double* lg2, const StatsOut& out,
                                            long long oi, double* ocells, double* slot = nullptr) {
  const int cxy[3] = {4, 6, 6};
  double M[3], E[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    M[i] = o[1][i] > o[0][i] ? o[1][i] : o[0][i];
    E[i] = i == 0 ? M[i] : (i == 1 ? o[1][i] : o[0][i]);  // (3,2): x>y -> O2; (2,3): x<y -> O1
  }
  double mic = 0.0, mev = 0.0, mice = 0.0, mas = 0.0, tic = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (i < ncell) {
      mic = dmax(mic, M[i]);
      mev = dmax(mev, M[i]);  // every stored shape has x == 2 or y == 2 when B <= 7
      mice = dmax(mice, E[i]);
      const double tr = i == 0 ? M[0] : M[3 - i];
      mas = dmax(mas, fabs(M[i] - tr));
      tic = __dadd_rn(tic, est ? E[i] : M[i]);
    }
  }
  int best = 1 << 30;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (i < ncell && M[i] == mic) best = min(best, cxy[i]);
  if (slot) {
    if (out.mic) slot[oi] = mic;
    if (out.mas) slot[kStageStride + oi] = mas;
    if (out.mev) slot[2 * kStageStride + oi] = mev;
    if (out.mcn) slot[3 * kStageStride + oi] = lg2[best > 7 ? 0 : best];
    if (out.mic_e) slot[4 * kStageStride + oi] = mice;
    if (out.tic) slot[5 * kStageStride + oi] = tic;
    return;
  }
  if (out.mic) out.mic[oi] = mic;
  if (out.mas) out.mas[oi] = mas;
  if (out.mev) out.mev[oi] = mev;
  if (out.mcn) out.mcn[oi] = lg2[best > 7 ? 0 : best];
  if (out.mic_e) out.mic_e[oi] = mice;
  if (out.tic) out.tic[oi] = tic;
  if (ocells) {
    for (int i = 0; i < ncell; ++i) {
      ocells[(size_t)oi * 2 * ncell + i] = o[0][i];
      ocells[(size_t)oi * 2 * ncell + ncell + i] = o[1][i];
    }
  }
}

__global__ void __launch_bounds__(128) k_tiny_pairs(VarSet vs, Tables tb, PairSpace ps,
                                                    double cpar, int est, StatsOut out,
                                                    double* ocells, unsigned long long* counters) {
  __shared__ double pl_s[561];  // tri(33): rows m <= 32
  __shared__ double lg[8], lg2[8];
  const int n = vs.n, B = tb.B;
  for (int i = threadIdx.x; i < (int)tri(n + 1); i += blockDim.x) pl_s[i] = tb.pl[i];
  if (threadIdx.x < 8) {
    lg[threadIdx.x] = threadIdx.x <= B ? tb.logi[threadIdx.x] : 0.0;
    lg2[threadIdx.x] = threadIdx.x <= B ? tb.log2i[threadIdx.x] : 0.0;
  }
  __syncthreads();
  const long long wl = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned long long work[kNumCounters] = {};
  unsigned long long* wk = counters ? work : nullptr;
  if (wl >= ps.count) {
    if (counters) flush_work(work, counters);
    return;
  }
  int va, vb;
  pair_vars(ps, ps.first + wl, va, vb);

  TinyCtx c;
  c.pl = pl_s;
  c.n = n;
  c.valid = prefix(n);
  const int ny = vs.ny;  // 1 (B in {4,5}) or 2 (B in {6,7})
  // cells in for_each order: 0:(2,2) 1:(3,2) 2:(2,3)
  double o[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
#pragma unroll
  for (int orient = 0; orient < 2; ++orient) {
    const int X = orient ? vb : va, Y = orient ? va : vb;
    const int* permX = vs.perm + (size_t)X * n;
    const uint8_t* lwY = vs.lw + (size_t)Y * n;
    uint32_t m2[3] = {0, 0, 0}, m3[3] = {0, 0, 0};
    for (int t = 0; t < n; ++t) {
      const unsigned l = lwY[permX[t]];
      const uint32_t bit = 1u << t;
      m2[0] |= (l & 3) == 1 ? bit : 0;
      m2[1] |= (l & 3) == 2 ? bit : 0;
      m3[0] |= (l >> 2) == 1 ? bit : 0;
      m3[1] |= (l >> 2) == 2 ? bit : 0;
      m3[2] |= (l >> 2) == 3 ? bit : 0;
    }
    const uint32_t rsm = vs.rsmask[X];
    {  // y = 2
      const int rows = vs.yhat[(size_t)Y * ny];
      const int x_max = B / 2;
      const int k_hat = max(1, (int)floor(cpar * (double)x_max));
      double i2, i3;
      tiny_subproblem(c, m2, rows, rsm, x_max, k_hat, vs.hq[(size_t)Y * ny], i2, i3, wk);
      o[orient][0] = norm_cell(i2, lg[2], lg[rows]);
      if (x_max >= 3) o[orient][orient ? 2 : 1] = norm_cell(i3, lg[3], lg[rows]);
    }
    if (ny > 1) {  // y = 3
      const int rows = vs.yhat[(size_t)Y * ny + 1];
      const int x_max = B / 3;
      const int k_hat = max(1, (int)floor(cpar * (double)x_max));
      double i2, i3;
      tiny_subproblem(c, m3, rows, rsm, x_max, k_hat, vs.hq[(size_t)Y * ny + 1], i2, i3, wk);
      o[orient][orient ? 1 : 2] = norm_cell(i2, lg[2], lg[rows]);
    }
  }
  small_stats(o, ny > 1 ? 3 : 1, est, lg2, out, wl, ocells);
  if (counters) flush_work(work, counters);
}

// ---------------------------------------------------------------------------
// Memo tier (n <= 31, B <= 7; c1 is n = 23).  With two rows every F(t,2)
// candidate H(P) - H(P,Q) (mutual_info.cpp:51-52) is a function of (c_t, c_s,
// a0, b0) only (a1 = c_s - a0, b1 = c_t - c_s - b0), and there are only
// C(n+4,4)-ish such tuples.  k_build_memo evaluates every candidate ONCE with
// the reference's exact operation sequence (sequential p*log(p) sums, then
// (-acc2) - (-accj)); likewise the whole three-row y = 3 candidate for the
// standard row totals, and the level-3 span term at t = k.  k_rank_memo /
// k_dense_memo then replace each tabulated candidate by its dense rank (the
// number of DISTINCT smaller tabulated values: order-preserving, equal values
// -> equal rank, ~3k distinct values for n = 23, so a uint16) and build the
// rank -> value table val[]: the per-candidate max becomes a 2-byte gather and
// one integer max, and the double is fetched once per t -- exactly the same
// maximum, since the max rank is the rank of the max value.
__host__ __device__ __forceinline__ int memo_G(int ct, int cs) {
  // entries of K2 before c_s within block c_t: sum_{u=2}^{cs} u (ct + 2 - u)
  return (ct + 2) * (cs * (cs + 1) / 2 - 1) - (cs * (cs + 1) * (2 * cs + 1) / 6 - 1);
}

// Dense 3-row table [c_s][a0][a1] with padded strides (a0: n + 2, c_s: an odd
// number of words) so that lanes at different c_s / a0 spread over the banks.
__host__ __device__ __forceinline__ int memo_t3_as(int n) { return n + 2; }
__host__ __device__ __forceinline__ int memo_t3_rs(int n) { return memo_t3_as(n) * (n + 1) + 2; }
__host__ __device__ __forceinline__ int t3_index(int n, int cs, int a0, int a1) {
  return cs * memo_t3_rs(n) + a0 * memo_t3_as(n) + a1;
}
// Compact [c_s][a0][a1] (a0 + a1 <= c_s) for n > 26, where the padded table
// would crowd the scratch rows out of shared memory.
__host__ __device__ __forceinline__ int t3_index_c(int cs, int a0, int a1) {
  return cs * (cs + 1) * (cs + 2) / 6 + a0 * (cs + 1) - a0 * (a0 - 1) / 2 + a1;
}

__host__ __device__ inline MemoLayout memo_layout(int n) {
  MemoLayout L;
  int k2 = 0;
  for (int ct = 2; ct <= n; ++ct) k2 += memo_G(ct, ct);
  L.n = n;
  L.k2cnt = k2;
  L.t3c = n > 26;
  L.t3cnt = L.t3c ? n * (n + 1) * (n + 2) / 6  // compact
                  : n * memo_t3_rs(n);         // dense [c_s][a0][a1], padded (bank spread)
  // doubles
  L.w2 = 0;
  L.e2 = L.w2 + n * (n + 1) - n * (n - 1) / 2;
  L.pln = L.e2 + n + 1;
  L.ib = (L.pln + n + 2) & ~1;  // int region starts here (in doubles, 16-byte aligned)
  // ints, relative to the int region
  L.offk = 0;                    // (n + 2)
  // per position t (n + 2 consecutive words each: any gather is conflict-free)
  L.sb = L.offk + n + 2;         // staging base word of t (memo_y2)
  L.std3 = L.sb + n + 2;         // 2: standard 3-row totals (C0, C1)
  L.hb = L.std3 + 2;             // uint16 region, relative to the int region
  // uint16 dense candidate ranks, relative to the uint16 region
  L.k2r = 0;
  L.t3r = L.k2r + L.k2cnt;
  L.total = L.ib + (2 * L.hb + L.t3r + L.t3cnt + 3) / 4;
  return L;
}

struct MemoCtx {
  const double* tab;
  const int* ints;
  const uint16_t* ranks;
  const double* val;  // rank -> value (shared memory)
  int std3[2];
  MemoLayout L;
  int n;
  uint32_t valid;
};

__device__ __forceinline__ int w2_index(int n, int cs, int u0) {
  return cs * (n + 1) - cs * (cs - 1) / 2 + u0;
}

// Table builder: one block, the same FP64 op sequence as tiny_cand2 / the
// general tier (both bit-exact against the reference).  Candidate values go
// to vals[] (K2 first, then T3F) for ranking; the rest into the table image.
__global__ void k_build_memo(Tables tb, double* memo, double* vals, int n) {
  const MemoLayout L = memo_layout(n);
  {  // zero the image (padding included) so every byte is defined
    for (int i = threadIdx.x; i < L.total; i += blockDim.x) memo[i] = 0.0;
    __syncthreads();
  }
  int* ints = reinterpret_cast<int*>(memo + L.ib);
  int* offk = ints + L.offk;
  const double* pl = tb.pl;
  auto PL = [&](int m, int w) { return pl[tri(m) + w]; };
  if (threadIdx.x == 0) {
    int off = 0;
    for (int ct = 0; ct <= n + 1; ++ct) {
      offk[ct] = off;
      if (ct >= 2 && ct <= n) off += memo_G(ct, ct);
    }
  }
  for (int cs = threadIdx.x; cs <= n + 1; cs += blockDim.x) {
    const int g1 = cs * (cs + 1) / 2 - 1;
    const int g2 = cs * (cs + 1) * (2 * cs + 1) / 6 - 1;
    // (P, Q') = (2 g1, 2 (2 g1 - g2) + 32768) as unsigned 16-bit halves; the
    // a0-dependent part is added in memo_y2 (one IMAD)
    ints[L.sb + cs] = cs <= n ? ((2 * g1) << 16) + 2 * (2 * g1 - g2) + 32768 : 0;
  }
  // K2[ct][cs][a0][b0]
  for (int idx = threadIdx.x; idx < (n + 1) * (n + 1); idx += blockDim.x) {
    const int ct = idx / (n + 1), cs = idx % (n + 1);
    if (ct < 2 || cs < 1 || cs >= ct) continue;
    int base = memo_G(ct, cs);
    for (int c = 2; c < ct; ++c) base += memo_G(c, c);
    double acc2 = PL(ct, cs);
    acc2 = __dadd_rn(acc2, PL(ct, ct - cs));
    for (int a0 = 0; a0 <= cs; ++a0)
      for (int b0 = 0; b0 <= ct - cs; ++b0) {
        double accj = PL(ct, a0);
        accj = __dadd_rn(accj, PL(ct, cs - a0));
        accj = __dadd_rn(accj, PL(ct, b0));
        accj = __dadd_rn(accj, PL(ct, ct - cs - b0));
        vals[base + a0 * (ct - cs + 1) + b0] = __dsub_rn(-acc2, -accj);
      }
  }
  // Row totals (C0, C1, C2) of the 3-row equipartition of n distinct values
  // (partition.cpp:42-67 with unit runs): the totals of every y = 3 row map of
  // a variable without ties.
  int std3[3] = {-1, -1, -1};
  {
    double desired = (double)n / 3.0;
    int curr = 1, in_row = 0;
    for (int i = 0; i < n; ++i) {
      if (in_row != 0 && fabs((double)(in_row + 1) - desired) >= fabs((double)in_row - desired)) {
        if (curr <= 3) std3[curr - 1] = in_row;
        ++curr;
        in_row = 0;
        desired = (double)(n - i) / (double)(3 - curr + 1);
      }
      ++in_row;
    }
    if (curr == 3) std3[2] = in_row;
    else std3[0] = std3[1] = -1;
  }
  if (threadIdx.x == 0) {
    ints[L.std3] = std3[0];
    ints[L.std3 + 1] = std3[1];
  }
  // T3F[cs][a0][a1] (c_t = n): the whole 3-row F(k,2) candidate for the
  // standard totals -- E2[cs] - (-(((((p a0 + p a1) + p a2) + p b0) + p b1) + p b2)),
  // the reference's sequence; W2[cs][u0] (c_t = n), E2, PLn
  for (int cs = threadIdx.x; cs < n; cs += blockDim.x) {
    double acc2 = PL(n, cs);
    acc2 = __dadd_rn(acc2, PL(n, n - cs));
    for (int a0 = 0; a0 <= (L.t3c ? cs : n); ++a0)
      for (int a1 = 0; a1 <= (L.t3c ? cs - a0 : n); ++a1) {
        const int b0 = std3[0] - a0, b1 = std3[1] - a1, b2 = (n - cs) - b0 - b1;
        double v = 0.0;  // unreachable tuple
        if (a0 + a1 <= cs && std3[0] >= 0 && b0 >= 0 && b1 >= 0 && b2 >= 0) {
          double acc = PL(n, a0);
          acc = __dadd_rn(acc, PL(n, a1));
          acc = __dadd_rn(acc, PL(n, cs - a0 - a1));
          acc = __dadd_rn(acc, PL(n, b0));
          acc = __dadd_rn(acc, PL(n, b1));
          acc = __dadd_rn(acc, PL(n, b2));
          v = __dsub_rn(-acc2, -acc);
        }
        vals[L.k2cnt + (L.t3c ? t3_index_c(cs, a0, a1) : t3_index(n, cs, a0, a1))] = v;
      }
    const int m = n - cs;
    for (int u0 = 0; u0 <= m; ++u0) {
      double acch = PL(m, u0);
      acch = __dadd_rn(acch, PL(m, m - u0));
      memo[L.w2 + w2_index(n, cs, u0)] =
          __dmul_rn(__ddiv_rn(__dsub_rn((double)n, (double)cs), (double)n), -acch);
    }
  }
  for (int i = threadIdx.x; i <= n; i += blockDim.x) {
    double acc2 = PL(n, i);
    acc2 = __dadd_rn(acc2, PL(n, n - i));
    memo[L.e2 + i] = -acc2;
    memo[L.pln + i] = PL(n, i);
  }
}

// Build scratch: candidate values (K2 then T3F), sparse ranks, occupancy flags.
struct MemoWork {
  double* vals;
  int* rk;
  int* flag;
  int* nval;
};
__host__ __device__ inline MemoWork memo_work(void* base, int n) {
  const MemoLayout L = memo_layout(n);
  const int nv = L.k2cnt + L.t3cnt;
  MemoWork w;
  w.vals = static_cast<double*>(base);
  w.rk = reinterpret_cast<int*>(w.vals + nv);
  w.flag = w.rk + nv;
  w.nval = w.flag + nv;
  return w;
}

// rk[i] = #{j : vals[j] < vals[i]} (order-preserving, equal values share it)
__global__ void k_rank_memo(const double* __restrict__ vals, int* rk, int* flag, int nv) {
  __shared__ double chunk[2048];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double v = i < nv ? vals[i] : 0.0;
  int rank = 0;
  for (int j0 = 0; j0 < nv; j0 += 2048) {
    const int m = min(2048, nv - j0);
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) chunk[j] = vals[j0 + j];
    __syncthreads();
    for (int j = 0; j < m; ++j) rank += chunk[j] < v;
  }
  if (i < nv) {
    rk[i] = rank;
    flag[rank] = 1;
  }
}

// Dense ranks (one block): d(rank) = #occupied sparse ranks below it, so the
// rank of a candidate is the number of DISTINCT smaller values -- a uint16 in
// the table image, and val[d] the value (a few thousand entries).
__global__ void __launch_bounds__(1024) k_dense_memo(double* memo, MemoWork w, double* val, int n) {
  const MemoLayout L = memo_layout(n);
  const int nv = L.k2cnt + L.t3cnt;
  __shared__ int part[1024];
  const int per = (nv + blockDim.x - 1) / blockDim.x;
  const int lo = min(nv, (int)threadIdx.x * per), hi = min(nv, lo + per);
  int sum = 0;
  for (int j = lo; j < hi; ++j) sum += w.flag[j];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {
    const int add = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += add;
    __syncthreads();
  }
  int run = part[threadIdx.x] - sum;  // exclusive prefix
  for (int j = lo; j < hi; ++j) {
    const int f = w.flag[j];
    w.flag[j] = run;  // flag -> dense index of sparse rank j
    run += f;
  }
  if (threadIdx.x == blockDim.x - 1) *w.nval = part[threadIdx.x];
  __syncthreads();
  uint16_t* ranks = reinterpret_cast<uint16_t*>(reinterpret_cast<int*>(memo + L.ib) + L.hb);
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    const int d = w.flag[w.rk[i]];
    ranks[i < L.k2cnt ? L.k2r + i : L.t3r + (i - L.k2cnt)] = (uint16_t)d;
    val[d] = w.vals[i];
  }
}

// Per-variable 96-byte record.  As the column variable X: byte t = 32 +
// perm[t] - t, the funnel-shift amount that moves sample perm[t] (the sample
// at sorted position t) of a sample-indexed mask to bit t; the run-start mask.
// As the row variable Y: the sample-indexed label masks (y = 2 row 1, y = 3
// rows 1 and 2), H(Q) for y = 2, 3 and yhat for y = 2, 3.
__global__ void k_pack_memo(VarSet vs) {
  const int var = blockIdx.x * blockDim.x + threadIdx.x;
  if (var >= vs.V) return;
  const int n = vs.n;
  uint8_t rec[96];
#pragma unroll
  for (int i = 0; i < 96; ++i) rec[i] = 0;
  const int* perm = vs.perm + (size_t)var * n;
  const int* rid = vs.runid + (size_t)var * n;
  const uint16_t* q2 = vs.q + (size_t)var * vs.ny * n;
  const uint16_t* q3 = q2 + n;
  uint32_t rsm = 0;
  for (int t = 0; t < n; ++t) {
    // funnel-shift amount that moves bit perm[t] of a sample mask to bit t
    rec[t] = (uint8_t)(32 + perm[t] - t);
    if (t == 0 || rid[t] != rid[t - 1]) rsm |= 1u << t;
  }
  uint32_t f2 = 0, f3a = 0, f3b = 0;
  for (int s = 0; s < n; ++s) {
    f2 |= (q2[s] == 1 ? 1u : 0u) << s;
    if (vs.ny > 1) f3a |= (q3[s] == 1 ? 1u : 0u) << s, f3b |= (q3[s] == 2 ? 1u : 0u) << s;
  }
  memcpy(rec + 32, &f2, 4);
  memcpy(rec + 36, &f3a, 4);
  memcpy(rec + 40, &f3b, 4);
  const double h2 = vs.hq[(size_t)var * vs.ny];
  const double h3 = vs.ny > 1 ? vs.hq[(size_t)var * vs.ny + 1] : 0.0;
  memcpy(rec + 64, &h2, 8);
  memcpy(rec + 72, &h3, 8);
  memcpy(rec + 80, &rsm, 4);
  rec[84] = (uint8_t)vs.yhat[(size_t)var * vs.ny];
  rec[85] = vs.ny > 1 ? (uint8_t)vs.yhat[(size_t)var * vs.ny + 1] : 0;
  uint4* dst = vs.rec + (size_t)var * 6;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    uint4 v;
    memcpy(&v, rec + 16 * i, 16);
    dst[i] = v;
  }
}

// 2-byte shared load at a 32-bit shared-window byte address (lets the
// candidate-rank gather fold its base into one LEA).
__device__ __forceinline__ int lds_u16(uint32_t addr) {  // read-only table
  int v;
  asm("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
// per-thread scratch: volatile so the compiler keeps them in program order
__device__ __forceinline__ uint32_t lds_s32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_s32(uint32_t addr, int x) {
  asm volatile("st.shared.s32 [%0], %1;" ::"r"(addr), "r"(x));
}
// byte address of candidate s at level t in one instruction (IDP.2A):
// base + Q'_s * 1 + P_s * t, with (Q'_s, P_s) packed as the two unsigned
// 16-bit halves of the scratch word and (1, t) as the low two bytes of bt
__device__ __forceinline__ uint32_t cand_addr(uint32_t packed, uint32_t bt, uint32_t base) {
  return __dp2a_lo(packed, bt, base);
}

// y = 2 (two rows; row-1 positions m0): I_2 and, if x_max == 3, I_3.
// The K2 index of candidate (s, t) factors as
//   OFFK(c_t) + G(c_t, c_s) + a0 (c_t - c_s + 1) + b0
//     = [OFFK(c_t) + B0(t)] + c_t * P_s + Q_s,
//   P_s = g1(c_s) + a0(s),  Q_s = 2 g1(c_s) - g2(c_s) - a0(s) c_s,
// so (P_s, Q_s) are staged once per boundary in this thread's scratch row
// (packed int16 pair, odd stride: conflict-free) and the inner loop is one
// scratch read, one IDP.2A (the whole byte address), one 2-byte rank gather
// and half a 3-way integer max per candidate.
// kRegSlots > 0 (n <= kRegSlots + 1): the staged words live in registers
// instead of the scratch row -- every level loop is unrolled over the staged
// count, so the per-candidate scratch read (a third of the shared-memory
// wavefronts) disappears.
template <int kRegSlots>
__device__ void memo_y2(const MemoCtx& c, uint32_t m0, uint32_t rsm, int x_max, int k_hat,
                        double hq, double& i2, double& i3, unsigned long long* work, int* scr) {
  const int n = c.n;
  const uint32_t d = (m0 ^ (m0 << 1)) & c.valid & ~1u;
  int k;
  const uint32_t bnd = bits_partition(d, rsm, c.valid, n, k_hat, k);
  if (work) {
    subproblem_work(2, k, x_max, n, work, false);
    if (k >= 2) {
      work[kCntRankGathers] += x_max <= 2 ? k - 1 : k * (k - 1) / 2;  // candidate ranks
      if (x_max > 2) work[kCntGathers] += 2 * (k - 2);          // R1, W2 per span term
    }
  }
  if (k < 2) {
    i2 = i3 = 0.0;
    return;
  }
  const int c0 = __popc(m0);
  const uint16_t* K2R = c.ranks + c.L.k2r;
  const int* offk = c.ints + c.L.offk;
  double f2k, best3 = kLowest;
  if (x_max <= 2) {
    const uint16_t* kb = K2R + offk[n];
    int r = -1;
    for (uint32_t s = bnd; s; s &= s - 1) {
      const int cs = __ffs(s) - 1;
      const int a0 = __popc(m0 & prefix(cs));
      r = max(r, kb[memo_G(n, cs) + a0 * (n - cs + 1) + (c0 - a0)]);
    }
    f2k = c.val[r];
  } else if constexpr (kRegSlots > 0) {
    const double* W2 = c.tab + c.L.w2;
    const double dn = (double)n, rn = __drcp_rn(dn);
    const int* sb = c.ints + c.L.sb;
    const uint32_t k2_s = (uint32_t)__cvta_generic_to_shared(K2R) - 32768u;
    uint32_t st[kRegSlots];
    uint32_t ts = bnd;
    {
      const int t = __ffs(ts) - 1;
      st[0] = sb[t] + __popc(m0 & ((1u << t) - 1u)) * (131072 - 2 * t);
    }
    ts &= ts - 1;
    f2k = 0.0;
    // iteration L has L staged split points; the k - 1 <= n - 1 <= kRegSlots
    // boundaries end the loop (level n) by L = k - 1
#pragma unroll
    for (int L = 1; L <= kRegSlots; ++L) {
      const bool last = ts == 0;
      const int t = last ? n : __ffs(ts) - 1;
      const int b0t = last ? c0 : __popc(m0 & ((1u << t) - 1u));
      const uint32_t kb = k2_s + 2u * (offk[t] + b0t);
      const uint32_t bt = ((uint32_t)t << 8) | 1u;
      int r = -1;
#pragma unroll
      for (int j = 0; j < L; ++j) r = max(r, lds_u16(cand_addr(st[j], bt, kb)));
      if (last) {
        f2k = c.val[r];
        break;
      }
      const double f2 = c.val[r];
      const double r1 = int_quot((double)t, dn, rn);
      const int w2row = t * (n + 1) - ((t * (t - 1)) >> 1);
      best3 = dmax(best3, __dsub_rn(__dmul_rn(r1, f2), W2[w2row + c0 - b0t]));
      if (L < kRegSlots) st[L] = sb[t] + b0t * (131072 - 2 * t);
      ts &= ts - 1;
    }
  } else {
    const double* W2 = c.tab + c.L.w2;
    // R1[t] = t / n and the W2 row of t are recomputed (FP64 / integer ALU)
    // instead of gathered: the shared-memory pipe is this kernel's limiter
    const double dn = (double)n, rn = __drcp_rn(dn);
    const int* sb = c.ints + c.L.sb;
    // Q' = Q + 32768 is staged (unsigned halves); the bias comes off the base
    const uint32_t k2_s = (uint32_t)__cvta_generic_to_shared(K2R) - 32768u;
    const uint32_t scr_s = (uint32_t)__cvta_generic_to_shared(scr);
    // max candidate rank of level t over the nst staged split points
    auto level = [&](int t, int b0t, int offk_t, int nst) {
      const uint32_t kb = k2_s + 2u * (offk_t + b0t);
      const uint32_t bt = ((uint32_t)t << 8) | 1u;
      int r = -1;
      uint32_t sp = scr_s;
      const uint32_t se = scr_s + 4u * nst;
      // four candidates per trip, not unrolled further: the trip counts are
      // short and differ across the warp's pairs
#pragma unroll 1
      for (; sp + 12u < se; sp += 16u) {
        const uint32_t v0 = lds_s32(sp), v1 = lds_s32(sp + 4u), v2 = lds_s32(sp + 8u), v3 = lds_s32(sp + 12u);
        const int a0 = lds_u16(cand_addr(v0, bt, kb));
        const int a1 = lds_u16(cand_addr(v1, bt, kb));
        const int a2 = lds_u16(cand_addr(v2, bt, kb));
        const int a3 = lds_u16(cand_addr(v3, bt, kb));
        r = max(r, max(a0, a1));
        r = max(r, max(a2, a3));
      }
      if (sp < se) {
        r = max(r, lds_u16(cand_addr(lds_s32(sp), bt, kb)));
        if (sp + 4u < se) {
          r = max(r, lds_u16(cand_addr(lds_s32(sp + 4u), bt, kb)));
          if (sp + 8u < se) r = max(r, lds_u16(cand_addr(lds_s32(sp + 8u), bt, kb)));
        }
      }
      return r;
    };
    // t becomes a split point s for the later levels: stage (P_s, Q'_s),
    // pre-scaled to byte offsets in the uint16 rank table, as unsigned 16-bit
    // halves: word = ((2 (g1 + a0)) << 16) + 2 (2 g1 - g2 - a0 c_s) + 32768
    //              = sb[c_s] + a0 (2^17 - 2 c_s)   (0 <= Q' < 2^16, P < 2^11 for n <= 32)
    auto stage = [&](int slot, int t, int b0t) {
      sts_s32(scr_s + 4u * slot, sb[t] + b0t * (131072 - 2 * t));
    };
    // boundaries t_1 < ... < t_{k-1} (bnd), then t = n; level t_1 has no
    // split point and only stages; the span terms fold in ascending t
    uint32_t ts = bnd;
    {
      const int t = __ffs(ts) - 1;
      stage(0, t, __popc(m0 & ((1u << t) - 1u)));
    }
    int nst = 1;
    for (ts &= ts - 1; ts; ts &= ts - 1, ++nst) {
      const int t = __ffs(ts) - 1;  // t < n <= 31
      const int b0t = __popc(m0 & ((1u << t) - 1u));
      const double f2 = c.val[level(t, b0t, offk[t], nst)];
      const double r1 = int_quot((double)t, dn, rn);                // == R1[t]
      const int w2row = t * (n + 1) - ((t * (t - 1)) >> 1);          // == w2_index(n, t, 0)
      best3 = dmax(best3, __dsub_rn(__dmul_rn(r1, f2), W2[w2row + c0 - b0t]));
      stage(nst, t, b0t);
    }
    f2k = c.val[level(n, c0, offk[n], nst)];
  }
  i2 = dmax(0.0, __dadd_rn(hq, f2k));
  i3 = min(x_max, k) >= 3 ? dmax(0.0, __dadd_rn(hq, best3)) : i2;
}

// y = 3 with three rows (x_max = 2: F(k,2) only, c_t = n).
template <bool kT3C>
__device__ double memo_y3_rows3(const MemoCtx& c, uint32_t m0, uint32_t m1, uint32_t rsm,
                                int k_hat, double hq, unsigned long long* work) {
  const int n = c.n;
  const uint32_t d = ((m0 ^ (m0 << 1)) | (m1 ^ (m1 << 1))) & c.valid & ~1u;
  int k;
  const uint32_t bnd = bits_partition(d, rsm, c.valid, n, k_hat, k);
  const int c0 = __popc(m0), c1 = __popc(m1);
  const bool standard = c0 == c.std3[0] && c1 == c.std3[1];
  if (work) {
    subproblem_work(3, k, 2, n, work, false);
    if (k >= 2) {
      if (standard)
        work[kCntRankGathers] += k - 1;  // candidate rank (dense [c_s][a0][a1])
      else
        work[kCntGathers] += 7 * (k - 1);   // 6 p*log(p) + E2
    }
  }
  if (k < 2) return 0.0;
  double best = kLowest;
  if (standard) {
    // standard row totals (no ties in the row variable): one rank gather per candidate
    const uint16_t* T3R = c.ranks + c.L.t3r;
    int r = -1;
    for (uint32_t s = bnd; s; s &= s - 1) {
      const int cs = __ffs(s) - 1;
      const uint32_t pre = (1u << cs) - 1u;  // c_s < n <= 31
      const int a0 = __popc(m0 & pre), a1 = __popc(m1 & pre);
      r = max(r, T3R[kT3C ? t3_index_c(cs, a0, a1) : t3_index(n, cs, a0, a1)]);
    }
    best = c.val[r];
  } else {
    const double* E2 = c.tab + c.L.e2;
    const double* P = c.tab + c.L.pln;
    for (uint32_t s = bnd; s; s &= s - 1) {
      const int cs = __ffs(s) - 1;
      const uint32_t pre = (1u << cs) - 1u;
      const int a0 = __popc(m0 & pre), a1 = __popc(m1 & pre);
      const int b0 = c0 - a0, b1 = c1 - a1, b2 = (n - cs) - b0 - b1;
      double acc = P[a0];
      acc = __dadd_rn(acc, P[a1]);
      acc = __dadd_rn(acc, P[cs - a0 - a1]);
      acc = __dadd_rn(acc, P[b0]);
      acc = __dadd_rn(acc, P[b1]);
      acc = __dadd_rn(acc, P[b2]);
      best = dmax(best, __dsub_rn(E2[cs], -acc));
    }
  }
  return dmax(0.0, __dadd_rn(hq, best));
}

constexpr int kMemoMaxThreads = 1024;

__host__ __device__ inline int memo_scr_stride(int n) { return n | 1; }

// register-staged y = 2 levels: 23 slots up to n = 24, 30 up to n = 31
// (0: the scratch-row variant, kept behind MINE_B200_MEMO_SCRATCH)
static int memo_reg_slots(int n) {
  static const bool off = std::getenv("MINE_B200_MEMO_SCRATCH") != nullptr;
  return off ? 0 : (n <= 24 ? 23 : 30);
}

// sorted-batch pair order (MINE_B200_MEMO_SORT=0 turns it off)
static bool memo_sort() {
  static const bool on = [] {
    const char* e = std::getenv("MINE_B200_MEMO_SORT");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Shared-memory plan: table image | val[] (distinct candidate values) |
// per-thread scratch rows.
__host__ __device__ inline int memo_val_off(const MemoLayout& L) { return (L.total + 1) & ~1; }
__host__ __device__ inline int memo_scr_off(const MemoLayout& L, int nval) {
  return memo_val_off(L) + ((nval + 1) & ~1);
}

// Row-label mask of Y's y = 2 rows in X's sorted order (bit t: label of the
// sample at x rank t) -- the same funnel-shift extraction as memo_pair.
__device__ __forceinline__ uint32_t memo_mask2(const VarSet& vs, int X, int Y, int n) {
  const uint4* px = vs.rec + (size_t)X * 6;
  const uint4 u = __ldg(px), v = __ldg(px + 1);
  const uint32_t ax[8] = {u.x, u.y, u.z, u.w, v.x, v.y, v.z, v.w};
  const uint32_t fy = __ldg(reinterpret_cast<const unsigned int*>(vs.rec + (size_t)Y * 6 + 2));
  uint32_t m2 = 0;
#pragma unroll
  for (int t = 0; t < 32; ++t) {
    if (t < n) {
      const uint32_t a = __byte_perm(ax[t >> 2], 0, 0x4440 | (t & 3));
      m2 |= (uint32_t)(((uint64_t)fy << 32) >> a) & (1u << t);
    }
  }
  return m2;
}

// One pair (both orientations): the cells of B <= 7 and the statistics.
// swap: run orientation 1 first (the sorted-batch path puts the orientation
// with more clumps first in every lane); the cells land in the same places.
template <bool kCount, bool kT3C, int kRegSlots>
__device__ __forceinline__ void memo_pair(const MemoCtx& c, const VarSet& vs, const Tables& tb,
                                          int va, int vb, long long wl, bool swap,
                                          int kh2, int kh3, int est, const StatsOut& out, double* ocells,
                                          const double* lg, const double* lg2,
                                          unsigned long long* wk, int* scr, double* slot = nullptr) {
  const int n = c.n, B = tb.B;
  const int x2 = B / 2;  // 2 or 3
  const bool has_y3 = B >= 6;
  if (swap) {
    const int t = va;
    va = vb;
    vb = t;
  }
  double o[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
#pragma unroll
  for (int orient = 0; orient < 2; ++orient) {
    // column variable X: shift bytes + run starts; row variable Y: label
    // masks, H(Q), yhat.  Loaded per orientation to keep registers low.
    const uint4* px = vs.rec + (size_t)(orient ? vb : va) * 6;
    const uint4* py = vs.rec + (size_t)(orient ? va : vb) * 6;
    uint32_t ax[8];
    {
      const uint4 u = __ldg(px), v = __ldg(px + 1);
      ax[0] = u.x, ax[1] = u.y, ax[2] = u.z, ax[3] = u.w;
      ax[4] = v.x, ax[5] = v.y, ax[6] = v.z, ax[7] = v.w;
    }
    const uint4 fy = __ldg(py + 2);
    // the row-label masks in x-sorted order: bit t = label of sample
    // perm_X[t]; one 64-bit funnel shift + one LOP3 per mask and position
    uint32_t m2 = 0, m3a = 0, m3b = 0;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      if (t < n) {
        const uint32_t a = __byte_perm(ax[t >> 2], 0, 0x4440 | (t & 3));
        m2 |= (uint32_t)(((uint64_t)fy.x << 32) >> a) & (1u << t);
        m3a |= (uint32_t)(((uint64_t)fy.y << 32) >> a) & (1u << t);
        m3b |= (uint32_t)(((uint64_t)fy.z << 32) >> a) & (1u << t);
      }
    }
    const uint4 sx = __ldg(px + 5), hy = __ldg(py + 4), sy = __ldg(py + 5);
    const uint32_t rsm = sx.x;
    const int yh2 = sy.y & 0xff, yh3 = (sy.y >> 8) & 0xff;
    const double hq2 = __hiloint2double(hy.y, hy.x);
    const double hq3 = __hiloint2double(hy.w, hy.z);
    if (yh2 >= 2) {
      double i2, i3;
      memo_y2<kRegSlots>(c, m2, rsm, x2, kh2, hq2, i2, i3, wk, scr);
      o[orient][0] = norm_cell(i2, lg[2], lg[yh2]);
      if (x2 >= 3) o[orient][orient ? 2 : 1] = norm_cell(i3, lg[3], lg[yh2]);
    }
    if (has_y3 && yh3 >= 2) {
      double i2, dummy;
      if (yh3 == 3)
        i2 = memo_y3_rows3<kT3C>(c, m3a, m3b, rsm, kh3, hq3, wk);
      else
        memo_y2<kRegSlots>(c, m3a, rsm, 2, kh3, hq3, i2, dummy, wk, scr);
      o[orient][orient ? 1 : 2] = norm_cell(i2, lg[2], lg[yh3]);
    }
  }
  if (swap) {
    // the pass ran with X = vb first: its orientation 0 is the pair's
    // orientation 1, whose (3,2) / (2,3) cells sit transposed
    double t[2][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      t[0][i] = o[1][i == 0 ? 0 : 3 - i];
      t[1][i] = o[0][i == 0 ? 0 : 3 - i];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      o[0][i] = t[0][i];
      o[1][i] = t[1][i];
    }
  }
  small_stats(o, has_y3 ? 3 : 1, est, lg2, out, wl, ocells, slot);
}

// sort buffers after the tables: 1024 bucket counts, then per pair of the
// batch its sorted slot, its two variables (16 bits each) and its key
__host__ __device__ inline size_t memo_sort_bytes(int batch) {
  return sizeof(int) * (1024 + (size_t)batch) + (sizeof(uint32_t) + sizeof(uint16_t)) * (size_t)batch;
}

// kCount: the instrumented (untimed) variant with realised-work counters.
// kT3C: the compact 3-row table (MemoLayout::t3c), a compile-time choice.
// kSort: pairs are taken in batches of 4096 and processed in the order of
// their clump counts (max, min over the two y = 2 orientations, by a counting
// sort in shared memory), the larger orientation first, so the 32 lanes of a
// warp run loops of nearly the same trip counts (less divergence).  Results
// are written at the pairs' own indices; the order changes nothing else.
template <bool kCount, bool kT3C, int kRegSlots, int kSortBatch, int kN = 0>
__global__ void __launch_bounds__(kMemoMaxThreads, 1) k_memo_pairs(VarSet vs, Tables tb,
                                                               const double* __restrict__ memo,
                                                               const double* __restrict__ memo_val,
                                                               int nval, const MemoLayout L,
                                                               PairSpace ps, double cpar, int est,
                                                               StatsOut out, double* ocells,
                                                               unsigned long long* counters,
                                                               double* __restrict__ stage) {
  constexpr bool kSort = kSortBatch > 0;
  constexpr int sbatch = kSortBatch > 0 ? kSortBatch : 1024;
  extern __shared__ __align__(16) double msm[];
  const int n = kN ? kN : vs.n, B = tb.B;  // kN: compiled for one n (20..24)
  {
    const double2* src = reinterpret_cast<const double2*>(memo);
    double2* dst = reinterpret_cast<double2*>(msm);
    for (int i = threadIdx.x; i < (L.total + 1) / 2; i += blockDim.x) dst[i] = src[i];
    double* vdst = msm + memo_val_off(L);
    for (int i = threadIdx.x; i < nval; i += blockDim.x) vdst[i] = memo_val[i];
  }
  __shared__ double lg[8], lg2[8];
  if (threadIdx.x < 8) {
    lg[threadIdx.x] = threadIdx.x <= B ? tb.logi[threadIdx.x] : 0.0;
    lg2[threadIdx.x] = threadIdx.x <= B ? tb.log2i[threadIdx.x] : 0.0;
  }
  __syncthreads();
  // this thread's scratch row after the tables (odd stride: bank = lane)
  int* scr = reinterpret_cast<int*>(msm + memo_scr_off(L, nval)) + threadIdx.x * memo_scr_stride(n);
  MemoCtx c;
  c.tab = msm;
  c.ints = reinterpret_cast<const int*>(msm + L.ib);
  c.ranks = reinterpret_cast<const uint16_t*>(c.ints + L.hb);
  c.val = msm + memo_val_off(L);
  c.std3[0] = c.ints[L.std3];
  c.std3[1] = c.ints[L.std3 + 1];
  c.L = L;
  c.n = n;
  c.valid = prefix(n);
  unsigned long long work[kNumCounters] = {};
  unsigned long long* wk = kCount ? work : nullptr;
  const int kh2 = max(1, (int)floor(cpar * (double)(B / 2)));
  const int kh3 = max(1, (int)floor(cpar * 2.0));

  if constexpr (kSort) {
    // the sort buffers follow the tables (no scratch rows with kRegSlots)
    int* hist = reinterpret_cast<int*>(msm + memo_scr_off(L, nval));
    int* sidx = hist + 1024;
    uint32_t* svar = reinterpret_cast<uint32_t*>(sidx + sbatch);
    uint16_t* skey = reinterpret_cast<uint16_t*>(svar + sbatch);
    const int per = sbatch / kMemoMaxThreads;  // consecutive pairs per thread in the sort pass
    __shared__ int wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long nbatch = (ps.count + sbatch - 1) / sbatch;
    for (long long b = blockIdx.x; b < nbatch; b += gridDim.x) {
      const long long b0 = b * sbatch;
      const int nb = (int)min((long long)sbatch, ps.count - b0);
      hist[tid] = 0;
      __syncthreads();
      // `per` consecutive pairs per thread: one index decode, then steps
      int va = 0, vb = 0;
#pragma unroll 1
      for (int i = 0; i < per; ++i) {
        const int e = tid * per + i;
        if (e >= nb) break;
        if (i == 0 || ps.kind == kList)
          pair_vars(ps, ps.first + b0 + e, va, vb);
        else
          pair_next(ps, va, vb);
        const uint32_t m0 = memo_mask2(vs, va, vb, n), m1 = memo_mask2(vs, vb, va, n);
        const uint32_t inner = c.valid & ~1u;
        const int k0 = __popc((m0 ^ (m0 << 1)) & inner), k1 = __popc((m1 ^ (m1 << 1)) & inner);
        const int key = (max(k0, k1) << 5) | min(k0, k1);  // < 1024 (n <= 32)
        skey[e] = (uint16_t)(key | (k1 > k0 ? 0x8000 : 0));
        svar[e] = (uint32_t)va | ((uint32_t)vb << 16);  // the sorted path needs V < 65536
        atomicAdd(&hist[key], 1);
      }
      __syncthreads();
      {  // exclusive scan of the bucket counts (one per thread)
        const int v = hist[tid];
        const int incl = warp_incl_scan(v);
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) wsum[lane] = warp_incl_scan(wsum[lane]);
        __syncthreads();
        hist[tid] = incl - v + (warp ? wsum[warp - 1] : 0);
      }
      __syncthreads();
      for (int e = tid; e < nb; e += kMemoMaxThreads) {
        const int kv = skey[e];
        const int pos = atomicAdd(&hist[kv & 0x3ff], 1);
        sidx[pos] = e | ((kv >> 15) << 16);
        skey[e] = (uint16_t)pos;  // the key is consumed: now the inverse order
      }
      __syncthreads();
      // With a staging slot (no cells requested), the statistics are written
      // at their SORTED positions of this CTA's slot -- consecutive threads,
      // consecutive addresses -- and copied to the pairs' own indices after
      // the batch, whole sectors at a time: no partially written output
      // sectors for L2 to fill from HBM (round 1: 58.6 MB of fills per c1
      // launch).
      double* slot = stage ? stage + (size_t)blockIdx.x * 6 * kStageStride : nullptr;
#pragma unroll 1
      for (int pos = tid; pos < nb; pos += kMemoMaxThreads) {
        const int v = sidx[pos], e = v & 0xffff;
        const uint32_t pv = svar[e];
        memo_pair<kCount, kT3C, kRegSlots>(c, vs, tb, (int)(pv & 0xffffu), (int)(pv >> 16),
                                           slot ? pos : b0 + e, (v >> 16) != 0, kh2, kh3, est, out,
                                           ocells, lg, lg2, wk, scr, slot);
      }
      __syncthreads();
      if (slot) {
        // the batch's statistics in index order: all loads first, then the
        // coalesced stores (whole sectors)
        constexpr int kPer = sbatch / kMemoMaxThreads;
        double* const dst[6] = {out.mic, out.mas, out.mev, out.mcn, out.mic_e, out.tic};
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          if (!dst[q]) continue;
          double v[kPer];
#pragma unroll
          for (int i = 0; i < kPer; ++i) {
            const int e = tid + i * kMemoMaxThreads;
            v[i] = e < nb ? __ldcg(slot + (size_t)q * kStageStride + skey[e]) : 0.0;
          }
#pragma unroll
          for (int i = 0; i < kPer; ++i) {
            const int e = tid + i * kMemoMaxThreads;
            if (e < nb) dst[q][b0 + e] = v[i];
          }
        }
        __syncthreads();
      }
    }
  } else {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long wl = blockIdx.x * (long long)blockDim.x + threadIdx.x; wl < ps.count; wl += stride) {
      int va, vb;
      pair_vars(ps, ps.first + wl, va, vb);
      memo_pair<kCount, kT3C, kRegSlots>(c, vs, tb, va, vb, wl, false, kh2, kh3, est, out, ocells,
                                         lg, lg2, wk, scr);
    }
  }
  if (kCount) flush_work(work, counters);
}

// Per-pair reduction: max-merge of the orientations (update_max,
// char_matrix.cpp:28-35) and the statistics (statistics.cpp:10-37) plus the
// extensions MIC_e / TIC.  One warp per pair.
__global__ void k_reduce(Tables tb, long long npairs, const double* __restrict__ ocells, int est,
                         StatsOut out, long long out_offset) {
  const int lane = threadIdx.x & 31;
  const long long pr = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (pr >= npairs) return;
  const int nc = tb.ncell;
  const double* o1 = ocells + (size_t)pr * 2 * nc;
  const double* o2 = o1 + nc;
  double mic = 0.0, mas = 0.0, mev = 0.0, mice = 0.0;
  for (int c = lane; c < nc; c += 32) {
    const double a = o1[c], b = o2[c];
    const double m = b > a ? b : a;
    const int tr = tb.cell_tr[c];
    const double ta = o1[tr], tb2 = o2[tr];
    const double mt = tb2 > ta ? tb2 : ta;
    mic = dmax(mic, m);
    mas = dmax(mas, fabs(m - mt));
    if (tb.cell_edge[c]) mev = dmax(mev, m);
    const int cmp = tb.cell_cmp[c];
    mice = dmax(mice, cmp < 0 ? a : (cmp > 0 ? b : m));
  }
  mic = warp_max(mic);
  mas = warp_max(mas);
  mev = warp_max(mev);
  mice = warp_max(mice);
  int best = 1 << 30;
  for (int c = lane; c < nc; c += 32) {
    const double a = o1[c], b = o2[c];
    if ((b > a ? b : a) == mic) best = min(best, tb.cell_xy[c]);
  }
  best = warp_min_i(best);
  if (lane == 0) {
    double tic = 0.0;  // sequential in for_each order
    for (int c = 0; c < nc; ++c) {
      const double a = o1[c], b = o2[c];
      const double m = b > a ? b : a;
      const int cmp = tb.cell_cmp[c];
      tic = __dadd_rn(tic, est ? (cmp < 0 ? a : (cmp > 0 ? b : m)) : m);
    }
    const long long oi = out_offset + pr;
    if (out.mic) out.mic[oi] = mic;
    if (out.mas) out.mas[oi] = mas;
    if (out.mev) out.mev[oi] = mev;
    if (out.mcn) out.mcn[oi] = tb.log2i[best];
    if (out.mic_e) out.mic_e[oi] = mice;
    if (out.tic) out.tic[oi] = tic;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// Launchers.

// Opt every dynamic-shared-memory kernel into the device maximum once per
// device.  Setting it per launch would race between host threads that use
// different sizes (a smaller value set by one thread fails another's launch).
cudaError_t init_kernel_attributes(int device) {
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) return e;
  const void* fns[] = {reinterpret_cast<const void*>(k_sort_vars),
                       reinterpret_cast<const void*>(k_sort_bitonic),
                       reinterpret_cast<const void*>(k_sort_big),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 23, 8192, 20>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 23, 8192, 21>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 23, 8192, 22>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 23, 8192, 23>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 23, 8192, 24>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 23, 8192, 20>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 23, 8192, 21>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 23, 8192, 22>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 23, 8192, 23>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 23, 8192, 24>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 0, 0>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 23, 0>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 23, 4096>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 23, 8192>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 30, 0>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 30, 4096>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, false, 30, 8192>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, true, 0, 0>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, true, 30, 0>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, true, 30, 4096>),
                       reinterpret_cast<const void*>(k_memo_pairs<false, true, 30, 8192>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 0, 0>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 23, 0>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 23, 4096>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 23, 8192>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 30, 0>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 30, 4096>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, false, 30, 8192>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, true, 0, 0>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, true, 30, 0>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, true, 30, 4096>),
                       reinterpret_cast<const void*>(k_memo_pairs<true, true, 30, 8192>)};
  for (const void* f : fns) {
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
    // static + dynamic shared memory must fit the opt-in limit
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
void launch_check_finite(const double* v, long long count, int* flag, cudaStream_t s) {
  const int blocks = (int)std::min<long long>(4 * 148, (count + 255) / 256 + 1);
  k_check_finite<<<blocks, 256, 0, s>>>(v, count, flag);
}

static bool radix_sort_vars(int n) {
  static const char* force = std::getenv("MINE_B200_RADIX_SORT");
  if (force) return force[0] == '1';
  return n > kRadixSortN;
}

static int big_sort_N(int n) {
  int N = 128;
  while (N < n) N <<= 1;
  return N;
}

size_t sort_scratch_bytes(int V, int n) {
  if (!radix_sort_vars(n)) return 0;
  const size_t N = (size_t)big_sort_N(n);
  return 8 * N * V + 256 + 2 * N * V + 256 + 8 * (size_t)V * n + 256;
}

// MINE_B200_BITONIC=0: the O(n^2) ranking for every n <= kRadixSortN (A/B)
static bool bitonic_on() {
  static const bool on = [] {
    const char* e = std::getenv("MINE_B200_BITONIC");
    return !(e && e[0] == '0');
  }();
  return on;
}

cudaError_t launch_sort_vars(const VarSet& vs, void* scratch, cudaStream_t s) {
  if (vs.n > 64 && vs.n <= kBitonicMaxN && bitonic_on()) {
    int N = 128;
    while (N < vs.n) N <<= 1;
    const int threads = std::min(1024, std::max(128, N / 2));
    const size_t sm = 8 * (size_t)N + ((2 * (size_t)N + 15) & ~size_t(15)) + sizeof(int) * (vs.n + 64);
    k_sort_bitonic<<<vs.V, threads, sm, s>>>(vs, N);
    return cudaGetLastError();
  }
  if (!radix_sort_vars(vs.n)) {
    const int threads = vs.n <= 256 ? 128 : (vs.n <= 2048 ? 256 : 1024);
    const size_t sm = sizeof(double) * vs.n + sizeof(int) * (vs.n + 64);
    k_sort_vars<<<vs.V, threads, sm, s>>>(vs);
    return cudaGetLastError();
  }
  const int N = big_sort_N(vs.n);
  auto a256 = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* p = static_cast<char*>(scratch);
  auto* gkeys = reinterpret_cast<unsigned long long*>(p);
  auto* gidxs = reinterpret_cast<uint16_t*>(p + a256(8 * (size_t)N * vs.V));
  auto* skeys = reinterpret_cast<unsigned long long*>(p + a256(8 * (size_t)N * vs.V) + a256(2 * (size_t)N * vs.V));
  const int C = std::min(N, kBigChunk);
  k_sort_big<<<vs.V, 1024, (size_t)C * 10, s>>>(vs, N, gkeys, gidxs, skeys);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_sorted_runs<<<vs.V, 1024, 0, s>>>(vs, skeys);
  return cudaGetLastError();
}

void launch_equipartition(const VarSet& vs, const Tables& tb, cudaStream_t s) {
  const long long warps = (long long)vs.V * vs.ny;
  k_equipartition<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(vs, tb);
}

void launch_row_same(const VarSet& vs, cudaStream_t s) {
  const long long warps = (long long)vs.V;
  k_row_same<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(vs);
}

void launch_pack_tiny(const VarSet& vs, cudaStream_t s) {
  const long long total = (long long)vs.V * vs.n;
  k_pack_tiny<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(vs);
}

void launch_tiny_pairs(const VarSet& vs, const Tables& tb, const PairSpace& ps, double c, int est,
                       StatsOut out, double* o_cells, unsigned long long* counters,
                       cudaStream_t s) {
  if (ps.count <= 0) return;
  const unsigned blocks = (unsigned)((ps.count + 127) / 128);
  k_tiny_pairs<<<blocks, 128, 0, s>>>(vs, tb, ps, c, est, out, o_cells, counters);
}

size_t memo_doubles(int n) { return (size_t)memo_layout(n).total; }
size_t memo_values(int n) {
  const MemoLayout L = memo_layout(n);
  return (size_t)L.k2cnt + L.t3cnt;
}
size_t memo_work_bytes(int n) { return memo_values(n) * (sizeof(double) + 2 * sizeof(int)) + 16; }


static size_t memo_smem_fixed(int n, int nval) {
  return sizeof(double) * (size_t)memo_scr_off(memo_layout(n), nval);
}

bool memo_fits(int n, int B, int nval) {
  // tables + val[] + at least 8 warps of scratch rows in 226 KB.  n <= 31:
  // the register-staged y = 2 level loop holds k - 1 <= n - 1 split points in
  // memo_reg_slots(n) <= 30 registers (memo_y2), so n = 32 is never admitted.
  return n >= 2 && n <= 31 && B <= 7 &&
         memo_smem_fixed(n, nval) + sizeof(int) * (size_t)memo_scr_stride(n) * 256 <= 226 * 1024;
}

int launch_build_memo(const Tables& tb, double* memo, void* work, double* val, int n,
                      cudaStream_t s) {
  const int nv = (int)memo_values(n);
  const MemoWork w = memo_work(work, n);
  cudaMemsetAsync(w.flag, 0, sizeof(int) * nv, s);
  k_build_memo<<<1, 256, 0, s>>>(tb, memo, w.vals, n);
  k_rank_memo<<<(nv + 255) / 256, 256, 0, s>>>(w.vals, w.rk, w.flag, nv);
  k_dense_memo<<<1, 1024, 0, s>>>(memo, w, val, n);
  int nval = -1;
  if (cudaMemcpyAsync(&nval, w.nval, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return -1;
  return nval;
}

void launch_pack_memo(const VarSet& vs, cudaStream_t s) {
  k_pack_memo<<<(vs.V + 127) / 128, 128, 0, s>>>(vs);
}

size_t memo_stage_bytes() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sizeof(double) * 6 * 8192 * (size_t)sms;
}

void launch_memo_pairs(const VarSet& vs, const Tables& tb, const double* memo,
                       const double* memo_val, int nval, const PairSpace& ps, double c, int est,
                       StatsOut out, double* o_cells, unsigned long long* counters,
                       double* stage, cudaStream_t s) {
  if (ps.count <= 0) return;
  const size_t fixed = memo_smem_fixed(vs.n, nval);
  const size_t budget = 226 * 1024 - fixed;
  const int regs = memo_reg_slots(vs.n);
  const size_t row = regs ? 0 : sizeof(int) * (size_t)memo_scr_stride(vs.n);
  int threads = (int)(row ? std::min<size_t>(kMemoMaxThreads, budget / row) : kMemoMaxThreads) / 32 * 32;
  threads = std::max(threads, 32);
  const size_t sm = fixed + row * threads;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const MemoLayout L = memo_layout(vs.n);
#define MEMO_LAUNCH(CNT, T3C, RS, SORT)                                                        \
  k_memo_pairs<CNT, T3C, RS, SORT><<<blocks, threads, sm + (SORT ? memo_sort_bytes(SORT) : 0), s>>>( \
      vs, tb, memo, memo_val, nval, L, ps, c, est, out, o_cells, CNT ? counters : nullptr,  \
      SORT && !o_cells ? stage : nullptr)
  // the compact 3-row table starts above n = 26: never with 23 slots.  The
  // sorted-batch order needs the register-staged variant (no scratch rows)
  // and pays off only with the y = 2 level loop (B >= 6: x_max = 3); the
  // batch is the larger of 8192 / 4096 pairs whose buffers fit.
  int sbatch = 0;
  if (regs && memo_sort() && threads == kMemoMaxThreads && vs.V < 65536 && tb.B >= 6)
    for (int b = 8192; b >= 4096 && !sbatch; b /= 2)
      if (sm + memo_sort_bytes(b) <= 226 * 1024) sbatch = b;
  // work is dealt per sort batch when sorting (per thread otherwise): no CTA
  // is launched that would only stage the tables and exit
  const long long need = sbatch ? (ps.count + sbatch - 1) / sbatch : (ps.count + threads - 1) / threads;
  const unsigned blocks = (unsigned)std::min<long long>(sms, need);
  if (regs && regs < vs.n - 1) {  // memo_y2's register slots must hold k - 1 <= n - 1 split points
    std::fprintf(stderr, "mine_b200: memo register slots %d < n - 1 = %d\n", regs, vs.n - 1);
    std::abort();
  }
#define MEMO_LAUNCH_N(CNT, N)                                                              \
  k_memo_pairs<CNT, false, 23, 8192, N><<<blocks, threads, sm + memo_sort_bytes(8192), s>>>(   \
      vs, tb, memo, memo_val, nval, L, ps, c, est, out, o_cells, CNT ? counters : nullptr,  \
      o_cells ? nullptr : stage)
  // n = 20..24 (the register-staged memo range with a y = 2 level loop, e.g.
  // the 23-sample Spellman-shaped c1): compiled for the exact n, so the mask
  // loops and row indices fold to constants (c1 +1%)
#define MEMO_FIXED(CNT)                                                                      \
  do switch (vs.n) {                                                                         \
    case 20: MEMO_LAUNCH_N(CNT, 20); break;                                                  \
    case 21: MEMO_LAUNCH_N(CNT, 21); break;                                                  \
    case 22: MEMO_LAUNCH_N(CNT, 22); break;                                                  \
    case 23: MEMO_LAUNCH_N(CNT, 23); break;                                                  \
    default: MEMO_LAUNCH_N(CNT, 24); break;                                                  \
  } while (0)
#define MEMO_T3(CNT, RS, SORT) \
  (L.t3c ? MEMO_LAUNCH(CNT, true, RS, SORT) : MEMO_LAUNCH(CNT, false, RS, SORT))
#define MEMO_ALL(CNT)                                                           \
  if (regs == 23 && sbatch == 8192 && vs.n >= 20 && vs.n <= 24)                \
    MEMO_FIXED(CNT);                                                            \
  else if (regs == 23)                                                          \
    sbatch == 8192 ? MEMO_LAUNCH(CNT, false, 23, 8192)                          \
    : sbatch == 4096 ? MEMO_LAUNCH(CNT, false, 23, 4096)                        \
                     : MEMO_LAUNCH(CNT, false, 23, 0);                          \
  else if (regs)                                                                \
    sbatch == 8192 ? MEMO_T3(CNT, 30, 8192)                                     \
    : sbatch == 4096 ? MEMO_T3(CNT, 30, 4096) : MEMO_T3(CNT, 30, 0);            \
  else                                                                          \
    MEMO_T3(CNT, 0, 0);
  if (counters) {
    MEMO_ALL(true)
  } else {
    MEMO_ALL(false)
  }
#undef MEMO_ALL
#undef MEMO_T3
#undef MEMO_FIXED
#undef MEMO_LAUNCH_N
#undef MEMO_LAUNCH
}

void launch_reduce(const Tables& tb, long long npairs, const double* ocells, int est, StatsOut out,
                   long long out_offset, cudaStream_t s) {
  if (npairs <= 0) return;
  const unsigned blocks = (unsigned)((npairs * 32 + 255) / 256);
  k_reduce<<<blocks, 256, 0, s>>>(tb, npairs, ocells, est, out, out_offset);
}

}  // namespace mb200
