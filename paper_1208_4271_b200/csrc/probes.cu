// Measurement probes (bench.py only, not part of the engine ABI): the
// sustained FP64 add rate and the shared-memory 8-byte and 2-byte gather rates of this
// B200, the denominators of the roofline for the exact MINE DP, which is
// neither HBM- nor tensor-core-bound.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"  // mb200::int_quot, the engine's quotient

namespace {

constexpr int kChains = 8;

__global__ void k_dadd(double* out, int iters, double inc) {
  double a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a[c]) : "d"(inc));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += a[c];
  if (s == 12345.678) out[0] = s;
}

// Random 8-byte gathers from a 561-entry shared table (the tiny tier's
// p*log(p) table size), 8 independent streams per thread.
__global__ void k_lds(double* out, int iters) {
  __shared__ double tab[561];
  for (int i = threadIdx.x; i < 561; i += blockDim.x) tab[i] = i * 0.5;
  __syncthreads();
  uint32_t st = 2654435761u * (threadIdx.x + 1) + blockIdx.x;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      st = st * 1664525u + 1013904223u;
      acc += tab[(st >> 8) % 561u];
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

// Random 2-byte gathers from a 16384-entry shared uint16 table (the size
// class of the memo tier's dense candidate-rank tables) folded with an
// integer max, 8 independent streams per thread.
__global__ void k_lds2(int* out, int iters, int key) {
  extern __shared__ unsigned short htab[];
  constexpr uint32_t kN = 16384;
  for (int i = threadIdx.x; i < (int)kN; i += blockDim.x) htab[i] = (unsigned short)(i * 7);
  __syncthreads();
  uint32_t st[kChains];
  int acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) st[c] = 2654435761u * (threadIdx.x + 1) + blockIdx.x * 977u + c, acc[c] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      st[c] = st[c] * 1664525u + 1013904223u;
      acc[c] = max(acc[c], (int)htab[(st[c] >> 10) & (kN - 1)]);
    }
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s ^= acc[c];
  if (s == key) out[0] = s;  // key < 0 at run time: never true, not provable
}

// Exhaustive check of the engine's integer quotient (device_common.cuh
// int_quot) against IEEE division: every 0 <= a <= b, 1 <= b <= nmax.
__global__ void k_check_quot(int nmax, unsigned long long* out) {
  unsigned long long bad = 0, cnt = 0;
  for (int b = blockIdx.x + 1; b <= nmax; b += gridDim.x) {
    const double db = (double)b, rcp = __drcp_rn(db);
    for (int a = threadIdx.x; a <= b; a += blockDim.x) {
      const double da = (double)a;
      bad += __double_as_longlong(mb200::int_quot(da, db, rcp)) != __double_as_longlong(__ddiv_rn(da, db));
      ++cnt;
    }
  }
  atomicAdd(out, bad);
  atomicAdd(out + 1, cnt);
}

// Random 8-byte gathers from a global table of `entries` doubles (L2-resident
// up to ~100 MB): the span-term lookups of the general tier's p*log(p) table
// (rows m = c_t - c_s scattered across the table).  8 independent streams per
// thread, so each warp keeps 8 gathers in flight.
__global__ void k_ldg_rand(const double* __restrict__ tab, unsigned entries, double* out, int iters) {
  uint32_t st[kChains];
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c)
    st[c] = 2654435761u * (blockIdx.x * blockDim.x + threadIdx.x + 1) + 40503u * c, acc[c] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      st[c] = st[c] * 1664525u + 1013904223u;
      acc[c] += __ldg(tab + (st[c] >> 4) % entries);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

// The exact DP candidate (mutual_info.cpp:62-63 as the engine issues it:
// DMUL, DADD, then libstdc++'s max = DSETP + two selects), 8 independent max
// chains per thread: the FP64 pipe's candidate rate.
__global__ void k_dcand(double* out, int iters, double a, double w) {
  double f[kChains], m[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) f[c] = -(threadIdx.x * 1e-3 + c), m[c] = -1e300;
  const long long abits = __double_as_longlong(a);
  for (int i = 0; i < iters; ++i) {
    // the multiplier changes every iteration by an integer op (ALU pipe), so
    // nothing is loop-invariant and the FP64 pipe sees only the candidate ops
    const double ai = __longlong_as_double(abits ^ (long long)(i & 7));
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      const double v = __dsub_rn(__dmul_rn(ai, f[c]), w);
      m[c] = m[c] < v ? v : m[c];
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += m[c];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
float time_ms(F&& launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();  // warm-up
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms;
}

}  // namespace

extern "C" int mine_b200_probe(int device, double* dadd_per_s, double* lds_per_s,
                               double* lds2_per_s) {
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return -1;
  const int blocks = sms * 8, threads = 256, iters = 4096;
  float ms = time_ms([&] { k_dadd<<<blocks, threads>>>(out, iters, 1e-9); });
  *dadd_per_s = (double)blocks * threads * iters * kChains / (ms * 1e-3);
  const int liters = 2048;
  ms = time_ms([&] { k_lds<<<blocks, threads>>>(out, liters); });
  *lds_per_s = (double)blocks * threads * liters * kChains / (ms * 1e-3);
  const size_t sm2 = 16384 * sizeof(unsigned short);
  const int b2 = sms * 4;  // 4 x 32 KB tables per SM
  ms = time_ms([&] { k_lds2<<<b2, 512, sm2>>>(reinterpret_cast<int*>(out), liters, -1); });
  *lds2_per_s = (double)b2 * 512 * liters * kChains / (ms * 1e-3);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

extern "C" int mine_b200_check_quotients(int device, int nmax, unsigned long long* mismatches,
                                         unsigned long long* checked) {
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 2 * sizeof(unsigned long long)) != cudaSuccess) return -1;
  cudaMemset(d, 0, 2 * sizeof(unsigned long long));
  k_check_quot<<<4096, 256>>>(nmax, d);
  unsigned long long h[2] = {0, 0};
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  *mismatches = h[0];
  *checked = h[1];
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// Extra roofline denominators for the general tier: random 8-byte L2 gathers
// per second from a `table_bytes` table, and exact DP candidates per second
// (k_dcand: DMUL + DADD + DSETP + two selects per candidate, as the DP's
// inner loop issues them).
extern "C" int mine_b200_probe_general(int device, double table_bytes, double* l2_gathers_per_s,
                                       double* candidates_per_s) {
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const unsigned entries = (unsigned)(table_bytes / 8);
  double* tab = nullptr;
  double* out = nullptr;
  if (cudaMalloc(&tab, sizeof(double) * (size_t)entries) != cudaSuccess) return -1;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return -1;
  cudaMemset(tab, 0, sizeof(double) * (size_t)entries);
  const int blocks = sms * 8, threads = 256, iters = 512;
  float ms = time_ms([&] { k_ldg_rand<<<blocks, threads>>>(tab, entries, out, iters); });
  *l2_gathers_per_s = (double)blocks * threads * iters * kChains / (ms * 1e-3);
  const int citers = 2048;
  ms = time_ms([&] { k_dcand<<<blocks, threads>>>(out, citers, 0.75, 1e-9); });
  *candidates_per_s = (double)blocks * threads * citers * kChains / (ms * 1e-3);
  cudaFree(tab);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
