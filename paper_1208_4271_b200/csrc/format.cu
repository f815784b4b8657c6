// Results-file records on the device: format_record
// (io.cpp:37-47) for a block of pairs, straight from the HBM-resident
// statistics -- "name_x,name_y,MIC,MAS,MEV,MCN,pearson,nonlinearity\n" with
// "%.6g" values and "nan" -- into one contiguous text buffer, so only the
// text crosses PCIe and the host only writes it.
//
// "%.6g" is the exact integer algorithm of records.cpp fmt6g_fast (the same
// text glibc's printf produces: exact scaling of v = m 2^e by a power of ten in
// 128-bit integers, ties to even, exponent after rounding, trailing zeros
// stripped).  Values outside 1e-17 <= |v| < 1e15 raise a flag and the host
// formats that block instead (no MINE statistic gets there).
//
//   k_rec_len   one thread per record: its byte length (and the fallback flag)
//   k_scan_*    exclusive scan of the lengths (tile sums, their scan, tile scans)
//   k_rec_write one thread per record: the bytes at its offset
#include "device_common.cuh"
#include "mine_kernels.h"

namespace mb200 {
namespace {

__device__ __forceinline__ int fmt6g_dev(double v, char* out, bool& fallback) {
  if (isnan(v)) {
    out[0] = 'n', out[1] = 'a', out[2] = 'n';
    return 3;
  }
  char* o = out;
  if (signbit(v)) *o++ = '-';
  if (v == 0.0) {
    *o++ = '0';
    return (int)(o - out);
  }
  const double a = fabs(v);
  if (!(a >= 1e-17) || !(a < 1e15)) {
    fallback = true;
    return 0;
  }
  int e2;
  const double fr = frexp(a, &e2);
  const unsigned long long m = (unsigned long long)ldexp(fr, 53);  // exact
  const int e = e2 - 53;
  int X = (int)floor((e2 - 1) * 0.30102999566398120);
  unsigned long long D = 0;
  for (int iter = 0; iter < 4; ++iter) {
    const int p = 5 - X;
    if (p < -9 || p > 22 || e >= 0) {
      fallback = true;
      return 0;
    }
    unsigned __int128 num = m, den = 1;
    const int pp = p >= 0 ? p : -p;
    unsigned __int128 p10 = 1;
    for (int i = 0; i < pp; ++i) p10 *= 10u;
    unsigned __int128 q, r;
    const int s = -e;
    if (p >= 0) {
      num = (unsigned __int128)m * p10;
      if (s >= 127) {
        fallback = true;
        return 0;
      }
      q = num >> s;
      r = num - (q << s);
      den = (unsigned __int128)1 << s;
    } else {
      den = p10 << s;
      q = num / den;
      r = num - q * den;
    }
    if (q < 100000) {
      --X;
      continue;
    }
    if (q >= 1000000) {
      ++X;
      continue;
    }
    D = (unsigned long long)q;
    if (2 * r > den || (2 * r == den && (D & 1))) ++D;
    if (D == 1000000) {
      D = 100000;
      ++X;
    }
    break;
  }
  if (D == 0) {
    fallback = true;
    return 0;
  }
  char dig[6];
  for (int i = 5; i >= 0; --i, D /= 10) dig[i] = (char)('0' + D % 10);
  int nd = 6;
  while (nd > 1 && dig[nd - 1] == '0') --nd;
  if (X >= -4 && X < 6) {
    if (X >= 0) {
      for (int i = 0; i <= X; ++i) *o++ = i < nd ? dig[i] : '0';
      if (nd > X + 1) {
        *o++ = '.';
        for (int i = X + 1; i < nd; ++i) *o++ = dig[i];
      }
    } else {
      *o++ = '0';
      *o++ = '.';
      for (int i = 0; i < -X - 1; ++i) *o++ = '0';
      for (int i = 0; i < nd; ++i) *o++ = dig[i];
    }
  } else {
    *o++ = dig[0];
    if (nd > 1) {
      *o++ = '.';
      for (int i = 1; i < nd; ++i) *o++ = dig[i];
    }
    *o++ = 'e';
    *o++ = X < 0 ? '-' : '+';
    const int ax = X < 0 ? -X : X;
    if (ax >= 100) *o++ = (char)('0' + ax / 100);
    *o++ = (char)('0' + ax / 10 % 10);
    *o++ = (char)('0' + ax % 10);
  }
  return (int)(o - out);
}

struct RecArgs {
  PairSpace ps;                 // pair w -> (x, y) of the call; records print min/max
  const double* stat[6];        // mic mas mev mcn pearson nonlinearity (indexed w - 0)
  const char* names;            // concatenated labels
  const long long* name_off;    // p + 1 offsets into names
  long long count;
};

// The record of pair w into out (<= 2 names + 6 x 13 + 8 bytes); returns the
// byte count.  out == nullptr: length only.
__device__ int record(const RecArgs& a, long long w, char* out, bool& fallback) {
  int x, y;
  pair_vars(a.ps, a.ps.first + w, x, y);
  const int lo = min(x, y), hi = max(x, y);
  char buf[16];
  int len = 0;
  auto put_name = [&](int v) {
    const long long b = a.name_off[v], e = a.name_off[v + 1];
    if (out)
      for (long long i = b; i < e; ++i) out[len + (i - b)] = a.names[i];
    len += (int)(e - b);
  };
  put_name(lo);
  if (out) out[len] = ',';
  ++len;
  put_name(hi);
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    if (out) out[len] = ',';
    ++len;
    const int n = fmt6g_dev(a.stat[k][w], buf, fallback);
    if (out)
      for (int i = 0; i < n; ++i) out[len + i] = buf[i];
    len += n;
  }
  if (out) out[len] = '\n';
  return len + 1;
}

__global__ void k_rec_len(RecArgs a, unsigned long long* len, int* fallback) {
  const long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (w >= a.count) return;
  bool fb = false;
  len[w] = (unsigned long long)record(a, w, nullptr, fb);
  if (fb) *fallback = 1;
}

__global__ void k_rec_write(RecArgs a, const unsigned long long* off, char* text) {
  const long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (w >= a.count) return;
  bool fb = false;
  record(a, w, text + off[w], fb);
}

// test hook: "%.6g" of n values into 24-byte slots (length 0: host fallback)
__global__ void k_format_values(const double* v, long long n, char* out, int* len) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool fb = false;
  char buf[24];
  const int l = fmt6g_dev(v[i], buf, fb);
  len[i] = fb ? 0 : l;
  for (int k = 0; k < l; ++k) out[i * 24 + k] = buf[k];
}

// Exclusive scan of m 64-bit lengths in tiles of kScanTile: per-tile sums, a
// one-CTA scan of the tile sums (m <= 2^31: at most 2^18 tiles), then each
// tile's own scan from its offset.  Three launches, ~3 passes over 8 m bytes.
constexpr int kScanThreads = 1024, kScanPer = 8, kScanTile = kScanThreads * kScanPer;

__device__ __forceinline__ unsigned long long block_excl_scan_u64(unsigned long long v,
                                                                  unsigned long long* total) {
  __shared__ unsigned long long wsum[32];
  __shared__ unsigned long long btot;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();  // wsum / btot of a previous call are no longer read
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned long long t = lane < nw ? wsum[lane] : 0ull, u = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, u, o);
      if (lane >= o) u += y;
    }
    if (lane < nw) wsum[lane] = u - t;
    if (lane == 31) btot = u;
  }
  __syncthreads();
  if (total) *total = btot;
  return x - v + wsum[w];
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tile_sums(const unsigned long long* in, long long m,
                                                                 unsigned long long* tile_sum) {
  const long long base = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanPer;
  unsigned long long v = 0;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i)
    if (base + i < m) v += in[base + i];
  unsigned long long tot;
  block_excl_scan_u64(v, &tot);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tile_offsets(unsigned long long* tile_sum, int tiles) {
  unsigned long long carry = 0;
  for (int t0 = 0; t0 < tiles; t0 += kScanThreads) {
    const int t = t0 + threadIdx.x;
    const unsigned long long v = t < tiles ? tile_sum[t] : 0ull;
    unsigned long long tot;
    const unsigned long long ex = block_excl_scan_u64(v, &tot);
    if (t < tiles) tile_sum[t] = carry + ex;
    carry += tot;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const unsigned long long* in, long long m,
                                                             const unsigned long long* tile_off,
                                                             unsigned long long* out) {
  const long long base = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanPer;
  unsigned long long x[kScanPer], v = 0;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    x[i] = base + i < m ? in[base + i] : 0ull;
    v += x[i];
  }
  unsigned long long run = tile_off[blockIdx.x] + block_excl_scan_u64(v, nullptr);
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    if (base + i < m) out[base + i] = run;
    run += x[i];
  }
}

}  // namespace

cudaError_t format_values_device(const double* v, long long n, char* out, int* len, cudaStream_t s) {
  k_format_values<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(v, n, out, len);
  return cudaGetLastError();
}

size_t format_scratch_bytes(long long count) {
  const size_t tiles = (size_t)(count + 1 + kScanTile - 1) / kScanTile;
  return sizeof(unsigned long long) * (2 * (size_t)(count + 1) + tiles) + 256;
}

// Formats records [0, count) of the pair space; returns the text size in
// bytes (in *bytes) once the stream is synchronised, or *fallback != 0.
cudaError_t launch_format_records(const PairSpace& ps, const double* const stat[6],
                                  const char* names, const long long* name_off, long long count,
                                  void* scratch, char* text, size_t text_cap, size_t* bytes,
                                  int* d_flag, int* h_fallback, cudaStream_t s) {
  RecArgs a;
  a.ps = ps;
  for (int k = 0; k < 6; ++k) a.stat[k] = stat[k];
  a.names = names;
  a.name_off = name_off;
  a.count = count;
  auto* len = static_cast<unsigned long long*>(scratch);
  auto* off = len + (count + 1);
  auto* tile_sum = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(off + (count + 1)) + 255) & ~uintptr_t(255));
  const long long m = count + 1;
  const int tiles = (int)((m + kScanTile - 1) / kScanTile);
  cudaMemsetAsync(d_flag, 0, sizeof(int), s);
  cudaMemsetAsync(len + count, 0, sizeof(unsigned long long), s);
  const unsigned blocks = (unsigned)((count + 255) / 256);
  k_rec_len<<<blocks, 256, 0, s>>>(a, len, d_flag);
  k_scan_tile_sums<<<tiles, kScanThreads, 0, s>>>(len, m, tile_sum);
  k_scan_tile_offsets<<<1, kScanThreads, 0, s>>>(tile_sum, tiles);
  k_scan_tiles<<<tiles, kScanThreads, 0, s>>>(len, m, tile_sum, off);
  unsigned long long total = 0;
  cudaMemcpyAsync(&total, off + count, sizeof total, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(h_fallback, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  *bytes = (size_t)total;
  if (*h_fallback || total > text_cap) return cudaSuccess;
  k_rec_write<<<blocks, 256, 0, s>>>(a, off, text);
  return cudaGetLastError();
}

}  // namespace mb200
