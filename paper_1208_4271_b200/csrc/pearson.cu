// Pearson r and non-linearity on the device:
// statistics.cpp:39-51, the two MineStatistics fields next to MIC/MAS/MEV/MCN.
//
//   mean  = sum(x) / n                      (Eigen .mean(): sum() / size())
//   dx    = x - mean;   sxx = sum(dx * dx)  (statistics.cpp:42-44)
//   r     = sum(dx * dy) / sqrt(sxx * syy), clamped to [-1, 1]  (:47-48)
//   r     = NaN if !(sxx > 0) || !(syy > 0)                     (:46)
//   nonlinearity = mic - r * r                                  (:51)
//
// Every sum runs sequentially in sample order, without FMA contraction (the
// library is built with -fmad=false), i.e. the order of the oracle's build of
// the reference; a real-Eigen build vectorises these reductions, so parity is
// stated to 1e-12, bit-exact against the oracle build.
//
// k_center_vars: one thread per variable (the sums are sequential by
// definition); dx is written variable-major so k_pearson_pairs reads each
// variable's row contiguously (L1/L2-resident: V x n x 8 B).
#include <cuda_runtime.h>

#include <cmath>

#include "device_common.cuh"
#include "mine_kernels.h"

namespace mb200 {
namespace {

__global__ void k_center_vars(VarSet vs) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= vs.V) return;
  const int n = vs.n;
  const double* x = vs.vals + (size_t)v * n;
  double* dx = vs.dx + (size_t)v * n;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, x[i]);
  const double mean = __ddiv_rn(s, (double)n);
  double sxx = 0.0;
  for (int i = 0; i < n; ++i) {
    const double d = __dsub_rn(x[i], mean);
    dx[i] = d;
    sxx = __dadd_rn(sxx, __dmul_rn(d, d));
  }
  vs.sxx[v] = sxx;
}

__global__ void k_pearson_pairs(VarSet vs, PairSpace ps, const double* __restrict__ mic,
                                double* pearson, double* nonlin) {
  const long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (w >= ps.count) return;
  int va, vb;
  pair_vars(ps, ps.first + w, va, vb);
  const int n = vs.n;
  const double* a = vs.dx + (size_t)va * n;
  const double* b = vs.dx + (size_t)vb * n;
  const double sxx = vs.sxx[va], syy = vs.sxx[vb];
  double r;
  if (!(sxx > 0.0) || !(syy > 0.0)) {
    r = __longlong_as_double(0x7ff8000000000000LL);  // std::numeric_limits<double>::quiet_NaN()
  } else {
    double sxy = 0.0;
    for (int i = 0; i < n; ++i) sxy = __dadd_rn(sxy, __dmul_rn(__ldg(a + i), __ldg(b + i)));
    r = __ddiv_rn(sxy, __dsqrt_rn(__dmul_rn(sxx, syy)));
    r = r < -1.0 ? -1.0 : (1.0 < r ? 1.0 : r);  // std::clamp(r, -1.0, 1.0)
  }
  if (pearson) pearson[w] = r;
  if (nonlin) nonlin[w] = __dsub_rn(mic[w], __dmul_rn(r, r));
}

// analysis.cpp:98-100: sample variance = sum((x - mean)^2) / (n - 1)
__global__ void k_variances(VarSet vs, double* var) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < vs.V) var[v] = __ddiv_rn(vs.sxx[v], (double)(vs.n - 1));
}

}  // namespace

void launch_variances(const VarSet& vs, double* var, cudaStream_t s) {
  k_variances<<<(vs.V + 127) / 128, 128, 0, s>>>(vs, var);
}

void launch_center_vars(const VarSet& vs, cudaStream_t s) {
  k_center_vars<<<(vs.V + 127) / 128, 128, 0, s>>>(vs);
}

void launch_pearson_pairs(const VarSet& vs, const PairSpace& ps, const double* mic,
                          double* pearson, double* nonlin, cudaStream_t s) {
  if (ps.count <= 0) return;
  k_pearson_pairs<<<(unsigned)((ps.count + 255) / 256), 256, 0, s>>>(vs, ps, mic, pearson, nonlin);
}

}  // namespace mb200
