// Drop-in GPU backend for the reference's hot path.
//
// A maintainer of /root/reference/proj links this translation unit INSTEAD of
// src/char_matrix.cpp: it defines the same functions against the unchanged
// header include/mine/char_matrix.hpp, and mine::compute_score
// (char_matrix.cpp:70-81) now runs on the B200 through the C ABI of
// include/mine_b200.h.  Everything above it -- compute_statistics
// (statistics.cpp:53-63), run_analysis (analysis.cpp:133-191) and the CLI --
// is untouched and keeps its semantics; the characteristic matrix it receives
// is bit-identical to the CPU engine's.  See INTEGRATION.md.
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "mine/char_matrix.hpp"
#include "mine_b200.h"

namespace mine {

// char_matrix.cpp:11-15
void validate_parameters(const Parameters& params) {
  if (!(params.alpha > 0.0) || params.alpha > 1.0)
    throw std::invalid_argument("parameters: alpha must be in (0, 1]");
  if (!(params.c > 0.0)) throw std::invalid_argument("parameters: c must be > 0");
}

// char_matrix.cpp:17-20 (same arithmetic, computed by the library)
int grid_bound(Eigen::Index n, double alpha) {
  return mine_b200_grid_bound(static_cast<long long>(n), alpha);
}

// char_matrix.cpp:22-26: jagged storage, one row per y = 2..B/2.
CharacteristicMatrix::CharacteristicMatrix(int bound) : bound_(bound) {
  rows_.reserve(static_cast<std::size_t>(max_row_target() > 1 ? max_row_target() - 1 : 0));
  for (int y = 2; y <= max_row_target(); ++y) rows_.push_back(Arr1D::Zero(max_col_target(y) - 1));
}

// char_matrix.cpp:28-35
void CharacteristicMatrix::update_max(int x, int y, double value) {
  if (value > 1.0) value = 1.0;
  double& slot = rows_[y - 2][x - 2];
  if (value > slot) slot = value;
}

namespace {
// One engine context per calling thread (run_analysis scores pairs from
// several worker threads, analysis.cpp:163-187).
mine_b200_ctx* thread_ctx() {
  struct Holder {
    mine_b200_ctx* ctx = nullptr;
    ~Holder() { mine_b200_destroy(ctx); }
  };
  thread_local Holder h;
  if (!h.ctx) {
    h.ctx = mine_b200_create(0);
    if (!h.ctx) throw std::runtime_error(std::string("mine_b200: ") + mine_b200_last_error());
  }
  return h.ctx;
}
}  // namespace

// char_matrix.cpp:70-81, on the GPU.  The two per-orientation matrices come
// back from the device and are merged with the reference's own update_max,
// in the reference's order (orientation xs->ys first).
CharacteristicMatrix compute_score(const Arr1D& xs, const Arr1D& ys, const Parameters& params) {
  validate_parameters(params);
  if (xs.size() != ys.size()) throw std::invalid_argument("compute_score: input lengths differ");
  if (xs.size() < 2) throw std::invalid_argument("compute_score: need at least 2 samples");
  if (!xs.allFinite() || !ys.allFinite())
    throw std::invalid_argument("compute_score: inputs must be finite");
  const int n = static_cast<int>(xs.size());
  CharacteristicMatrix m(grid_bound(n, params.alpha));
  const int ncell = mine_b200_cell_count(m.bound());
  std::vector<double> vars(2 * static_cast<std::size_t>(n)), cells(2 * static_cast<std::size_t>(ncell));
  for (int i = 0; i < n; ++i) {
    vars[i] = xs[i];
    vars[n + i] = ys[i];
  }
  const int xi = 0, yi = 1;
  double mic = 0.0;
  mine_stats_out out{};
  out.mic = &mic;
  out.cells = cells.data();
  const mine_parameter par{params.alpha, params.c, MINE_EST_MIC_APPROX};
  if (mine_b200_pairs(thread_ctx(), vars.data(), 2, n, &xi, &yi, 1, &par, nullptr, &out) != 0)
    throw std::invalid_argument(mine_b200_last_error());
  int c = 0;
  for (int y = 2; y <= m.max_row_target(); ++y)
    for (int x = 2; x <= m.max_col_target(y); ++x, ++c) m.update_max(x, y, cells[c]);
  c = 0;
  for (int y = 2; y <= m.max_row_target(); ++y)
    for (int x = 2; x <= m.max_col_target(y); ++x, ++c) m.update_max(x, y, cells[ncell + c]);
  return m;
}

}  // namespace mine
