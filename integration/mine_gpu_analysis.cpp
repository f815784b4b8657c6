// Batch drop-in for the reference's batch driver.
//
// A maintainer of /root/reference/proj links this translation unit INSTEAD of
// src/analysis.cpp (and mine_gpu_adapter.cpp instead of src/char_matrix.cpp):
// it defines every symbol of the unchanged header include/mine/analysis.hpp.
// mine::run_analysis (analysis.cpp:133-191) no longer scores one pair per
// worker-thread call; it hands whole blocks of the task's pair sequence to the
// GPU batch entry points of include/mine_b200.h -- mine_b200_pairwise over
// condensed-index windows for all_pairs (with reuse_vars after the first
// block, so the per-variable sort / equipartition runs once per job), and
// mine_b200_pairs for master_vs_all / single_pair -- then emits the records in
// PairSequence order, block by block, exactly as the reference does.  Memory
// stays bounded by the block size.  Records are bit-identical to the CPU
// engine's (MIC/MAS/MEV/MCN are the reference's reductions of a bit-identical
// matrix; Pearson r / non-linearity follow statistics.cpp:39-51).
//
// expand_pairs / PairSequence / filter_low_variance keep the reference's
// contract (the pair order and the error messages are part of it); the
// variances of filter_low_variance come from the GPU (mine_b200_variances,
// the same keep set, tests/test_frontend.py).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "mine/analysis.hpp"
#include "mine_b200.h"

namespace mine {

namespace {

[[noreturn]] void fail_from_engine() {
  const std::string msg = mine_b200_last_error();
  throw std::invalid_argument(msg);
}

// One engine context per calling thread, like the per-pair adapter.
mine_b200_ctx* batch_ctx() {
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

void check_index(long long idx, long long p, const char* what) {
  if (idx < 1 || idx > p)
    throw std::out_of_range(std::string("expand_pairs: ") + what + " index out of range");
}

}  // namespace

// analysis.cpp:12-40
std::vector<std::pair<int, int>> expand_pairs(const AnalysisTask& task, Eigen::Index p) {
  const PairSequence seq(task, p);
  std::vector<std::pair<int, int>> pairs;
  pairs.reserve(seq.size());
  for (std::size_t w = 0; w < seq.size(); ++w) pairs.push_back(seq.at(w));
  return pairs;
}

// analysis.cpp:42-64
PairSequence::PairSequence(const AnalysisTask& task, Eigen::Index p)
    : mode_(task.mode), p_(p), master_(task.master), first_(task.first), second_(task.second) {
  switch (mode_) {
    case AnalysisMode::all_pairs:
      size_ = static_cast<std::size_t>(p_ * (p_ - 1) / 2);
      break;
    case AnalysisMode::master_vs_all:
      check_index(master_, p_, "master");
      size_ = static_cast<std::size_t>(p_ - 1);
      break;
    case AnalysisMode::single_pair:
      check_index(first_, p_, "first");
      check_index(second_, p_, "second");
      if (first_ == second_) throw std::invalid_argument("expand_pairs: pair indices must differ");
      size_ = 1;
      break;
  }
}

// analysis.cpp:66-90: w-th pair of the sequence, 1-based.  The all-pairs
// row is found from the end of the condensed order (the row of first index i
// holds p - i pairs).
std::pair<int, int> PairSequence::at(std::size_t w) const {
  if (mode_ == AnalysisMode::master_vs_all) {
    const long long j = static_cast<long long>(w) + 1;
    return {static_cast<int>(master_), static_cast<int>(j < master_ ? j : j + 1)};
  }
  if (mode_ == AnalysisMode::single_pair) return {static_cast<int>(first_), static_cast<int>(second_)};
  const long long total = p_ * (p_ - 1) / 2;
  const long long left = total - static_cast<long long>(w);
  long long rows = static_cast<long long>((std::sqrt(8.0 * static_cast<double>(left) + 1.0) - 1.0) / 2.0);
  while (rows * (rows + 1) / 2 < left) ++rows;
  while (rows >= 1 && (rows - 1) * rows / 2 >= left) --rows;
  const long long i = p_ - rows;
  const long long j = i + 1 + (static_cast<long long>(w) - (total - rows * (rows + 1) / 2));
  return {static_cast<int>(i), static_cast<int>(j)};
}

// analysis.cpp:92-113, variances on the GPU.
Dataset filter_low_variance(const Dataset& dataset, double threshold) {
  if (threshold < 0.0) throw std::invalid_argument("filter_low_variance: threshold must be >= 0");
  const int p = static_cast<int>(dataset.p()), n = static_cast<int>(dataset.n());
  std::vector<double> var(static_cast<std::size_t>(std::max(p, 1)));
  if (p > 0 && mine_b200_variances(batch_ctx(), dataset.values.data(), p, n, var.data()) != 0)
    fail_from_engine();
  std::vector<Eigen::Index> keep;
  for (int j = 0; j < p; ++j)
    if (!(var[static_cast<std::size_t>(j)] < threshold)) keep.push_back(j);
  if (keep.empty()) throw std::invalid_argument("filter_low_variance: no variables pass the threshold");
  Dataset out;
  out.values.resize(n, static_cast<Eigen::Index>(keep.size()));
  out.names.reserve(keep.size());
  for (std::size_t j = 0; j < keep.size(); ++j) {
    out.values.col(static_cast<Eigen::Index>(j)) = dataset.values.col(keep[j]);
    out.names.push_back(dataset.names[static_cast<std::size_t>(keep[j])]);
  }
  return out;
}

// analysis.cpp:133-191 on the GPU: blocks of the pair sequence are scored by
// one batch call each and emitted in order.
void run_analysis(const Dataset& dataset, const AnalysisTask& task,
                  const std::function<void(const ResultRecord&)>& emit) {
  if (task.workers < 1) throw std::invalid_argument("run_analysis: workers must be positive");
  const Dataset* ds = &dataset;
  Dataset filtered;
  if (task.min_variance) {
    filtered = filter_low_variance(dataset, *task.min_variance);
    ds = &filtered;
  }
  const PairSequence pairs(task, ds->p());
  const std::size_t total = pairs.size();
  if (total == 0) return;
  const int p = static_cast<int>(ds->p()), n = static_cast<int>(ds->n());
  if (n < 2) throw std::invalid_argument("compute_score: need at least 2 samples");
  // Mat2D is column-major: column j (variable j) is contiguous, i.e. the
  // values are already the p x n variable-major matrix the ABI takes.
  const double* vars = ds->values.data();
  const mine_parameter par{task.params.alpha, task.params.c, MINE_EST_MIC_APPROX};
  mine_b200_ctx* ctx = batch_ctx();

  constexpr std::size_t kBlock = std::size_t(1) << 20;
  const std::size_t block = std::min(kBlock, total);
  std::vector<double> mic(block), mas(block), mev(block), mcn(block), r(block), nl(block);
  std::vector<int> xi, yi;
  ResultRecord rec;
  for (std::size_t base = 0; base < total; base += block) {
    const std::size_t count = std::min(block, total - base);
    mine_stats_out out{};
    out.mic = mic.data();
    out.mas = mas.data();
    out.mev = mev.data();
    out.mcn = mcn.data();
    out.pearson_r = r.data();
    out.nonlinearity = nl.data();
    int rc;
    if (task.mode == AnalysisMode::all_pairs) {
      mine_b200_opts o{};
      o.first = static_cast<long long>(base);
      o.count = static_cast<long long>(count);
      o.reuse_vars = base > 0;  // the same variables for every block of the job
      rc = mine_b200_pairwise(ctx, vars, p, n, &par, &o, &out);
    } else if (task.mode == AnalysisMode::single_pair) {
      // only the two variables are validated and scored, as score_pair does
      const auto [i, j] = pairs.at(0);
      const int lo = std::min(i, j) - 1, hi = std::max(i, j) - 1;
      std::vector<double> two(2 * static_cast<std::size_t>(n));
      std::memcpy(two.data(), vars + static_cast<std::size_t>(lo) * n, sizeof(double) * n);
      std::memcpy(two.data() + n, vars + static_cast<std::size_t>(hi) * n, sizeof(double) * n);
      const int a = 0, b = 1;
      rc = mine_b200_pairs(ctx, two.data(), 2, n, &a, &b, 1, &par, nullptr, &out);
    } else {
      // score_pair (analysis.cpp:117-129) orients every record lower index first
      xi.resize(count);
      yi.resize(count);
      for (std::size_t w = 0; w < count; ++w) {
        const auto [i, j] = pairs.at(base + w);
        xi[w] = std::min(i, j) - 1;
        yi[w] = std::max(i, j) - 1;
      }
      mine_b200_opts o{};
      o.reuse_vars = base > 0;
      rc = mine_b200_pairs(ctx, vars, p, n, xi.data(), yi.data(), static_cast<long long>(count),
                           &par, &o, &out);
    }
    if (rc != 0) fail_from_engine();
    for (std::size_t w = 0; w < count; ++w) {
      const auto [i, j] = pairs.at(base + w);
      const int lo = std::min(i, j), hi = std::max(i, j);
      rec.name_x = ds->names[static_cast<std::size_t>(lo - 1)];
      rec.name_y = ds->names[static_cast<std::size_t>(hi - 1)];
      rec.stats.mic = mic[w];
      rec.stats.mas = mas[w];
      rec.stats.mev = mev[w];
      rec.stats.mcn = mcn[w];
      rec.stats.pearson_r = r[w];
      rec.stats.nonlinearity = nl[w];
      emit(rec);
    }
  }
}

std::vector<ResultRecord> run_analysis(const Dataset& dataset, const AnalysisTask& task) {
  std::vector<ResultRecord> out;
  run_analysis(dataset, task, [&](const ResultRecord& rec) { out.push_back(rec); });
  return out;
}

}  // namespace mine
