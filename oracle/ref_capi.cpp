// C entry points over the REFERENCE's own C++ engine, compiled unmodified from
// /root/reference/proj/src against oracle/eigen_shim (see oracle/Makefile).
// TEST INFRASTRUCTURE ONLY: used to pin the C restatement (oracle/mine_oracle.c)
// and the committed golden fixtures, and as the timed CPU reference arm of
// bench.py.  Nothing in the product library links or calls this.
//
// Every function returns 0 on success and -1 if the reference threw; the
// message is then available from ref_last_error().
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "mine/analysis.hpp"
#include "mine/char_matrix.hpp"
#include "mine/io.hpp"
#include "mine/mutual_info.hpp"
#include "mine/oracle.hpp"
#include "mine/partition.hpp"
#include "mine/statistics.hpp"

using namespace mine;

namespace {
thread_local std::string g_err;

Arr1D to_arr(const double* p, int n) {
  Arr1D a(n);
  for (int i = 0; i < n; ++i) a[i] = p[i];
  return a;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

CellCounts cells_from_counts(const int* counts_rowmajor, int rows, int k) {
  CellCounts cells;
  cells.counts = Mat2I::Zero(rows, k);
  for (int r = 0; r < rows; ++r)
    for (int j = 0; j < k; ++j) cells.counts(r, j) = counts_rowmajor[r * k + j];
  cells.cumulative = Mat2I::Zero(rows, k + 1);
  for (int j = 0; j < k; ++j)
    cells.cumulative.col(j + 1) = cells.cumulative.col(j) + cells.counts.col(j);
  cells.boundaries = Arr1I::Zero(k + 1);
  for (int j = 0; j < k; ++j) cells.boundaries[j + 1] = cells.boundaries[j] + cells.counts.col(j).sum();
  return cells;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_grid_bound(long n, double alpha) { return grid_bound(n, alpha); }

// Characteristic matrix in for_each order (y = 2..B/2 outer, x = 2..B/y inner).
// `cells` must hold at least ref_cell_count(B) doubles.
int ref_compute_score(int n, const double* x, const double* y, double alpha, double c,
                      int* bound, double* cells) {
  return guarded([&] {
    const CharacteristicMatrix m = compute_score(to_arr(x, n), to_arr(y, n), Parameters{alpha, c});
    *bound = m.bound();
    long i = 0;
    m.for_each([&](int, int, double v) { cells[i++] = v; });
  });
}

// out6 = mic, mas, mev, mcn, pearson_r, nonlinearity (statistics.hpp:10-17).
int ref_compute_statistics(int n, const double* x, const double* y, double alpha, double c,
                           double* out6) {
  return guarded([&] {
    const MineStatistics s = compute_statistics(to_arr(x, n), to_arr(y, n), Parameters{alpha, c});
    out6[0] = s.mic;
    out6[1] = s.mas;
    out6[2] = s.mev;
    out6[3] = s.mcn;
    out6[4] = s.pearson_r;
    out6[5] = s.nonlinearity;
  });
}

// One compute_score, then the reference's own reductions (statistics.cpp:10-37)
// over that matrix: cells in for_each order plus out4 = mic, mas, mev, mcn.
// Used for the full-size c4 fixtures, where a second compute_score (as
// compute_statistics would run) doubles minutes of CPU time per pair.
int ref_score_statistics(int n, const double* x, const double* y, double alpha, double c,
                         int* bound, double* cells, double* out4) {
  return guarded([&] {
    const CharacteristicMatrix m = compute_score(to_arr(x, n), to_arr(y, n), Parameters{alpha, c});
    *bound = m.bound();
    long i = 0;
    m.for_each([&](int, int, double v) { cells[i++] = v; });
    out4[0] = mic(m);
    out4[1] = mas(m);
    out4[2] = mev(m);
    out4[3] = mcn(m);
  });
}

// Cache-free recount path (oracle.cpp:145-164), guarded to n <= 200.
int ref_reference_statistics(int n, const double* x, const double* y, double alpha, double c,
                             double* out6) {
  return guarded([&] {
    const MineStatistics s =
        reference_statistics(to_arr(x, n), to_arr(y, n), Parameters{alpha, c});
    out6[0] = s.mic;
    out6[1] = s.mas;
    out6[2] = s.mev;
    out6[3] = s.mcn;
    out6[4] = s.pearson_r;
    out6[5] = s.nonlinearity;
  });
}

// The reference batch driver over a variable-major p x n matrix (each variable
// contiguous, like Dataset.values' columns).  mode: 0 all_pairs, 1
// master_vs_all (1-based master), 2 single_pair.  Writes 6 stats per record
// into out (records x 6), returns the record count in *records.
int ref_run_analysis(const double* values, int p, int n, int mode, int a, int b, double alpha,
                     double c, unsigned workers, double* out, long* records) {
  return guarded([&] {
    Dataset ds;
    ds.values.resize(n, p);
    ds.names.reserve(static_cast<std::size_t>(p));
    for (int j = 0; j < p; ++j) {
      ds.names.push_back("V" + std::to_string(j + 1));
      for (int i = 0; i < n; ++i) ds.values(i, j) = values[static_cast<long>(j) * n + i];
    }
    AnalysisTask task;
    task.mode = mode == 0 ? AnalysisMode::all_pairs
                          : (mode == 1 ? AnalysisMode::master_vs_all : AnalysisMode::single_pair);
    task.master = a;
    task.first = a;
    task.second = b;
    task.params = Parameters{alpha, c};
    task.workers = workers;
    long w = 0;
    run_analysis(ds, task, [&](const ResultRecord& rec) {
      double* o = out + 6 * w;
      o[0] = rec.stats.mic;
      o[1] = rec.stats.mas;
      o[2] = rec.stats.mev;
      o[3] = rec.stats.mcn;
      o[4] = rec.stats.pearson_r;
      o[5] = rec.stats.nonlinearity;
      ++w;
    });
    *records = w;
  });
}

// The reference's file-to-file batch path (what run_cli does after parsing,
// cli.cpp:108-118): read_dataset -> run_analysis (optional variance filter)
// -> ResultWriter.  mode / a / b as ref_run_analysis; min_variance < 0: none.
int ref_analysis_file(const char* in_path, const char* out_path, int mode, int a, int b,
                      double alpha, double c, double min_variance, unsigned workers, long* records) {
  return guarded([&] {
    const Dataset ds = read_dataset(in_path);
    AnalysisTask task;
    task.mode = mode == 0 ? AnalysisMode::all_pairs
                          : (mode == 1 ? AnalysisMode::master_vs_all : AnalysisMode::single_pair);
    task.master = a;
    task.first = a;
    task.second = b;
    task.params = Parameters{alpha, c};
    task.workers = workers;
    if (min_variance >= 0.0) task.min_variance = min_variance;
    ResultWriter writer(out_path);
    long w = 0;
    run_analysis(ds, task, [&](const ResultRecord& rec) {
      writer.write(rec);
      ++w;
    });
    writer.close();
    *records = w;
  });
}

// read_dataset (io.cpp:48-120): dimensions, then values (variable-major) and
// the '\n'-joined names.
int ref_read_dataset(const char* path, int* p, int* n, double* values, long cap_values,
                     char* names, long cap_names) {
  return guarded([&] {
    const Dataset ds = read_dataset(path);
    *p = static_cast<int>(ds.p());
    *n = static_cast<int>(ds.n());
    if (values && cap_values >= static_cast<long>(ds.p() * ds.n()))
      for (long j = 0; j < ds.p(); ++j)
        for (long i = 0; i < ds.n(); ++i) values[j * ds.n() + i] = ds.values(i, j);
    std::string joined;
    for (const auto& nm : ds.names) joined += nm + "\n";
    if (names && cap_names > static_cast<long>(joined.size()))
      std::memcpy(names, joined.c_str(), joined.size() + 1);
  });
}

// filter_low_variance (analysis.cpp:92-113) on a variable-major matrix: the
// kept variable indices (0-based) in keep[], their count in *nkeep.
int ref_filter_low_variance(const double* values, int p, int n, double threshold, int* keep,
                            int* nkeep) {
  return guarded([&] {
    Dataset ds;
    ds.values.resize(n, p);
    for (int j = 0; j < p; ++j) {
      ds.names.push_back(std::to_string(j));
      for (int i = 0; i < n; ++i) ds.values(i, j) = values[static_cast<long>(j) * n + i];
    }
    const Dataset out = filter_low_variance(ds, threshold);
    *nkeep = static_cast<int>(out.p());
    for (int j = 0; j < out.p(); ++j) keep[j] = std::stoi(out.names[static_cast<std::size_t>(j)]);
  });
}

// One (orientation, row-target) subproblem replayed through the reference's
// public stage functions exactly as score_orientation calls them
// (char_matrix.cpp:44-56).  Columns are on `col_var`, rows on `row_var`.
// Outputs (caller-sized to n, n+1, x_max-1):
//   row_count, q_x[n] (row label per x-sorted position), clump_count (raw
//   clumps), k (after superclumps), bounds[k+1], h_q, values[x_max-1].
int ref_subproblem(int n, const double* col_var, const double* row_var, int y_target, int x_max,
                   int k_hat, int* row_count, int* q_x, int* clump_count, int* k, int* bounds,
                   double* h_q, double* values) {
  return guarded([&] {
    const Arr1D cv = to_arr(col_var, n), rv = to_arr(row_var, n);
    const SortedPairs by_second = sort_by_second(cv, rv);
    const SortedPairs by_first = sort_by_first(cv, rv);
    const RowPartition q = equipartition_y_axis(by_second, y_target);
    const RowPartition qx = reindex_to_first_order(q, by_second, by_first);
    const ColumnPartition raw = get_clumps_partition(by_first, qx);
    const ColumnPartition p = get_superclumps_partition(by_first, qx, k_hat);
    const CellCounts cells = build_cell_counts(by_first, qx, p);
    const MiProfile prof = optimize_x_axis(cells, x_max);
    *row_count = q.row_count;
    for (int i = 0; i < n; ++i) q_x[i] = qx.assignment[i];
    *clump_count = raw.clump_count;
    *k = p.clump_count;
    for (int j = 0; j <= p.clump_count; ++j) bounds[j] = p.boundaries[j];
    *h_q = prof.h_q;
    for (int l = 0; l < x_max - 1; ++l) values[l] = prof.values[l];
  });
}

// Row map per point (original order) of equipartition_y_axis (1-based).
int ref_equipartition(int n, const double* x, const double* y, int y_target, int* rows_per_point,
                      int* row_count) {
  return guarded([&] {
    const SortedPairs by_second = sort_by_second(to_arr(x, n), to_arr(y, n));
    const RowPartition q = equipartition_y_axis(by_second, y_target);
    for (int i = 0; i < n; ++i) rows_per_point[by_second.order[i]] = q.assignment[i];
    *row_count = q.row_count;
  });
}

// Clump / superclump map per point (original order); k_hat <= 0 means plain clumps.
int ref_clumps(int n, const double* x, const double* y, int y_target, int k_hat, int* cols_per_point,
               int* k) {
  return guarded([&] {
    const Arr1D xs = to_arr(x, n), ys = to_arr(y, n);
    const SortedPairs by_second = sort_by_second(xs, ys);
    const SortedPairs by_first = sort_by_first(xs, ys);
    const RowPartition qx =
        reindex_to_first_order(equipartition_y_axis(by_second, y_target), by_second, by_first);
    const ColumnPartition p =
        k_hat > 0 ? get_superclumps_partition(by_first, qx, k_hat) : get_clumps_partition(by_first, qx);
    for (int i = 0; i < n; ++i) cols_per_point[by_first.order[i]] = p.assignment[i];
    *k = p.clump_count;
  });
}

// optimize_x_axis / brute_force_max_mi on an explicit rows x k count grid.
int ref_optimize_x_axis(const int* counts_rowmajor, int rows, int k, int x, double* values,
                        double* h_q) {
  return guarded([&] {
    const MiProfile prof = optimize_x_axis(cells_from_counts(counts_rowmajor, rows, k), x);
    for (int l = 0; l < x - 1; ++l) values[l] = prof.values[l];
    *h_q = prof.h_q;
  });
}

int ref_brute_force(const int* counts_rowmajor, int rows, int k, int x, double* values,
                    long long* enumerated) {
  return guarded([&] {
    const OracleResult r = brute_force_max_mi(cells_from_counts(counts_rowmajor, rows, k), x);
    for (int l = 0; l < x - 1; ++l) values[l] = r.values[l];
    *enumerated = r.enumerated;
  });
}

int ref_entropy(const double* w, int len, double* out) {
  return guarded([&] {
    Arr1D a(len);
    for (int i = 0; i < len; ++i) a[i] = w[i];
    *out = entropy(a);
  });
}

}  // extern "C"
