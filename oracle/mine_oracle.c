/* CPU restatement of the reference MINE engine -- TEST INFRASTRUCTURE ONLY.
 * See mine_oracle.h for scope, pinning and the extension definitions.
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  Build: oracle/Makefile (-ffp-contract=off: like the
 * reference's x86-64 build, no FMA contraction anywhere). */
#define _GNU_SOURCE
#include "mine_oracle.h"

#include <float.h>
#include <limits.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
const char* mo_last_error(void) { return g_err; }
static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}

/* std::max / std::min with the libstdc++ argument order: max(a,b) = a<b?b:a. */
static inline double dmax(double a, double b) { return a < b ? b : a; }
static inline double dmin(double a, double b) { return b < a ? b : a; }

/* ------------------------------------------------------------------------ */
/* partition.cpp:13-38 sort_pairs: std::stable_sort of indices by (p, q)
 * with `p[l] != p[r] ? p[l] < p[r] : q[l] < q[r]`, then gather.            */
typedef struct {
  double* a;
  double* b;
  int* order;
  int n;
} sorted_pairs;

static int pair_less(const double* p, const double* q, int l, int r) {
  return p[l] != p[r] ? p[l] < p[r] : q[l] < q[r];
}

/* Bottom-up merge sort: stable, so the result equals std::stable_sort's. */
static void stable_sort_idx(int* idx, int n, const double* p, const double* q) {
  int* tmp = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  for (int w = 1; w < n; w *= 2) {
    for (int lo = 0; lo < n; lo += 2 * w) {
      int mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
      int i = lo, j = mid, o = lo;
      while (i < mid && j < hi) tmp[o++] = pair_less(p, q, idx[j], idx[i]) ? idx[j++] : idx[i++];
      while (i < mid) tmp[o++] = idx[i++];
      while (j < hi) tmp[o++] = idx[j++];
    }
    memcpy(idx, tmp, sizeof(int) * (size_t)n);
  }
  free(tmp);
}

static void sort_pairs(const double* x, const double* y, int n, int by_second, sorted_pairs* out) {
  out->n = n;
  out->a = (double*)malloc(sizeof(double) * (size_t)n);
  out->b = (double*)malloc(sizeof(double) * (size_t)n);
  out->order = (int*)malloc(sizeof(int) * (size_t)n);
  for (int i = 0; i < n; ++i) out->order[i] = i;
  if (by_second)
    stable_sort_idx(out->order, n, y, x);
  else
    stable_sort_idx(out->order, n, x, y);
  for (int i = 0; i < n; ++i) {
    out->a[i] = x[out->order[i]];
    out->b[i] = y[out->order[i]];
  }
}

static void free_pairs(sorted_pairs* s) {
  free(s->a);
  free(s->b);
  free(s->order);
}

/* partition.cpp:42-67 equipartition_runs: greedy scan over tie runs; the
 * desired row size stays a real number.  Returns row_count. */
static int equipartition_runs(const double* values, int n, int rows, int* assignment) {
  double desired = (double)n / (double)rows;
  int curr = 1, in_row = 0, i = 0;
  while (i < n) {
    int j = i + 1;
    while (j < n && values[j] == values[i]) ++j;
    const int run = j - i;
    if (in_row != 0 && fabs((double)(in_row + run) - desired) >= fabs((double)in_row - desired)) {
      ++curr;
      in_row = 0;
      desired = (double)(n - i) / (double)(rows - curr + 1); /* :58-59 */
    }
    for (int t = i; t < j; ++t) assignment[t] = curr;
    in_row += run;
    i = j;
  }
  return curr;
}

/* partition.cpp:69-74 */
static void boundaries_from_assignment(const int* assignment, int n, int k, int* bounds) {
  for (int j = 0; j <= k; ++j) bounds[j] = 0;
  for (int i = 0; i < n; ++i) bounds[assignment[i]] += 1;
  for (int j = 1; j <= k; ++j) bounds[j] += bounds[j - 1];
}

/* partition.cpp:94-106 reindex_to_first_order */
static void reindex_to_first_order(const int* q, const sorted_pairs* by_second,
                                   const sorted_pairs* by_first, int* qx) {
  const int n = by_second->n;
  int* per_point = (int*)malloc(sizeof(int) * (size_t)n);
  for (int i = 0; i < n; ++i) per_point[by_second->order[i]] = q[i];
  for (int i = 0; i < n; ++i) qx[i] = per_point[by_first->order[i]];
  free(per_point);
}

/* partition.cpp:108-146 get_clumps_partition (Alg. 1): sentinel-fuse x-tie runs
 * spanning several rows, then a new clump at every label change. Returns k. */
static int get_clumps_partition(const sorted_pairs* pts, const int* q, int* assignment) {
  const int n = pts->n;
  int* labels = (int*)malloc(sizeof(int) * (size_t)n);
  memcpy(labels, q, sizeof(int) * (size_t)n);
  int sentinel = -1, i = 0;
  while (i < n) {
    int j = i + 1, spans_rows = 0;
    while (j < n && pts->a[j] == pts->a[i]) {
      if (labels[j] != labels[i]) spans_rows = 1;
      ++j;
    }
    if (spans_rows) {
      for (int t = i; t < j; ++t) labels[t] = sentinel;
      --sentinel;
    }
    i = j;
  }
  assignment[0] = 1;
  int k = 1;
  for (int t = 1; t < n; ++t) {
    if (labels[t] != labels[t - 1]) ++k;
    assignment[t] = k;
  }
  free(labels);
  return k;
}

/* partition.cpp:148-165 get_superclumps_partition (Alg. 2). Writes the final
 * assignment and boundaries (size >= k+1); returns k; *raw_k = plain clumps. */
static int get_superclumps_partition(const sorted_pairs* pts, const int* q, int k_hat,
                                     int* assignment, int* bounds, int* raw_k) {
  const int n = pts->n;
  int k = get_clumps_partition(pts, q, assignment);
  if (raw_k) *raw_k = k;
  if (k > k_hat) {
    double* ordinals = (double*)malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) ordinals[i] = (double)assignment[i];
    k = equipartition_runs(ordinals, n, k_hat, assignment);
    free(ordinals);
  }
  boundaries_from_assignment(assignment, n, k, bounds);
  return k;
}

/* ------------------------------------------------------------------------ */
/* mutual_info.hpp:16-31 entropy: sequential total, then acc += p*log(p) over
 * positive weights, returns -acc (nats). */
static double entropy_w(const double* w, int len) {
  double total = 0.0;
  for (int i = 0; i < len; ++i) total += w[i];
  double acc = 0.0;
  for (int i = 0; i < len; ++i) {
    if (w[i] > 0.0) {
      const double p = w[i] / total;
      acc += p * log(p);
    }
  }
  return -acc;
}

/* mutual_info.cpp:26-72 optimize_x_axis.  cum is rows x (k+1) row-major
 * (cumulative counts over clumps, mutual_info.cpp:9-24), c the boundaries. */
static void optimize_x_axis(const int* cum, const int* cb, int rows, int k, int x, double* values,
                            double* h_q_out) {
  const int kk = k + 1;
  double* w = (double*)malloc(sizeof(double) * (size_t)(2 * rows + 2));
  for (int r = 0; r < rows; ++r) w[r] = (double)cum[r * kk + k];
  const double h_q = entropy_w(w, rows); /* :33 */
  *h_q_out = h_q;
  for (int l = 0; l < x - 1; ++l) values[l] = 0.0;
  if (k < 2) { /* :34 */
    free(w);
    return;
  }
  double* c = (double*)malloc(sizeof(double) * (size_t)kk);
  for (int j = 0; j <= k; ++j) c[j] = (double)cb[j];

  /* :39-41 h_span(s, t) = entropy(cum.col(t) - cum.col(s)) */
  double* h_span = (double*)malloc(sizeof(double) * (size_t)kk * (size_t)kk);
  for (int s = 0; s < k; ++s)
    for (int t = s + 1; t <= k; ++t) {
      for (int r = 0; r < rows; ++r) w[r] = (double)(cum[r * kk + t] - cum[r * kk + s]);
      h_span[(size_t)s * kk + t] = entropy_w(w, rows);
    }

  const int l_max = x < k ? x : k; /* :43 */
  const int lw = l_max + 1;
  double* f = (double*)malloc(sizeof(double) * (size_t)kk * (size_t)lw);
  for (size_t i = 0; i < (size_t)kk * (size_t)lw; ++i) f[i] = -DBL_MAX;
  /* :47-56 F(t,2) = max_s H(P) - H(P,Q) */
  for (int t = 2; t <= k; ++t) {
    double best = -DBL_MAX;
    for (int s = 1; s < t; ++s) {
      double two[2] = {c[s], c[t] - c[s]};
      const double h_p = entropy_w(two, 2);
      for (int r = 0; r < rows; ++r) {
        w[r] = (double)cum[r * kk + s];
        w[rows + r] = (double)(cum[r * kk + t] - cum[r * kk + s]);
      }
      const double cand = h_p - entropy_w(w, 2 * rows); /* entropy_joint == entropy(concat) */
      best = dmax(best, cand);
    }
    f[(size_t)t * lw + 2] = best;
  }
  /* :57-66 F(t,l) = max_s (c_s/c_t) F(s,l-1) - ((c_t-c_s)/c_t) h_span(s,t) */
  for (int l = 3; l <= l_max; ++l) {
    for (int t = l; t <= k; ++t) {
      double best = -DBL_MAX;
      for (int s = l - 1; s < t; ++s) {
        const double cand = (c[s] / c[t]) * f[(size_t)s * lw + l - 1] -
                            ((c[t] - c[s]) / c[t]) * h_span[(size_t)s * kk + t];
        best = dmax(best, cand);
      }
      f[(size_t)t * lw + l] = best;
    }
  }
  /* :68-70 */
  for (int l = 2; l <= x; ++l)
    values[l - 2] = l <= l_max ? dmax(0.0, h_q + f[(size_t)k * lw + l]) : values[l_max - 2];
  free(f);
  free(h_span);
  free(c);
  free(w);
}

/* mutual_info.cpp:9-24 build_cell_counts -> cumulative rows x (k+1) row-major */
static void build_cumulative(const int* q, const int* p, int n, int rows, int k, int* cum) {
  const int kk = k + 1;
  memset(cum, 0, sizeof(int) * (size_t)rows * (size_t)kk);
  for (int i = 0; i < n; ++i) cum[(q[i] - 1) * kk + p[i]] += 1; /* counts in col p (1-based) */
  for (int r = 0; r < rows; ++r)
    for (int j = 1; j <= k; ++j) cum[r * kk + j] += cum[r * kk + j - 1];
}

int mo_optimize_x_axis(const int* counts_rowmajor, int rows, int k, int x, double* values,
                       double* h_q) {
  if (x < 2) return fail("optimize_x_axis: column target must be >= 2");
  int* cum = (int*)calloc((size_t)rows * (size_t)(k + 1), sizeof(int));
  int* cb = (int*)calloc((size_t)(k + 1), sizeof(int));
  for (int r = 0; r < rows; ++r)
    for (int j = 0; j < k; ++j) cum[r * (k + 1) + j + 1] = cum[r * (k + 1) + j] + counts_rowmajor[r * k + j];
  for (int j = 0; j <= k; ++j)
    for (int r = 0; r < rows; ++r) cb[j] += cum[r * (k + 1) + j];
  optimize_x_axis(cum, cb, rows, k, x, values, h_q);
  free(cum);
  free(cb);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* char_matrix.cpp:17-20 grid_bound */
int mo_grid_bound(long n, double alpha) {
  const int b = (int)floor(pow((double)n, alpha));
  return b > 4 ? b : 4;
}

/* char_matrix.hpp:43-47 for_each order: y = 2..B/2, x = 2..B/y */
int mo_cell_count(int bound) {
  int cnt = 0;
  for (int y = 2; y <= bound / 2; ++y) cnt += bound / y - 1;
  return cnt;
}
static int cell_index(int bound, int x, int y) {
  int off = 0;
  for (int yy = 2; yy < y; ++yy) off += bound / yy - 1;
  return off + x - 2;
}

/* char_matrix.cpp:28-35 update_max */
static void update_max(double* slot, double value) {
  if (value > 1.0) value = 1.0;
  if (value > *slot) *slot = value;
}

typedef struct {
  int n, y_target, x_max, k_hat;
  const sorted_pairs *by_second, *by_first;
  int *q, *qx, *assign, *bounds, *cum;
  int row_count, raw_k, k;
  double h_q;
  double* values;
} subproblem;

/* The stage sequence of score_orientation (char_matrix.cpp:49-56). */
static void run_subproblem(subproblem* s) {
  s->row_count = equipartition_runs(s->by_second->b, s->n, s->y_target, s->q);   /* :49 */
  reindex_to_first_order(s->q, s->by_second, s->by_first, s->qx);                /* :51 */
  s->k = get_superclumps_partition(s->by_first, s->qx, s->k_hat, s->assign, s->bounds,
                                   &s->raw_k);                                    /* :54 */
  s->cum = (int*)malloc(sizeof(int) * (size_t)s->row_count * (size_t)(s->k + 1));
  build_cumulative(s->qx, s->assign, s->n, s->row_count, s->k, s->cum);          /* :55 */
  optimize_x_axis(s->cum, s->bounds, s->row_count, s->k, s->x_max, s->values, &s->h_q); /* :56 */
  free(s->cum);
}

static int k_hat_for(double c, int x_max) { /* char_matrix.cpp:52-53 */
  const int kh = (int)floor(c * (double)x_max);
  return kh > 1 ? kh : 1;
}

/* char_matrix.cpp:42-66 score_orientation, into a per-orientation matrix o
 * (cells: (l, y), or (y, l) when swapped). */
static void score_orientation(const double* col_var, const double* row_var, int n, int bound,
                              double c, int swapped, double* o) {
  sorted_pairs by_second, by_first;
  sort_pairs(col_var, row_var, n, 1, &by_second); /* :44 */
  sort_pairs(col_var, row_var, n, 0, &by_first);  /* :45 */
  int* q = (int*)malloc(sizeof(int) * (size_t)n);
  int* qx = (int*)malloc(sizeof(int) * (size_t)n);
  int* assign = (int*)malloc(sizeof(int) * (size_t)n);
  int* bounds = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  double* values = (double*)malloc(sizeof(double) * (size_t)(bound + 1));
  for (int y = 2; y <= bound / 2; ++y) {
    subproblem s = {0};
    s.n = n;
    s.y_target = y;
    s.x_max = bound / y;
    s.k_hat = k_hat_for(c, s.x_max);
    s.by_second = &by_second;
    s.by_first = &by_first;
    s.q = q;
    s.qx = qx;
    s.assign = assign;
    s.bounds = bounds;
    s.values = values;
    run_subproblem(&s);
    const double norm_rows = log((double)s.row_count); /* :50 */
    for (int l = 2; l <= s.x_max; ++l) {               /* :57-64 */
      const double norm = dmin(log((double)l), norm_rows);
      const double value = norm > 0.0 ? values[l - 2] / norm : 0.0;
      update_max(&o[swapped ? cell_index(bound, y, l) : cell_index(bound, l, y)], value);
    }
  }
  free(values);
  free(bounds);
  free(assign);
  free(qx);
  free(q);
  free_pairs(&by_second);
  free_pairs(&by_first);
}

/* char_matrix.cpp:11-15 + :71-75 validation */
static int validate(int n, const double* x, const double* y, double alpha, double c) {
  if (!(alpha > 0.0) || alpha > 1.0) return fail("parameters: alpha must be in (0, 1]");
  if (!(c > 0.0)) return fail("parameters: c must be > 0");
  if (n < 2) return fail("compute_score: need at least 2 samples");
  for (int i = 0; i < n; ++i)
    if (!isfinite(x[i]) || !isfinite(y[i])) return fail("compute_score: inputs must be finite");
  return 0;
}

int mo_compute_score(int n, const double* x, const double* y, double alpha, double c, double* o1,
                     double* o2, double* m) {
  if (validate(n, x, y, alpha, c)) return -1;
  const int bound = mo_grid_bound(n, alpha);
  const int cells = mo_cell_count(bound);
  double* a = (double*)calloc((size_t)cells, sizeof(double));
  double* b = (double*)calloc((size_t)cells, sizeof(double));
  score_orientation(x, y, n, bound, c, 0, a); /* :78 */
  score_orientation(y, x, n, bound, c, 1, b); /* :79 */
  if (o1) memcpy(o1, a, sizeof(double) * (size_t)cells);
  if (o2) memcpy(o2, b, sizeof(double) * (size_t)cells);
  if (m) /* the two update_max passes on one matrix == max(o1, o2) with ">" */
    for (int i = 0; i < cells; ++i) m[i] = b[i] > a[i] ? b[i] : a[i];
  free(a);
  free(b);
  return bound;
}

/* statistics.cpp:10-37 mic/mas/mev/mcn (+ extensions MIC_e, TIC). */
void mo_reduce(int bound, const double* o1, const double* o2, int est, double* out) {
  const int cells = mo_cell_count(bound);
  double* m = (double*)malloc(sizeof(double) * (size_t)cells);
  double* e = (double*)malloc(sizeof(double) * (size_t)cells);
  int i = 0;
  for (int y = 2; y <= bound / 2; ++y)
    for (int x = 2; x <= bound / y; ++x, ++i) {
      m[i] = o2[i] > o1[i] ? o2[i] : o1[i];
      e[i] = x < y ? o1[i] : (x > y ? o2[i] : m[i]);
    }
  double mic = 0.0, mas = 0.0, mev = 0.0, mice = 0.0, tic = 0.0;
  long best_xy = LONG_MAX;
  i = 0;
  for (int y = 2; y <= bound / 2; ++y)
    for (int x = 2; x <= bound / y; ++x, ++i) {
      mic = dmax(mic, m[i]);                                           /* :10-14 */
      mas = dmax(mas, fabs(m[i] - m[cell_index(bound, y, x)]));       /* :16-20 */
      if (x == 2 || y == 2) mev = dmax(mev, m[i]);                     /* :22-28 */
      mice = dmax(mice, e[i]);
      tic += est ? e[i] : m[i];
    }
  i = 0;
  for (int y = 2; y <= bound / 2; ++y) /* :30-37, exact equality (SPEC eps = 0) */
    for (int x = 2; x <= bound / y; ++x, ++i)
      if (m[i] == mic && (long)x * y < best_xy) best_xy = (long)x * y;
  out[MO_MIC] = mic;
  out[MO_MAS] = mas;
  out[MO_MEV] = mev;
  out[MO_MCN] = log2((double)best_xy);
  out[MO_MICE] = mice;
  out[MO_TIC] = tic;
  free(m);
  free(e);
}

int mo_statistics(int n, const double* x, const double* y, double alpha, double c, int est,
                  double* out) {
  if (validate(n, x, y, alpha, c)) return -1;
  const int bound = mo_grid_bound(n, alpha);
  const int cells = mo_cell_count(bound);
  double* o1 = (double*)malloc(sizeof(double) * (size_t)cells);
  double* o2 = (double*)malloc(sizeof(double) * (size_t)cells);
  mo_compute_score(n, x, y, alpha, c, o1, o2, NULL);
  mo_reduce(bound, o1, o2, est, out);
  free(o1);
  free(o2);
  return 0;
}

int mo_pearson(int n, const double* x, const double* y, double* r) {
  if (n < 2) return fail("pearson: need at least 2 samples");
  double sx = 0.0, sy = 0.0; /* :42-43 xs.mean() = sum() / size() */
  for (int i = 0; i < n; ++i) sx += x[i];
  for (int i = 0; i < n; ++i) sy += y[i];
  const double mx = sx / (double)n, my = sy / (double)n;
  double sxx = 0.0, syy = 0.0, sxy = 0.0; /* :44-45, :47 */
  for (int i = 0; i < n; ++i) sxx += (x[i] - mx) * (x[i] - mx);
  for (int i = 0; i < n; ++i) syy += (y[i] - my) * (y[i] - my);
  if (!(sxx > 0.0) || !(syy > 0.0)) { /* :46 */
    *r = NAN;
    return 0;
  }
  for (int i = 0; i < n; ++i) sxy += (x[i] - mx) * (y[i] - my);
  const double v = sxy / sqrt(sxx * syy);
  *r = v < -1.0 ? -1.0 : (1.0 < v ? 1.0 : v); /* :48 std::clamp */
  return 0;
}

int mo_subproblem(int n, const double* col_var, const double* row_var, int y_target, int x_max,
                  int k_hat, int* row_count, int* q_x, int* clump_count, int* k, int* bounds,
                  double* h_q, double* values) {
  if (n < 2) return fail("equipartition_y_axis: need at least 2 points");
  if (y_target < 2) return fail("equipartition_y_axis: row target must be >= 2");
  if (k_hat < 1) return fail("get_superclumps_partition: clump budget must be >= 1");
  if (x_max < 2) return fail("optimize_x_axis: column target must be >= 2");
  sorted_pairs by_second, by_first;
  sort_pairs(col_var, row_var, n, 1, &by_second);
  sort_pairs(col_var, row_var, n, 0, &by_first);
  subproblem s = {0};
  s.n = n;
  s.y_target = y_target;
  s.x_max = x_max;
  s.k_hat = k_hat;
  s.by_second = &by_second;
  s.by_first = &by_first;
  s.q = (int*)malloc(sizeof(int) * (size_t)n);
  s.qx = q_x;
  s.assign = (int*)malloc(sizeof(int) * (size_t)n);
  s.bounds = bounds;
  s.values = values;
  run_subproblem(&s);
  *row_count = s.row_count;
  *clump_count = s.raw_k;
  *k = s.k;
  *h_q = s.h_q;
  free(s.q);
  free(s.assign);
  free_pairs(&by_second);
  free_pairs(&by_first);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* analysis.cpp:66-81 PairSequence::at (all_pairs), returned 0-based. */
void mo_pair_at(long p, long w, int* i, int* j) {
  const long long total = (long long)p * (p - 1) / 2;
  const long long r = total - (long long)w;
  long long m = (long long)((sqrt(8.0 * (double)r + 1.0) - 1.0) / 2.0);
  while (m * (m + 1) / 2 < r) ++m;
  while (m >= 1 && (m - 1) * m / 2 >= r) --m;
  const long long ii = p - m;
  const long long row_start = total - m * (m + 1) / 2;
  const long long jj = ii + 1 + ((long long)w - row_start);
  *i = (int)ii - 1;
  *j = (int)jj - 1;
}

typedef struct {
  int kind; /* 0 pairwise, 1 cross, 2 list */
  const double *a, *b;
  int p, py, n, est;
  double alpha, c;
  long first, count;
  const int *xi, *yi;
  double* out;
  long next;
  pthread_mutex_t mu;
  int err;
} batch;

static void* batch_worker(void* arg) {
  batch* B = (batch*)arg;
  for (;;) {
    pthread_mutex_lock(&B->mu);
    const long begin = B->next;
    B->next += 16;
    pthread_mutex_unlock(&B->mu);
    if (begin >= B->count) break;
    const long end = begin + 16 < B->count ? begin + 16 : B->count;
    for (long w = begin; w < end; ++w) {
      const double *x, *y;
      if (B->kind == 0) {
        int i, j;
        mo_pair_at(B->p, B->first + w, &i, &j);
        x = B->a + (long)i * B->n;
        y = B->a + (long)j * B->n;
      } else if (B->kind == 1) {
        x = B->a + (w / B->py) * (long)B->n;
        y = B->b + (w % B->py) * (long)B->n;
      } else {
        x = B->a + (long)B->xi[w] * B->n;
        y = B->a + (long)B->yi[w] * B->n;
      }
      if (mo_statistics(B->n, x, y, B->alpha, B->c, B->est, B->out + w * MO_NSTAT)) B->err = 1;
    }
  }
  return NULL;
}

static int run_batch(batch* B, int threads) {
  if (threads < 1) threads = 1;
  pthread_mutex_init(&B->mu, NULL);
  B->next = 0;
  B->err = 0;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, batch_worker, B);
  batch_worker(B);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&B->mu);
  return B->err ? -1 : 0;
}

int mo_pairwise(const double* vars, int p, int n, double alpha, double c, int est, int threads,
                long first, long count, double* out) {
  batch B = {0};
  B.kind = 0;
  B.a = vars;
  B.p = p;
  B.n = n;
  B.alpha = alpha;
  B.c = c;
  B.est = est;
  B.first = first;
  B.count = count;
  B.out = out;
  return run_batch(&B, threads);
}

int mo_cross(const double* X, int px, const double* Y, int py, int n, double alpha, double c,
             int est, int threads, double* out) {
  batch B = {0};
  B.kind = 1;
  B.a = X;
  B.b = Y;
  B.p = px;
  B.py = py;
  B.n = n;
  B.alpha = alpha;
  B.c = c;
  B.est = est;
  B.count = (long)px * py;
  B.out = out;
  return run_batch(&B, threads);
}

int mo_pairs(const double* vars, int n, const int* xi, const int* yi, long npairs, double alpha,
             double c, int est, int threads, double* out) {
  batch B = {0};
  B.kind = 2;
  B.a = vars;
  B.n = n;
  B.xi = xi;
  B.yi = yi;
  B.alpha = alpha;
  B.c = c;
  B.est = est;
  B.count = npairs;
  B.out = out;
  return run_batch(&B, threads);
}
