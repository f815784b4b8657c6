/* CPU restatement of the reference MINE engine (TEST INFRASTRUCTURE ONLY).
 *
 * Plain-C, line-for-line restatement of /root/reference/proj/src/{partition,
 * mutual_info,char_matrix,statistics}.cpp + analysis.cpp:66-90, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.  It is
 * never linked into, imported by, or called from the product library.
 *
 * Pinned: bit-exact against the reference itself (oracle/_ref/libmine_ref.so,
 * built from the unmodified reference sources) on the reference's golden
 * vectors and on seeded random pairs -- see tests/test_oracle_pins.py.
 *
 * Extensions (NOT in the reference, parity unpinned):
 *   O1/O2    per-orientation matrices (cells as in char_matrix.cpp:57-64 before
 *            the max-merge), M = max(O1, O2) is the reference matrix;
 *   E        equicharacteristic matrix: E(x,y) = O1(x,y) if x<y, O2(x,y) if
 *            x>y, max of both if x==y (the axis with more bins is the
 *            equipartitioned one, Reshef et al. 2016);
 *   MIC_e    max E;  TIC = sum over cells (for_each order) of M (est=0) or E
 *            (est=1).
 */
#ifndef MINE_ORACLE_H
#define MINE_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Statistic slots written by mo_statistics / batch calls. */
enum { MO_MIC = 0, MO_MAS, MO_MEV, MO_MCN, MO_MICE, MO_TIC, MO_NSTAT };

int mo_grid_bound(long n, double alpha);
/* Number of stored cells for bound B (char_matrix.hpp:43-47). */
int mo_cell_count(int bound);

/* compute_score (char_matrix.cpp:70-81). o1/o2/m may be NULL; each holds
 * mo_cell_count(B) doubles in for_each order.  Returns B, or -1 on an input the
 * reference rejects (message via mo_last_error). */
int mo_compute_score(int n, const double* x, const double* y, double alpha, double c,
                     double* o1, double* o2, double* m);

/* Statistics from the per-orientation matrices: out[MO_NSTAT]. */
void mo_reduce(int bound, const double* o1, const double* o2, int est, double* out);

/* compute_score + mo_reduce; returns 0 / -1. */
int mo_statistics(int n, const double* x, const double* y, double alpha, double c, int est,
                  double* out);

/* One (orientation, row-target) subproblem, the stage sequence of
 * score_orientation (char_matrix.cpp:44-56); outputs as ref_subproblem. */
int mo_subproblem(int n, const double* col_var, const double* row_var, int y_target, int x_max,
                  int k_hat, int* row_count, int* q_x, int* clump_count, int* k, int* bounds,
                  double* h_q, double* values);

/* optimize_x_axis (mutual_info.cpp:26-72) on an explicit rows x k grid. */
int mo_optimize_x_axis(const int* counts_rowmajor, int rows, int k, int x, double* values,
                       double* h_q);

/* Batch drivers (threads >= 1).  Variable-major inputs (variable v at v*n).
 *   pairwise: all i<j in PairSequence order (analysis.cpp:66-81), out[w*MO_NSTAT]
 *   cross:    X (px) x Y (py) row-major, out[(i*py+j)*MO_NSTAT]
 *   pairs:    explicit list (xi[w], yi[w]) of variable indices (0-based)      */
int mo_pairwise(const double* vars, int p, int n, double alpha, double c, int est, int threads,
                long first, long count, double* out);
int mo_cross(const double* X, int px, const double* Y, int py, int n, double alpha, double c,
             int est, int threads, double* out);
int mo_pairs(const double* vars, int n, const int* xi, const int* yi, long npairs, double alpha,
             double c, int est, int threads, double* out);

/* pearson (statistics.cpp:39-49): sequential sums in sample order (the
 * reference's Eigen reductions, as the oracle build's Eigen subset runs them);
 * NaN when either variance is zero.  Returns 0 / -1 (length / n < 2). */
int mo_pearson(int n, const double* x, const double* y, double* r);

/* Condensed index -> (i, j), 0-based, the PairSequence::at arithmetic. */
void mo_pair_at(long p, long w, int* i, int* j);

const char* mo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
