/*
 * mine_b200.h -- C ABI of the B200-native MINE score engine (libmine_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path.
 * The reference (/root/reference/proj) exposes the path as C++ free functions;
 * the paper names the C engine's entry point mine_compute_score() and "three
 * structures", which minepy spells mine_problem /
 * mine_parameter / mine_score.  Each declaration below cites the reference
 * interface it replaces.  Conventions:
 *   - plain pointers and sizes, no C++ or CUDA types;
 *   - no exceptions cross the ABI: functions return 0 / NULL on failure and
 *     mine_b200_last_error() (thread-local) names the condition the reference
 *     would have thrown std::invalid_argument / std::out_of_range for;
 *   - every result is computed on the GPU (sm_100a); there is no CPU fallback,
 *     and a missing / unusable GPU is an error;
 *   - results are bit-identical to the reference for MIC, MAS, MEV, MCN (the
 *     characteristic matrix itself is bit-identical), whatever the batch size,
 *     tier or number of GPUs.
 * Extensions absent from the reference (parity unpinned):
 *   MIC_e (equicharacteristic matrix), TIC, the est switch, cross batches.
 */
#ifndef MINE_B200_H
#define MINE_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MINE_B200_VERSION 100

/* est: which characteristic matrix mine_score.M / TIC refer to. */
#define MINE_EST_MIC_APPROX 0 /* the reference's CharacteristicMatrix (char_matrix.hpp:25-49) */
#define MINE_EST_MIC_E 1      /* extension: equicharacteristic matrix */

/* <-> mine::Parameters {alpha = 0.6, c = 15} (char_matrix.hpp:11-14), plus est. */
typedef struct mine_parameter {
  double alpha;
  double c;
  int est;
} mine_parameter;

/* <-> the (xs, ys) arguments of mine::compute_score (char_matrix.hpp:57). */
typedef struct mine_problem {
  int n;
  double* x;
  double* y;
} mine_problem;

/* <-> mine::CharacteristicMatrix (char_matrix.hpp:25-49): row i holds y = i+2,
 * column j holds x = j+2, m[i] = floor(B/(i+2)) - 1 columns.  Library-owned;
 * release with mine_free_score(). */
typedef struct mine_score {
  int n;         /* rows: B/2 - 1 */
  int* m;        /* columns per row */
  double** M;    /* matrix selected by param.est (MIC_approx: the reference's M) */
  double** M_e;  /* extension: equicharacteristic matrix (always filled) */
  int B;         /* grid bound, char_matrix.cpp:17-20 */
  int est;
} mine_score;

/* Variable-major data matrix: n variables (rows) x m samples, row-major -- the
 * layout of mine::Dataset::values' columns (analysis.hpp:16-22). */
typedef struct mine_matrix {
  double* data;
  int n;
  int m;
} mine_matrix;

/* minepy-style batch results: MIC and TIC per pair. */
typedef struct mine_pstats {
  long long n; /* pairs: p(p-1)/2 in PairSequence order (analysis.cpp:66-81) */
  double* mic;
  double* tic;
} mine_pstats;
typedef struct mine_cstats {
  long long n; /* X variables */
  long long m; /* Y variables; results are n x m row-major */
  double* mic;
  double* tic;
} mine_cstats;

/* Caller-allocated per-pair outputs; any pointer may be NULL.  mic/mas/mev/mcn
 * <-> MineStatistics (statistics.hpp:10-17, Pearson excluded), mic_e / tic are
 * extensions.  cells (optional): 2 * mine_b200_cell_count(B) doubles per pair,
 * the two per-orientation matrices in for_each order (debug / tests). */
typedef struct mine_stats_out {
  double* mic;
  double* mas;
  double* mev;
  double* mcn;
  double* mic_e;
  double* tic;
  double* cells;
  /* statistics.cpp:39-51 (the remaining MineStatistics fields) */
  double* pearson_r;     /* NaN when either variable has zero variance */
  double* nonlinearity;  /* mic - pearson_r^2 */
} mine_stats_out;

/* Engine context: one per host thread (calls on one context are serialised). */
typedef struct mine_b200_ctx mine_b200_ctx;

/* Options for batch calls (zero-initialise for defaults). */
typedef struct mine_b200_opts {
  int device_io;     /* 1: inputs and outputs are device pointers (HBM-resident) */
  int async;         /* 1 (with device_io): enqueue on `stream` and return;
                        mine_b200_sync() reports the finite-input check */
  void* stream;      /* cudaStream_t or NULL for the context's stream */
  int tier;          /* 0 auto, 1 tiny (n<=32, B<=7), 2 general, 3 memo (n<=31, B<=7) */
  long long first;   /* first work item (pairwise/cross/list index) */
  long long count;   /* items to score; <= 0 means all from `first` */
  /* Measurement hooks (bench / profiling), all optional:
   *   counters: host array of MINE_B200_NCOUNTERS realised-work totals
   *             (the reference arithmetic's FP64 ops and p*log(p) lookups, DP
   *             candidates, span entries, subproblems; then the 8-byte and
   *             rank (2-byte) table gathers the executing tier needs; then the
   *             partition's point visits, then the F(t,2) level's candidates
   *             and the span terms' p*log(p) lookups),
   *             accumulated by the kernels;
   *   ev_begin / ev_end: cudaEvent_t recorded on the stream around the
   *             pair-scoring kernels (the dominant kernels of a call). */
  unsigned long long* counters;
  void* ev_begin;
  void* ev_end;
  /* 1: the variables are the SAME as in the previous call on this context
   * (same pointers, shapes, alpha; contents unchanged): skip their upload and
   * the per-variable stages (rank, equipartition, packing -- SURVEY 8f rank 1,
   * e.g. successive windows of one pairwise job, or master_vs_all over many
   * masters against one Y).  A call whose variables differ fails. */
  int reuse_vars;
  /* Multi-GPU (the GPU analogue of run_analysis's worker pool,
   * analysis.cpp:148-190).  ndevices > 1 spreads the call's items over the
   * listed CUDA devices -- an entry may repeat (virtual shards of one GPU) --
   * with one host thread and one engine context (owned by this context) per
   * entry.  The threads claim chunks of `shard_chunk` items (0: automatic,
   * about 16 chunks per entry) from a shared cursor, so expensive and cheap
   * pairs balance dynamically, and each chunk's results land at its offset of
   * the caller's buffers.  Host buffers only (device_io = 0; counters and
   * events are not available).  Results are bit-identical for any list. */
  int ndevices;
  const int* devices;
  long long shard_chunk;
} mine_b200_opts;
#define MINE_B200_NCOUNTERS 10

/* ---- engine API ---------------------------------------------------------- */
const char* mine_b200_last_error(void);
int mine_b200_version(void);
mine_b200_ctx* mine_b200_create(int device);
void mine_b200_destroy(mine_b200_ctx* ctx);
/* Grid bound B(n) = max(floor(n^alpha), 4) (char_matrix.cpp:17-20) and the
 * number of stored shapes for it. */
int mine_b200_grid_bound(long long n, double alpha);
int mine_b200_cell_count(int bound);
/* Kernel launches issued by the last batch call on this context. */
long long mine_b200_last_launches(mine_b200_ctx* ctx);
/* Waits for the context's last call.  After an async device-io call (which
 * returns before its finite-input check is read) it reports that check:
 * -1 with "compute_score: inputs must be finite" as the reference throws
 * (char_matrix.cpp:74-75).  The result is kept until the next call on the
 * context.  Calls on one context are ordered among themselves whatever
 * streams they use. */
int mine_b200_sync(mine_b200_ctx* ctx);

/* All pairs i < j of p variables (vars: p x n, variable-major), results in
 * condensed PairSequence order (analysis.cpp:66-81, run_analysis
 * all_pairs :133-191); item w of [first, first+count) goes to slot w-first. */
int mine_b200_pairwise(mine_b200_ctx* ctx, const double* vars, int p, int n,
                       const mine_parameter* param, const mine_b200_opts* opts,
                       mine_stats_out* out);
/* X (px x n) against Y (py x n), px*py results row-major.  px == 1 is the
 * reference's master_vs_all (analysis.cpp:25-30,82-85). */
int mine_b200_cross(mine_b200_ctx* ctx, const double* X, int px, const double* Y, int py, int n,
                    const mine_parameter* param, const mine_b200_opts* opts,
                    mine_stats_out* out);
/* Explicit pairs (xi[w], yi[w]) of nvars variables (x = column variable of
 * compute_score's first orientation). */
int mine_b200_pairs(mine_b200_ctx* ctx, const double* vars, int nvars, int n, const int* xi,
                    const int* yi, long long npairs, const mine_parameter* param,
                    const mine_b200_opts* opts, mine_stats_out* out);

/* Debug export of one (orientation, row target) subproblem computed by the
 * GPU general tier -- the stage sequence of score_orientation
 * (char_matrix.cpp:44-56): row_count (yhat), q_x[n] (row label per x-sorted
 * position, reindex_to_first_order), raw_k (get_clumps_partition), k and
 * bounds[k+1] (get_superclumps_partition), h_q and values[x_max-1]
 * (optimize_x_axis).  Columns on col_var, rows on row_var. */
int mine_b200_debug_subproblem(mine_b200_ctx* ctx, int n, const double* col_var,
                               const double* row_var, int y_target, int x_max, int k_hat,
                               int* row_count, int* q_x, int* raw_k, int* k, int* bounds,
                               double* h_q, double* values);

/* ---- minepy-compatible API (default context of the calling thread) -------- */
/* NULL if valid, else a static message <-> validate_parameters (char_matrix.cpp:11-15). */
char* mine_check_parameter(mine_parameter* param);
/* <-> mine::compute_score (char_matrix.cpp:70-81). */
mine_score* mine_compute_score(mine_problem* prob, mine_parameter* param);
void mine_free_score(mine_score** score);
/* Reductions of score->M <-> statistics.cpp:10-37 (mcn: eps = 0 is the
 * reference's exact-equality rule, eps > 0 the minepy relaxation). */
double mine_mic(mine_score* score);
double mine_mas(mine_score* score);
double mine_mev(mine_score* score);
double mine_mcn(mine_score* score, double eps);
double mine_mcn_general(mine_score* score);
/* Extensions: TIC = sum of score->M (norm != 0: divided by the cell count);
 * MIC_e = max of score->M_e. */
double mine_tic(mine_score* score, int norm);
double mine_mic_e(mine_score* score);
/* minepy 1.2 batch calls; release with mine_free_pstats / mine_free_cstats. */
mine_pstats* mine_compute_pstats(mine_matrix* X, mine_parameter* param);
mine_cstats* mine_compute_cstats(mine_matrix* X, mine_matrix* Y, mine_parameter* param);
void mine_free_pstats(mine_pstats** p);
void mine_free_cstats(mine_cstats** c);

/* ---- analysis front end (io.cpp, analysis.cpp) ----- */
/* A dataset as read_dataset builds it (io.cpp:48-120): p variables x n
 * samples, variable-major values, labels with duplicates suffixed. */
typedef struct mine_b200_dataset {
  int p;
  int n;
  double* values; /* p x n */
  char** names;   /* p NUL-terminated labels */
} mine_b200_dataset;

/* AnalysisTask (analysis.hpp:27-35). */
typedef struct mine_b200_task {
  int mode;                 /* 0 all_pairs, 1 master_vs_all, 2 single_pair */
  int master, first, second; /* 1-based variable indices */
  double alpha, c;          /* Parameters */
  int has_min_variance;     /* apply filter_low_variance(min_variance) first */
  double min_variance;
  int workers;              /* host threads formatting records (>= 1) */
} mine_b200_task;

/* read_dataset: 0 / -1 (message: mine_b200_last_error, as io.cpp throws). */
int mine_b200_read_dataset(const char* path, mine_b200_dataset** out);
void mine_b200_free_dataset(mine_b200_dataset* ds);
/* Sample variance of each variable on the GPU (analysis.cpp:98-100). */
int mine_b200_variances(mine_b200_ctx* ctx, const double* vars, int p, int n, double* var_out);
/* filter_low_variance (analysis.cpp:92-113): a new dataset of the kept variables. */
int mine_b200_filter_low_variance(mine_b200_ctx* ctx, const mine_b200_dataset* in,
                                  double threshold, mine_b200_dataset** out);
/* run_analysis + write_results (analysis.cpp:133-191, io.cpp:122-154): the
 * header and one format_record line per pair of the task, written through
 * "<out_path>.tmp" renamed into place.  Returns the record count, or -1. */
long long mine_b200_run_analysis(mine_b200_ctx* ctx, const mine_b200_dataset* ds,
                                 const mine_b200_task* task, const char* out_path);
/* Self-test of the exact "%.6g" record formatter against snprintf on `count`
 * generated values: the host formatter (device < 0) or the GPU one; returns
 * the mismatch count (0 expected), -1 on a CUDA error. */
long long mine_b200_check_format(long long count, unsigned long long seed, int device);

#ifdef __cplusplus
}
#endif
#endif /* MINE_B200_H */
