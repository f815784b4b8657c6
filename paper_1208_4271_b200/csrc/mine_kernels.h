// Device-side data structures and kernel launchers of the B200 MINE engine.
// Host code (engine.cpp) owns all allocations; these launchers only enqueue
// work on the given stream.  See DESIGN.md for the HBM layout.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace mb200 {

// Per-variable precompute of one call (K1 + K2), all device pointers.
// Layout is variable-major: variable v's n-length rows start at v * n.
struct VarSet {
  const double* vals = nullptr;  // V x n input samples (f64)
  int V = 0;                     // number of variables
  int n = 0;                     // samples per variable
  int ny = 0;                    // row targets y = 2 .. ny + 1  (ny = B/2 - 1)
  int* perm = nullptr;           // V x n      sample index at each sorted position
  int* runid = nullptr;          // V x n      tie-run ordinal of each sorted position
  int* runstart = nullptr;       // V x (n+1)  start position of run r; [nruns] = n
  int* nruns = nullptr;          // V
  uint16_t* q = nullptr;         // V x ny x n row label (1-based) of each sample
  int* yhat = nullptr;           // V x ny     realised row count
  double* hq = nullptr;          // V x ny     H(Q), reference-exact (mutual_info.cpp:33)
  uint16_t* qsame = nullptr;     // V x ny     general tier: smallest yi' with Q(yi') == Q(yi) (k_row_same), or null
  uint8_t* lw = nullptr;         // V x n      tiny tier: packed labels (y=2: bits 0-1, y=3: 2-3)
  uint32_t* rsmask = nullptr;    // V          tiny tier: run-start bitmask over sorted positions
  uint4* rec = nullptr;          // V x 6      memo tier: 96-byte per-variable record
  double* dx = nullptr;          // V x n      Pearson: centred samples (statistics.cpp:42-43)
  double* sxx = nullptr;         // V          Pearson: sum of squared deviations
};

// Memo-tier table layout (offsets in doubles), see mine_kernels.cu.
struct MemoLayout {
  // doubles: w2, e2, pln; ints from ib (in doubles): offk, sb, std3;
  // uint16 candidate ranks from hb (in ints): k2r, t3r; total in doubles
  int n, k2cnt, t3cnt, w2, e2, pln, ib, offk, sb, std3, hb, k2r, t3r, total;
  int t3c;  // 3-row table compact (n > 26) or padded dense
};

// Host-built constant tables (glibc libm, the reference's own arithmetic).
struct Tables {
  const double* pl = nullptr;     // p*log(p), p = w/m, at tri(m) + w, 0 <= w <= m <= n
  const double* logi = nullptr;   // log(i), 0 <= i <= B
  const double* log2i = nullptr;  // log2(i), 0 <= i <= B
  const int* cell_off = nullptr;  // offset of row y in for_each order, indexed by y (0..B/2+1)
  const int* cell_tr = nullptr;   // for cell c = (x, y): index of (y, x)
  const int* cell_xy = nullptr;   // x * y of cell c
  const uint8_t* cell_edge = nullptr;  // x == 2 || y == 2
  const int8_t* cell_cmp = nullptr;    // sign(x - y): which orientation feeds MIC_e
  const double* div = nullptr;    // w / m at tri(m) + w (exact IEEE quotients), n <= 4096 only
  // two-row span entropy sums H2(m, w) = pl(m, w) + pl(m, m - w) (the
  // reference's row-ordered sum of a two-row span, mutual_info.hpp:24-27, as
  // one term; symmetric in w <-> m - w, so only w <= m/2 is stored, at
  // h2_off(m) + min(w, m - w)); n <= kH2MaxN only, else null
  const double* h2 = nullptr;
  int n = 0;
  int B = 0;
  int ncell = 0;
  // span terms of three or more rows compute p*log(p) with the device replay
  // of the host libm's log (plog.cuh) instead of gathering table rows
  // c_t - c_s scattered over L2; set only after k_check_plog found every
  // table entry identical
  int span_log = 0;
};

// Which pairs of the variable set to score: work item w in [first, first+count).
enum PairKind : int { kPairwise = 0, kCross = 1, kList = 2 };
struct PairSpace {
  int kind = kPairwise;
  long long first = 0;
  long long count = 0;
  long long p = 0;          // pairwise: variable count
  int px = 0, py = 0;       // cross: X = vars [0, px), Y = vars [px, px + py)
  const int* xi = nullptr;  // list: explicit variable indices
  const int* yi = nullptr;
};

// Statistic outputs, SoA, indexed by (w - first); any pointer may be null.
struct StatsOut {
  double* mic = nullptr;
  double* mas = nullptr;
  double* mev = nullptr;
  double* mcn = nullptr;
  double* mic_e = nullptr;
  double* tic = nullptr;
};

// Realised-work counters: algorithmic FP64 ops of the
// reference arithmetic, p*log(p) lookups, DP candidates, span entries,
// subproblems.
enum { kCntFp64 = 0, kCntLookups, kCntCand, kCntSpans, kCntSub, kCntGathers, kCntRankGathers, kCntPoints, kCntF2, kCntSpanLookups, kNumCounters };
// kCntSpanLookups: the span terms' p*log(p) lookups (spans x rows), random
// rows m = c_t - c_s of the table.
// kCntF2: candidates of the first DP level F(t,2) (mutual_info.cpp:47-56); with
// kCntCand they make SURVEY 8d's C = sum over l = 2 .. l_max.
// kCntGathers / kCntRankGathers: 8-byte / narrow (rank) shared-memory table
// gathers the executing tier actually needs (memo tier: one 2-byte rank per F(t,2)
// candidate, ...); the other counters describe the reference's own
// arithmetic, independent of the tier.

// Parameters of one row target for the general tier.
struct YParams {
  int y, yi, x_max, k_hat;
};

// Optional debug export of one subproblem's integer partition (general tier).
struct SubDebug {
  int* row_count;   // [1]
  int* q_x;         // [n]   row label per x-sorted position
  int* raw_k;       // [1]   clumps before superclumping
  int* k;           // [1]
  int* bounds;      // [n+1]
  double* h_q;      // [1]
  double* values;   // [x_max - 1]  I_l before normalisation
};

// ---- launchers ------------------------------------------------------------
// Must run once per device (under a lock) before any launch.
cudaError_t init_kernel_attributes(int device);
void launch_check_finite(const double* v, long long count, int* flag, cudaStream_t s);
// K1: k_sort_bitonic / k_sort_vars (on chip) up to kRadixSortN samples, the
// chunked bitonic sort k_sort_big through an HBM scratch above (scratch:
// sort_scratch_bytes, 0 below the limit; MINE_B200_RADIX_SORT=1 forces it)
constexpr int kRadixSortN = 16384;
size_t sort_scratch_bytes(int V, int n);
cudaError_t launch_sort_vars(const VarSet& vs, void* scratch, cudaStream_t s);
void launch_equipartition(const VarSet& vs, const Tables& tb, cudaStream_t s);
void launch_pack_tiny(const VarSet& vs, cudaStream_t s);
// general tier: vs.qsame from vs.q / vs.yhat (after launch_equipartition)
void launch_row_same(const VarSet& vs, cudaStream_t s);

// Tiny tier (n <= 32, B <= 7): one thread per pair, stats (and optionally the
// per-orientation cells o1/o2, ncell each per pair) written directly.
void launch_tiny_pairs(const VarSet& vs, const Tables& tb, const PairSpace& ps, double c,
                       int est, StatsOut out, double* o_cells, unsigned long long* counters,
                       cudaStream_t s);

// Memo tier (n <= 25, B <= 7): every F(t,2) candidate precomputed per n.
size_t memo_doubles(int n);
size_t memo_work_bytes(int n);   // build scratch (candidate values, sparse ranks, flags)
size_t memo_values(int n);       // upper bound on distinct candidate values
// nval: distinct candidate values (0 before the build: the pre-check)
bool memo_fits(int n, int B, int nval);
// Builds the table image and the distinct-value table val[]; returns the
// number of distinct candidate values (synchronises the stream once).
int launch_build_memo(const Tables& tb, double* memo, void* work, double* val, int n,
                      cudaStream_t s);
void launch_pack_memo(const VarSet& vs, cudaStream_t s);
// stage: memo_stage_bytes() of scratch (one 8192-pair slot of 6 statistics
// per SM) through which sorted batches write their statistics in index order;
// may be null (direct scattered writes).
size_t memo_stage_bytes();
void launch_memo_pairs(const VarSet& vs, const Tables& tb, const double* memo,
                       const double* memo_val, int nval, const PairSpace& ps, double c, int est,
                       StatsOut out, double* o_cells, unsigned long long* counters,
                       double* stage, cudaStream_t s);

// General tier (mine_general.cu).  One launch GROUP covers many row targets
// y at once: k_part_f2 over every (y, subproblem) of the group (y-major, so
// the heaviest y = 2 blocks start first), then the persistent DP kernels pull
// subproblems y by y in ascending y -- a cost-sorted queue, y = 2 carrying
// ~(B/y)^3 of the work -- from per-y lists the partition kernel filled
// (k <= kSmallK: k_dp_warp, else k_dp).  A call runs one group per chunk of
// pairs unless the scratch of all y's would not fit (c4), then several.
struct GenScratch {  // the device view of one y's scratch (built per item)
  int* desc = nullptr;        // nsub x int4 {k, rows, raw k, l_max}
  int* cb = nullptr;          // nsub x (kc+1) clump boundaries
  int* cum = nullptr;         // nsub x cum_stride cumulative counts, row-major [r][j]
  double* f2 = nullptr;       // nsub x (kc+1) F(t,2)
  long long nsub = 0;
  int kc = 0;                 // min(n, k_hat)
  size_t cum_stride = 0;      // y * (kc+1)
  int small_ok = 0;           // the warp path is available at this y
  unsigned char* pts = nullptr;  // nsub x gen_pts_bytes per-point arrays (large n), or null
  int tables_global = 0;      // cb / cum used in place from this scratch (c B too large)
};
// One row target of a group (host-built, copied to the device).
struct GenY {
  YParams yp;
  int kc, small_ok, tables_global, pad;
  unsigned long long cum_stride;
  int* desc;
  int* cb;
  int* cum;
  double* f2;
  unsigned char* pts;
  long long* small_list;  // [nsub] subproblems with k <= kSmallK (when small_ok)
  long long* big_list;    // [nsub] the others needing levels >= 3
};
struct GenGroup {
  const GenY* ys = nullptr;      // device [ny]
  int ny = 0;
  long long nsub = 0;            // subproblems per y (2 per pair, 1 for one orientation)
  // [gi]: small count, [ny + gi]: big count, [2 ny + gi]: k_dp ticket,
  // [3 ny + gi]: k_dp_warp ticket
  unsigned long long* cnt = nullptr;
};
constexpr int kSmallK = 64;   // subproblems with k <= kSmallK take the warp path
constexpr int kGenSides = 5;  // side streams of a launch group: one per k_dp_warp F-width class
int gen_kc(int n, const YParams& yp);
size_t gen_scratch_per_sub(int n, const YParams& yp);  // incl. list entries
size_t gen_pts_bytes(int n, const YParams& yp);  // 0: the point arrays fit on chip
bool gen_tables_global(int n, const YParams& yp);
size_t gen_pf_smem(int n, const YParams& yp);
size_t gen_dp_smem(int n, const YParams& yp);
size_t gen_fslot_bytes(int n, const YParams& yp);
// Device memory one group needs besides its scratch: the F slots of its DP
// launches (k_dp CTAs keep F in an HBM slot each).
size_t gen_group_fslot_bytes(int n, const YParams* yps, int ny, long long nsub);
// Runs the whole general tier for `yps` over pairs [base, base + npairs) of
// ps: writes both orientations' cells of every y into ocells.  scratch:
// >= nsub * sum gen_scratch_per_sub; d_ys: >= ny GenY; d_cnt: >= 4 ny + 4
// counters; fslots: gen_group_fslot_bytes.  Everything runs on s0 except the
// warp path, whose launches (one per F-width class) run concurrently on
// sides[0 .. kGenSides) (when non-null), forked with ev[0] and joined with
// ev[1 .. kGenSides].  Returns the launch count.
int gen_run_group(const VarSet& vs, const Tables& tb, const PairSpace& ps, long long base,
                  long long npairs, const YParams* yps, int ny, void* scratch, GenY* d_ys,
                  unsigned long long* d_cnt, double* fslots, double* ocells, const SubDebug* dbg,
                  int orient_only, unsigned long long* counters, cudaStream_t s0,
                  const cudaStream_t* sides, cudaEvent_t* ev);
cudaError_t init_general_attributes(int device);
// Device p*log(p) against the host-built table pl (all (n+1)(n+2)/2
// entries): the number of differing entries (synchronises the stream), or -1
// when the build had no libm log data (plog.cuh).
long long check_plog_table(const double* pl, int n, unsigned long long* scratch, cudaStream_t s);
size_t div_table_doubles(int n);
void launch_build_div(double* div, int n, cudaStream_t s);
constexpr int kH2MaxN = 20000;
size_t h2_table_doubles(int n);
void launch_build_h2(const double* pl, double* h2, int n, cudaStream_t s);

void launch_reduce(const Tables& tb, long long npairs, const double* ocells, int est,
                   StatsOut out, long long out_offset, cudaStream_t s);

// Pearson r / non-linearity (pearson.cu, statistics.cpp:39-51).
void launch_center_vars(const VarSet& vs, cudaStream_t s);
// filter_low_variance's per-variable variance (analysis.cpp:98-100), after launch_center_vars
void launch_variances(const VarSet& vs, double* var, cudaStream_t s);
void launch_pearson_pairs(const VarSet& vs, const PairSpace& ps, const double* mic,
                          double* pearson, double* nonlin, cudaStream_t s);

// Results-file records on the device (format.cu, io.cpp:37-47).
size_t format_scratch_bytes(long long count);
cudaError_t format_values_device(const double* v, long long n, char* out, int* len, cudaStream_t s);
cudaError_t launch_format_records(const PairSpace& ps, const double* const stat[6],
                                  const char* names, const long long* name_off, long long count,
                                  void* scratch, char* text, size_t text_cap, size_t* bytes,
                                  int* d_flag, int* h_fallback, cudaStream_t s);

}  // namespace mb200
