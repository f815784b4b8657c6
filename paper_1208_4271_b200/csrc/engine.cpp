// Host runtime of the B200 MINE engine: contexts, host-built constant tables,
// device workspaces, pair batching / streaming, and the C ABI of
// include/mine_b200.h.  All per-pair work runs in the CUDA kernels of
// mine_kernels.cu; this file never scores a pair on the CPU.
//
// Compiled with -ffp-contract=off: the p*log(p) table must round exactly like
// the reference's `acc += p * std::log(p)` (mutual_info.hpp:24-27).
#include <algorithm>
#include <atomic>
#include <climits>
#include <exception>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "mine_b200.h"
#include "mine_kernels.h"

// NVTX ranges per call stage (SURVEY 5 tracing): host-side push/pop around
// the enqueue of each stage, so a timeline tool (nsys) lines the stages up
// with their kernels; free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

using namespace mb200;

namespace {

thread_local std::string g_err;

struct Failure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) throw Failure(std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* ensure(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      const size_t want = std::max<size_t>(bytes, 256);
      CK(cudaMalloc(&p, want));
      cap = want;
    }
    return p;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  ~DevBuf() { release(); }
};

inline unsigned long long tri(unsigned long long m) { return m * (m + 1) / 2; }

int grid_bound(long long n, double alpha) {  // char_matrix.cpp:17-20
  const int b = static_cast<int>(std::floor(std::pow(static_cast<double>(n), alpha)));
  return std::max(b, 4);
}

int cell_count(int B) {
  int c = 0;
  for (int y = 2; y <= B / 2; ++y) c += B / y - 1;
  return c;
}

// Host-built constant tables, cached per (n, B) on a context.
// Off by default: measured slower than the table gathers on every config
// (c3 48.0 -> 61.2 ms, c2 9.0 -> 11.1, c0 3.6 -> 4.6, c4 2.02 -> 2.59 s per
// window; ~35 instructions per computed term against one L2 gather).
// MINE_B200_SPAN_LOG=1 turns it on (still only after k_check_plog passed).
static bool span_log_on() {
  static const bool on = [] {
    const char* e = std::getenv("MINE_B200_SPAN_LOG");
    return e && e[0] == '1';
  }();
  return on;
}

struct TableSet {
  int n = -1, B = -1, ncell = 0;
  DevBuf pl, logi, log2i, cell_off, cell_tr, cell_xy, cell_edge, cell_cmp, div, h2, chk;
  bool has_div = false, has_h2 = false, span_log = false;
  std::vector<int> h_off;

  void build(int n_, int B_, cudaStream_t s) {
    if (n_ == n && B_ == B) return;
    // p*log(p) for p = w/m, 1 <= w <= m <= n -- exactly the reference's term
    // (mutual_info.hpp:24-27), with the same glibc libm.
    const unsigned long long entries = tri((unsigned long long)n_ + 1);
    std::vector<double> h(entries);
    auto fill = [&](int m0, int m1) {
      for (int m = m0; m < m1; ++m) {
        double* row = h.data() + tri(m);
        row[0] = 0.0;
        for (int w = 1; w <= m; ++w) {
          const double p = static_cast<double>(w) / static_cast<double>(m);
          row[w] = p * std::log(p);
        }
      }
    };
    const int nthreads = n_ >= 2048 ? std::max(1u, std::min(16u, std::thread::hardware_concurrency())) : 1;
    if (nthreads == 1) {
      fill(0, n_ + 1);
    } else {
      std::vector<std::thread> th;
      // balance by area: row m costs m
      std::vector<int> cut(nthreads + 1, 0);
      for (int t = 1; t < nthreads; ++t)
        cut[t] = static_cast<int>(std::sqrt(static_cast<double>(t) / nthreads) * (n_ + 1));
      cut[nthreads] = n_ + 1;
      for (int t = 0; t < nthreads; ++t) th.emplace_back(fill, cut[t], cut[t + 1]);
      for (auto& x : th) x.join();
    }
    CK(cudaMemcpyAsync(pl.ensure(entries * sizeof(double)), h.data(), entries * sizeof(double),
                       cudaMemcpyHostToDevice, s));
    std::vector<double> lg(B_ + 1), lg2(B_ + 1);
    for (int i = 0; i <= B_; ++i) {
      lg[i] = i ? std::log(static_cast<double>(i)) : 0.0;
      lg2[i] = i ? std::log2(static_cast<double>(i)) : 0.0;
    }
    // for_each order (char_matrix.hpp:43-47) and the derived cell tables
    h_off.assign(B_ / 2 + 2, 0);
    int c = 0;
    for (int y = 2; y <= B_ / 2; ++y) {
      h_off[y] = c;
      c += B_ / y - 1;
    }
    ncell = c;
    std::vector<int> tr(c), xy(c);
    std::vector<uint8_t> edge(c);
    std::vector<int8_t> cmp(c);
    int i = 0;
    for (int y = 2; y <= B_ / 2; ++y)
      for (int x = 2; x <= B_ / y; ++x, ++i) {
        tr[i] = h_off[x] + (y - 2);
        xy[i] = x * y;
        edge[i] = (x == 2 || y == 2);
        cmp[i] = x < y ? -1 : (x > y ? 1 : 0);
      }
    CK(cudaMemcpyAsync(logi.ensure(lg.size() * 8), lg.data(), lg.size() * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(log2i.ensure(lg2.size() * 8), lg2.data(), lg2.size() * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(cell_off.ensure(h_off.size() * 4), h_off.data(), h_off.size() * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(cell_tr.ensure(std::max(c, 1) * 4), tr.data(), c * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(cell_xy.ensure(std::max(c, 1) * 4), xy.data(), c * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(cell_edge.ensure(std::max(c, 1)), edge.data(), c, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(cell_cmp.ensure(std::max(c, 1)), cmp.data(), c, cudaMemcpyHostToDevice, s));
    // exact c_s / c_t quotients for the general tier's span terms (device-built)
    // Measured slower than IEEE DDIV in the span terms on B200 (the lookups
    // are L2-latency-bound, the FP64 pipe is not busy); kept behind a switch.
    has_div = n_ <= 4096 && std::getenv("MINE_B200_DIV_TABLE");
    if (has_div) {
      launch_build_div(static_cast<double*>(div.ensure(sizeof(double) * div_table_doubles(n_))), n_, s);
      CK(cudaGetLastError());
    }
    // the two-row span table, derived on the device from pl (same sums)
    has_h2 = n_ <= kH2MaxN && !std::getenv("MINE_B200_NO_H2");
    if (has_h2) {
      launch_build_h2(pl.as<double>(), static_cast<double*>(h2.ensure(sizeof(double) * h2_table_doubles(n_))),
                      n_, s);
      CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(s));  // host vectors go out of scope
    // span terms of >= 3 rows may compute p*log(p) on the device (plog.cuh):
    // only if the device replay of this host's libm log reproduces every
    // entry of the table just built (opt-in: MINE_B200_SPAN_LOG=1)
    span_log = false;
    if (span_log_on()) {
      const long long bad = check_plog_table(pl.as<double>(), n_,
                                             static_cast<unsigned long long*>(chk.ensure(8)), s);
      CK(cudaGetLastError());
      span_log = bad == 0;
    }
    n = n_;
    B = B_;
  }

  Tables view() const {
    Tables t;
    t.pl = pl.as<double>();
    t.logi = logi.as<double>();
    t.log2i = log2i.as<double>();
    t.cell_off = cell_off.as<int>();
    t.cell_tr = cell_tr.as<int>();
    t.cell_xy = cell_xy.as<int>();
    t.cell_edge = cell_edge.as<uint8_t>();
    t.cell_cmp = cell_cmp.as<int8_t>();
    t.div = has_div ? div.as<double>() : nullptr;
    t.h2 = has_h2 ? h2.as<double>() : nullptr;
    t.span_log = span_log ? 1 : 0;
    t.n = n;
    t.B = B;
    t.ncell = ncell;
    return t;
  }
};

}  // namespace

struct mine_b200_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;  // compute
  cudaStream_t copy = nullptr;    // result drain
  std::mutex mu;
  TableSet tables;
  DevBuf vals, perm, runid, runstart, nruns, q, yhat, hq, lw, rsmask, qsame;
  DevBuf ocells, stats, flag, idx, counters, memo, memo_vals, memo_val, rec, dx, sxx, micscr, sortscr, mstage;
  // general tier: one launch group per chunk of pairs (or per y-group when
  // the scratch of all y's would not fit): scratch regions, the group's y
  // table and counters, the DP launches' F slots; the DP launches of
  // different kernel variants and the warp path run on extra lanes
  // The y's of a y-group are dealt round-robin to kGenLanes lane groups that
  // run concurrently (one's partitions overlap another's DP); each has a main
  // and a side stream and its own buffers.
  static constexpr int kGenLanes = 8;
  struct GenLane {
    cudaStream_t s = nullptr, side[kGenSides] = {};
    cudaEvent_t ev[2 + kGenSides] = {};  // fork, side joins, lane done
    DevBuf scr, ys, cnt, fslots;
  } glane[kGenLanes];
  int memo_n = -1, memo_nval = 0;
  // per-variable state of the previous call (opts.reuse_vars)
  struct Prep {
    bool valid = false;
    int kind = -1, va = 0, vb = 0, n = 0, B = 0;
    const void* a = nullptr;
    const void* b = nullptr;
    bool dio = false, memo = false, tiny = false, centred = false, qsame = false;
    const double* dvals = nullptr;
  } prep;
  std::vector<cudaEvent_t> events;
  long long launches = 0;
  int sms = 148;
  // Ordering across calls: every call records `last_done` on its stream when
  // its last kernel / copy is enqueued, and the next call (whatever stream it
  // uses) waits on it before touching context-owned buffers.  An async
  // device-io call returns before its finite-input check is read; that
  // result is reported by mine_b200_sync().
  cudaEvent_t last_done = nullptr;
  bool last_recorded = false;
  bool async_pending = false;
  // multi-device calls (opts.ndevices > 1): one engine context per device
  // list entry, created on first use and kept (their tables / buffers are
  // reused by the next sharded call)
  std::vector<mine_b200_ctx*> shards;
};

namespace {

struct Call {
  int kind;                 // PairKind
  const double* a;          // pairwise / list: all variables; cross: X
  const double* b;          // cross: Y
  int va, vb;               // variable counts (cross: px, py; others: p, 0)
  int n;
  const int* xi;
  const int* yi;
  long long total;          // size of the pair space
};

void validate_param(const mine_parameter* par) {  // char_matrix.cpp:11-15
  if (!par) throw Failure("parameters: null");
  if (!(par->alpha > 0.0) || par->alpha > 1.0) throw Failure("parameters: alpha must be in (0, 1]");
  if (!(par->c > 0.0)) throw Failure("parameters: c must be > 0");
  if (par->est != MINE_EST_MIC_APPROX && par->est != MINE_EST_MIC_E)
    throw Failure("parameters: est must be MINE_EST_MIC_APPROX or MINE_EST_MIC_E");
}

// Every call waits for the previous call's work on this context (its stream
// may differ) before reusing the context's device buffers.
void order_after_last_call(mine_b200_ctx* ctx, cudaStream_t s) {
  if (ctx->last_recorded) CK(cudaStreamWaitEvent(s, ctx->last_done, 0));
}

void mark_call_done(mine_b200_ctx* ctx, cudaStream_t s) {
  CK(cudaEventRecord(ctx->last_done, s));
  ctx->last_recorded = true;
}

cudaEvent_t ctx_event(mine_b200_ctx* ctx, size_t i) {
  while (ctx->events.size() <= i) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->events.push_back(e);
  }
  return ctx->events[i];
}

// The memo tier's index-order output staging, MINE_B200_MEMO_STAGE=1 (off
// by default).  Measured on c1 (B200, 10-step bench): with staging the pair
// kernel's DRAM traffic is 157.9 MB per launch (algorithmic 153.5 MB) but the
// launch takes 1.477 ms; without it the sorted batches write their 8-byte
// statistics scattered inside each batch's 64 KB window, L2 fills 58.6 MB of
// partially written sectors from HBM (212.7 MB per launch, HBM at ~2% of its
// peak) and the launch takes 1.425 ms.  The fills cost no time; the staging
// epilogue does (3.6%).
bool memo_stage_on() {
  static const bool on = [] {
    const char* e = std::getenv("MINE_B200_MEMO_STAGE");
    return e && e[0] == '1';
  }();
  return on;
}

// Device memory budget of the general tier's per-chunk scratch
// (MINE_B200_GEN_BUDGET_MB overrides; the F slots come on top).
size_t gen_budget() {
  static const size_t b = [] {
    const char* e = std::getenv("MINE_B200_GEN_BUDGET_MB");
    return e ? (size_t)std::atoll(e) << 20 : (size_t)8 << 30;
  }();
  return b;
}

// Row-map dedup in the general tier (k_row_same / k_part_f2 / k_copy_dups):
// on unless MINE_B200_ROW_DEDUP=0 (the A/B and bit-identity tests)
static bool row_dedup_on() {
  static const bool on = [] {
    const char* e = std::getenv("MINE_B200_ROW_DEDUP");
    return !(e && e[0] == '0');
  }();
  return on;
}

static int gen_lanes() {
  static const int v = [] {
    const char* e = std::getenv("MINE_B200_GEN_LANES");
    const int x = e ? std::atoi(e) : 1;  // measured: 1 group is fastest (c0 / c3)
    return std::max(1, std::min(x, (int)mine_b200_ctx::kGenLanes));
  }();
  return v;
}

// The general tier for the row targets yps[0 .. ny) of pairs [0, npairs) of
// pc: y's dealt round-robin to the lane groups (ascending y within each), each
// group a gen_run_group on its own streams, forked from and joined into s.
int run_gen_group(mine_b200_ctx* ctx, const VarSet& vs, const Tables& tb, const PairSpace& pc,
                  long long npairs, const YParams* yps, int ny, double* ocells, const SubDebug* dbg,
                  int orient_only, unsigned long long* dcnt, cudaStream_t s) {
  NvtxRange nv("general: partitions + DP group");
  const long long nsub = npairs * (orient_only >= 0 ? 1 : 2);
  const int G = std::min(gen_lanes(), ny);
  CK(cudaEventRecord(ctx_event(ctx, 4), s));
  int launches = 0;
  for (int g = 0; g < G; ++g) {
    auto& L = ctx->glane[g];
    if (!L.s) {
      CK(cudaStreamCreateWithFlags(&L.s, cudaStreamNonBlocking));
      for (auto& sd : L.side) CK(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
      for (auto& e : L.ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    std::vector<YParams> mine;
    for (int i = g; i < ny; i += G) mine.push_back(yps[i]);
    size_t scr = 0;
    for (const auto& yp : mine) scr += nsub * (gen_scratch_per_sub(vs.n, yp) + 16 * 8);
    void* scratch = L.scr.ensure(scr);
    GenY* d_ys = static_cast<GenY*>(L.ys.ensure(sizeof(GenY) * mine.size()));
    auto* d_cnt = static_cast<unsigned long long*>(L.cnt.ensure(sizeof(unsigned long long) * (4 * mine.size() + 4)));
    double* fslots = static_cast<double*>(
        L.fslots.ensure(gen_group_fslot_bytes(vs.n, mine.data(), (int)mine.size(), nsub)));
    CK(cudaStreamWaitEvent(L.s, ctx_event(ctx, 4), 0));
    launches += gen_run_group(vs, tb, pc, 0, npairs, mine.data(), (int)mine.size(), scratch, d_ys, d_cnt,
                              fslots, ocells, dbg, orient_only, dcnt, L.s, L.side, L.ev);
    CK(cudaEventRecord(L.ev[1 + kGenSides], L.s));
    CK(cudaStreamWaitEvent(s, L.ev[1 + kGenSides], 0));
  }
  CK(cudaGetLastError());
  return launches;
}

// The per-variable state a successful call leaves on its context.
struct CtxPrepared {
  const Call& call;
  const double* dvals;
  int B;
  bool dio, memo, tiny, centred = false, qsame = false;
  template <typename PrepT>
  void commit(PrepT& P) const {
    P.valid = true;
    P.kind = call.kind;
    P.a = call.a;
    P.b = call.b;
    P.va = call.va;
    P.vb = call.vb;
    P.n = call.n;
    P.B = B;
    P.dio = dio;
    P.memo = memo;
    P.tiny = tiny;
    P.centred = centred;
    P.qsame = qsame;
    P.dvals = dvals;
  }
};

// Runs one batch call.  Everything from the input upload to the statistic
// drain is enqueued on the context streams; host work is limited to tables
// (cached) and launch bookkeeping.
void run_call(mine_b200_ctx* ctx, const Call& call, const mine_parameter* par,
              const mine_b200_opts* opts_in, mine_stats_out* out) {
  NvtxRange nv_call("mine_b200 call");
  validate_param(par);
  mine_b200_opts opts{};
  if (opts_in) opts = *opts_in;
  const int n = call.n;
  if (n < 2) throw Failure("compute_score: need at least 2 samples");
  if (n > 65535) throw Failure("mine_b200: n > 65535 samples is not supported");
  if (!out) throw Failure("mine_b200: null output");
  const long long first = opts.first;
  if (first < 0 || first > call.total) throw Failure("expand_pairs: first index out of range");
  long long count = opts.count > 0 ? opts.count : call.total - first;
  if (first + count > call.total) throw Failure("expand_pairs: pair range out of range");
  ctx->launches = 0;
  if (count == 0) return;

  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = opts.stream ? static_cast<cudaStream_t>(opts.stream) : ctx->stream;
  order_after_last_call(ctx, s);
  ctx->async_pending = false;  // an unsynced async call's check result expires here
  const bool dio = opts.device_io != 0;
  const int B = grid_bound(n, par->alpha);
  const int ny = B / 2 - 1;
  // Tier: 0 auto (memo > tiny > general), 1 tiny, 2 general, 3 memo.
  const bool tiny_ok = n <= 32 && B <= 7;
  const bool memo_pre = memo_fits(n, B, 0);
  if (opts.tier == 1 && !tiny_ok) throw Failure("mine_b200: tiny tier needs n <= 32 and B <= 7");
  if (opts.tier == 3 && !memo_pre) throw Failure("mine_b200: memo tier needs n <= 31 and B <= 7");
  bool memo = memo_pre && (opts.tier == 0 || opts.tier == 3);

  ctx->tables.build(n, B, s);
  const Tables tb = ctx->tables.view();
  if (memo && ctx->memo_n != n) {
    ctx->memo_n = -1;
    double* mt = static_cast<double*>(ctx->memo.ensure(sizeof(double) * memo_doubles(n)));
    void* mw = ctx->memo_vals.ensure(memo_work_bytes(n));
    double* mr = static_cast<double*>(ctx->memo_val.ensure(sizeof(double) * memo_values(n)));
    const int nval = launch_build_memo(tb, mt, mw, mr, n, s);
    CK(cudaGetLastError());
    if (nval <= 0 || nval > 65535) throw Failure("mine_b200: memo table build failed");
    ctx->memo_n = n;
    ctx->memo_nval = nval;
  }
  // the distinct-value table must fit shared memory too (known after the build)
  if (memo && !memo_fits(n, B, ctx->memo_nval)) {
    if (opts.tier == 3) throw Failure("mine_b200: memo tier tables exceed shared memory for this n");
    memo = false;
  }
  const bool tiny = tiny_ok && (opts.tier == 1 || (opts.tier == 0 && !memo));
  const int ncell = tb.ncell;

  // ---- variables -> device
  const int V = call.va + call.vb;
  const size_t vbytes = sizeof(double) * (size_t)V * n;
  auto& P = ctx->prep;
  const bool reuse = opts.reuse_vars != 0;
  if (reuse) {
    if (!P.valid || (P.kind == kCross) != (call.kind == kCross) || P.a != call.a || P.b != call.b ||
        P.va != call.va || P.vb != call.vb || P.n != n || P.B != B || P.dio != dio)
      throw Failure("reuse_vars: the variables differ from the previous call on this context");
  } else {
    P.valid = false;
  }
  const double* dvals;
  if (reuse) {
    dvals = P.dvals;
  } else if (dio && call.kind != kCross) {
    dvals = call.a;
  } else {
    double* d = static_cast<double*>(ctx->vals.ensure(vbytes));
    const cudaMemcpyKind kind = dio ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpyAsync(d, call.a, sizeof(double) * (size_t)call.va * n, kind, s));
    if (call.kind == kCross)
      CK(cudaMemcpyAsync(d + (size_t)call.va * n, call.b, sizeof(double) * (size_t)call.vb * n, kind, s));
    dvals = d;
  }
  int* flag = static_cast<int*>(ctx->flag.ensure(sizeof(int)));
  if (!reuse) {  // a reused set passed this check in the call that prepared it
    CK(cudaMemsetAsync(flag, 0, sizeof(int), s));
    launch_check_finite(dvals, (long long)V * n, flag, s);
    ++ctx->launches;
  }

  VarSet vs;
  vs.vals = dvals;
  vs.V = V;
  vs.n = n;
  vs.ny = ny;
  vs.perm = static_cast<int*>(ctx->perm.ensure(sizeof(int) * (size_t)V * n));
  vs.runid = static_cast<int*>(ctx->runid.ensure(sizeof(int) * (size_t)V * n));
  vs.runstart = static_cast<int*>(ctx->runstart.ensure(sizeof(int) * (size_t)V * (n + 1)));
  vs.nruns = static_cast<int*>(ctx->nruns.ensure(sizeof(int) * (size_t)V));
  vs.q = static_cast<uint16_t*>(ctx->q.ensure(sizeof(uint16_t) * (size_t)V * ny * n));
  vs.yhat = static_cast<int*>(ctx->yhat.ensure(sizeof(int) * (size_t)V * ny));
  vs.hq = static_cast<double*>(ctx->hq.ensure(sizeof(double) * (size_t)V * ny));
  if (!reuse) {
    NvtxRange nv("K1 sort + K2 equipartition");
    CK(launch_sort_vars(vs, ctx->sortscr.ensure(sort_scratch_bytes(V, n)), s));
    launch_equipartition(vs, tb, s);
    ctx->launches += 2;
    P.memo = P.tiny = P.centred = P.qsame = false;
  }
  if (memo) {
    vs.rec = static_cast<uint4*>(ctx->rec.ensure(sizeof(uint4) * 6 * (size_t)V));
    if (!P.memo) {
      launch_pack_memo(vs, s);
      ++ctx->launches;
    }
  } else if (tiny) {
    vs.lw = static_cast<uint8_t*>(ctx->lw.ensure((size_t)V * n));
    vs.rsmask = static_cast<uint32_t*>(ctx->rsmask.ensure(sizeof(uint32_t) * V));
    if (!P.tiny) {
      launch_pack_tiny(vs, s);
      ++ctx->launches;
    }
  } else if (row_dedup_on() && count >= 256) {  // general tier: row-map equality of consecutive y's
    // (a few pairs leave most SMs idle, so skipped subproblems save nothing
    // while the two extra launches cost latency)
    vs.qsame = static_cast<uint16_t*>(ctx->qsame.ensure(sizeof(uint16_t) * (size_t)V * ny));
    if (!P.qsame) {
      launch_row_same(vs, s);
      ++ctx->launches;
    }
  }
  // what this call leaves prepared (committed once the call succeeds)
  CtxPrepared done{call, dvals, B, dio, memo || P.memo, tiny || P.tiny};
  done.qsame = vs.qsame != nullptr || P.qsame;

  // ---- pair space
  PairSpace ps;
  ps.kind = call.kind;
  ps.p = call.va;
  ps.px = call.va;
  ps.py = call.vb;
  if (call.kind == kList) {
    if (dio) {
      ps.xi = call.xi;
      ps.yi = call.yi;
    } else {
      for (long long w = first; w < first + count; ++w)
        if (call.xi[w] < 0 || call.xi[w] >= V || call.yi[w] < 0 || call.yi[w] >= V)
          throw Failure("expand_pairs: pair index out of range");
      int* d = static_cast<int*>(ctx->idx.ensure(sizeof(int) * 2 * (size_t)call.total));
      CK(cudaMemcpyAsync(d, call.xi, sizeof(int) * call.total, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(d + call.total, call.yi, sizeof(int) * call.total, cudaMemcpyHostToDevice, s));
      ps.xi = d;
      ps.yi = d + call.total;
    }
  }

  // ---- outputs: device-resident, or a device staging area drained by the
  // copy stream chunk by chunk while the next chunk computes.
  constexpr int kStats = 8;  // mic mas mev mcn mic_e tic pearson_r nonlinearity
  double* const user_stat[kStats] = {out->mic,   out->mas, out->mev,       out->mcn,
                                     out->mic_e, out->tic, out->pearson_r, out->nonlinearity};
  const bool want_r = out->pearson_r || out->nonlinearity;
  if (want_r) {  // per-variable centring, once per variable set
    vs.dx = static_cast<double*>(ctx->dx.ensure(sizeof(double) * (size_t)V * n));
    vs.sxx = static_cast<double*>(ctx->sxx.ensure(sizeof(double) * (size_t)V));
    if (!(reuse && P.centred)) {
      launch_center_vars(vs, s);
      ++ctx->launches;
    }
  }
  done.centred = want_r || (reuse && P.centred);
  const bool small = tiny || memo;  // one thread per pair, stats written directly
  std::vector<YParams> yps;
  for (int y = 2; y <= B / 2; ++y) {
    YParams yp;
    yp.y = y;
    yp.yi = y - 2;
    yp.x_max = B / y;
    yp.k_hat = std::max(1, static_cast<int>(std::floor(par->c * static_cast<double>(yp.x_max))));
    yps.push_back(yp);
  }
  // General tier plan: every row target of a chunk in one launch group when
  // its scratch fits the budget with at least two pairs per SM; otherwise
  // (c4: B = 1000, 499 row targets) the y's are packed into consecutive
  // groups that each fit, and the chunk is as large as the biggest y allows.
  const size_t budget = gen_budget();
  long long gen_chunk = 0;
  std::vector<std::pair<int, int>> ygroups;  // [first, last) indices into yps
  if (!small) {
    size_t sub_sum = 0, sub_max = 0;
    for (const auto& yp : yps) {
      if (gen_pf_smem(n, yp) > 227 * 1024 || gen_dp_smem(n, yp) > 227 * 1024)
        throw Failure("mine_b200: general tier shared-memory plan exceeds 227 KB for n=" +
                      std::to_string(n) + " y=" + std::to_string(yp.y));
      const size_t b = gen_scratch_per_sub(n, yp) + 16 * 8;  // + the regions' alignment
      sub_sum += b;
      sub_max = std::max(sub_max, b);
    }
    const size_t cell_b = 16 * (size_t)ncell;
    gen_chunk = std::max<long long>(1, std::min<long long>(count, (long long)(budget / (cell_b + 2 * sub_sum))));
    if (gen_chunk < std::min<long long>(count, 2LL * ctx->sms)) {
      gen_chunk = std::max<long long>(1, std::min<long long>(count, (long long)(budget / (cell_b + 2 * sub_max))));
      const size_t room = budget - std::min(budget, cell_b * (size_t)gen_chunk);
      for (int i = 0; i < (int)yps.size();) {
        int j = i;
        size_t acc = 0;
        while (j < (int)yps.size()) {
          const size_t b = 2 * (size_t)gen_chunk * (gen_scratch_per_sub(n, yps[j]) + 16 * 8);
          if (j > i && acc + b > room) break;
          acc += b;
          ++j;
        }
        ygroups.push_back({i, j});
        i = j;
      }
    } else {
      ygroups.push_back({0, (int)yps.size()});
    }
  }
  // host io streams the small tiers in chunks of one 8192-pair sort batch
  // per SM (the memo kernel deals whole batches), so no SM idles per chunk
  const long long chunk = small ? (dio ? count : std::min<long long>(count, 8192LL * ctx->sms))
                               : gen_chunk;
  // Chunk schedule: equal chunks.  (A quarter-size first chunk, to start the
  // PCIe-bound drain earlier, measured 3% slower end to end: the memo kernel
  // deals whole 8192-pair batches, so a small chunk leaves most SMs idle.)
  std::vector<std::pair<long long, long long>> sched;  // (offset, count)
  for (long long c0 = 0; c0 < count; c0 += chunk) sched.push_back({c0, std::min(chunk, count - c0)});
  const long long nchunks = (long long)sched.size();
  const int nslots = dio ? 1 : 2;  // double-buffered staging for host io
  double* stage = nullptr;
  const size_t stage_stats = kStats * (size_t)chunk;
  const size_t stage_cells = out->cells ? 2 * (size_t)ncell * chunk : 0;
  if (!dio) stage = static_cast<double*>(ctx->stats.ensure(sizeof(double) * nslots * (stage_stats + stage_cells)));
  double* ocells = nullptr;
  if (!small) ocells = static_cast<double*>(ctx->ocells.ensure(sizeof(double) * 2 * (size_t)ncell * chunk));

  unsigned long long* dcnt = nullptr;
  if (opts.counters) {
    dcnt = static_cast<unsigned long long*>(ctx->counters.ensure(sizeof(unsigned long long) * kNumCounters));
    CK(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long) * kNumCounters, s));
  }
  if (opts.ev_begin) CK(cudaEventRecord(static_cast<cudaEvent_t>(opts.ev_begin), s));

  for (long long ci = 0; ci < nchunks; ++ci) {
    NvtxRange nv_chunk(memo ? "chunk: memo tier" : tiny ? "chunk: tiny tier" : "chunk: general tier");
    const long long c0 = sched[ci].first;
    const long long cn = sched[ci].second;
    const int slot = (int)(ci % nslots);
    StatsOut so;
    double* so_r = nullptr;   // pearson_r
    double* so_nl = nullptr;  // nonlinearity
    double* cells_dst = nullptr;
    if (dio) {
      so.mic = user_stat[0] ? user_stat[0] + c0 : nullptr;
      so.mas = user_stat[1] ? user_stat[1] + c0 : nullptr;
      so.mev = user_stat[2] ? user_stat[2] + c0 : nullptr;
      so.mcn = user_stat[3] ? user_stat[3] + c0 : nullptr;
      so.mic_e = user_stat[4] ? user_stat[4] + c0 : nullptr;
      so.tic = user_stat[5] ? user_stat[5] + c0 : nullptr;
      so_r = user_stat[6] ? user_stat[6] + c0 : nullptr;
      so_nl = user_stat[7] ? user_stat[7] + c0 : nullptr;
      if (so_nl && !so.mic)  // non-linearity needs MIC even when it is not requested
        so.mic = static_cast<double*>(ctx->micscr.ensure(sizeof(double) * (size_t)chunk));
      cells_dst = out->cells ? out->cells + (size_t)c0 * 2 * ncell : nullptr;
    } else {
      double* base = stage + (size_t)slot * (stage_stats + stage_cells);
      if (ci >= nslots) CK(cudaStreamWaitEvent(s, ctx_event(ctx, 2 * slot + 1), 0));  // slot drained
      double** so_p[kStats] = {&so.mic, &so.mas, &so.mev, &so.mcn, &so.mic_e, &so.tic, &so_r, &so_nl};
      for (int k = 0; k < kStats; ++k) *so_p[k] = user_stat[k] ? base + (size_t)k * chunk : nullptr;
      if (so_nl && !so.mic) so.mic = base;  // MIC for the non-linearity, not drained
      cells_dst = out->cells ? base + stage_stats : nullptr;
    }
    PairSpace pc = ps;
    pc.first = first + c0;
    pc.count = cn;
    if (memo) {
      launch_memo_pairs(vs, tb, ctx->memo.as<double>(), ctx->memo_val.as<double>(), ctx->memo_nval,
                        pc, par->c, par->est, so, cells_dst, dcnt,
                        memo_stage_on() ? static_cast<double*>(ctx->mstage.ensure(memo_stage_bytes()))
                                        : nullptr,
                        s);
      ++ctx->launches;
    } else if (tiny) {
      launch_tiny_pairs(vs, tb, pc, par->c, par->est, so, cells_dst, dcnt, s);
      ++ctx->launches;
    } else {
      // one launch group per y-group (usually all y's): partitions of every
      // (y, subproblem), then the DP kernels pulling subproblems y by y
      for (const auto& gr : ygroups)
        ctx->launches += run_gen_group(ctx, vs, tb, pc, cn, yps.data() + gr.first,
                                       gr.second - gr.first, ocells, nullptr, -1, dcnt, s);
      launch_reduce(tb, cn, ocells, par->est, so, 0, s);
      ++ctx->launches;
      if (cells_dst)
        CK(cudaMemcpyAsync(cells_dst, ocells, sizeof(double) * 2 * ncell * cn, cudaMemcpyDeviceToDevice, s));
    }
    if (want_r) {
      launch_pearson_pairs(vs, pc, so.mic, so_r, so_nl, s);
      ++ctx->launches;
    }
    CK(cudaGetLastError());
    if (!dio) {
      // drain this chunk on the copy stream
      CK(cudaEventRecord(ctx_event(ctx, 2 * slot), s));
      CK(cudaStreamWaitEvent(ctx->copy, ctx_event(ctx, 2 * slot), 0));
      const double* base = stage + (size_t)slot * (stage_stats + stage_cells);
      for (int k = 0; k < kStats; ++k)
        if (user_stat[k])
          CK(cudaMemcpyAsync(user_stat[k] + c0, base + (size_t)k * chunk, sizeof(double) * cn,
                             cudaMemcpyDeviceToHost, ctx->copy));
      if (out->cells)
        CK(cudaMemcpyAsync(out->cells + (size_t)c0 * 2 * ncell, base + stage_stats,
                           sizeof(double) * 2 * ncell * cn, cudaMemcpyDeviceToHost, ctx->copy));
      CK(cudaEventRecord(ctx_event(ctx, 2 * slot + 1), ctx->copy));
    }
  }
  if (opts.ev_end) CK(cudaEventRecord(static_cast<cudaEvent_t>(opts.ev_end), s));
  if (!dio) CK(cudaStreamWaitEvent(s, ctx_event(ctx, 2 * ((nchunks - 1) % nslots) + 1), 0));
  CK(cudaEventRecord(ctx->last_done, s));
  ctx->last_recorded = true;
  if (dio && opts.async && !opts.counters) {
    ctx->async_pending = true;
    done.commit(P);
    return;
  }
  if (!dio) CK(cudaStreamSynchronize(ctx->copy));
  CK(cudaStreamSynchronize(s));
  if (opts.counters)
    CK(cudaMemcpy(opts.counters, dcnt, sizeof(unsigned long long) * kNumCounters, cudaMemcpyDeviceToHost));
  int h_flag = 0;
  CK(cudaMemcpy(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost));
  if (h_flag) throw Failure("compute_score: inputs must be finite");
  done.commit(P);
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

// Multi-device call (opts.ndevices > 1): the GPU analogue of run_analysis's
// worker pool (analysis.cpp:148-190).  One host thread per device-list entry
// drives that entry's engine context; threads claim chunks of items from one
// atomic cursor and score them with run_call (host io), each chunk's results
// written at its offset of the caller's buffers.  A thread's first chunk
// prepares its context's per-variable state, later chunks reuse it.  The first
// failure is rethrown after every thread has joined, like the reference.
void run_sharded(mine_b200_ctx* ctx, const Call& call, const mine_parameter* par,
                 const mine_b200_opts& opts, mine_stats_out* out) {
  if (opts.device_io) throw Failure("mine_b200: multi-device calls take host buffers (device_io = 0)");
  if (opts.counters || opts.ev_begin || opts.ev_end || opts.reuse_vars)
    throw Failure("mine_b200: counters / events / reuse_vars are single-device options");
  if (!opts.devices) throw Failure("mine_b200: ndevices > 1 needs a device list");
  validate_param(par);
  if (call.n < 2) throw Failure("compute_score: need at least 2 samples");
  if (!out) throw Failure("mine_b200: null output");
  const long long first = opts.first;
  if (first < 0 || first > call.total) throw Failure("expand_pairs: first index out of range");
  const long long count = opts.count > 0 ? opts.count : call.total - first;
  if (first + count > call.total) throw Failure("expand_pairs: pair range out of range");
  const int G = opts.ndevices;
  while ((int)ctx->shards.size() < G) ctx->shards.push_back(nullptr);
  for (int g = 0; g < G; ++g) {
    mine_b200_ctx*& sc = ctx->shards[g];
    if (sc && sc->device != opts.devices[g]) {
      mine_b200_destroy(sc);
      sc = nullptr;
    }
    if (!sc) {
      sc = mine_b200_create(opts.devices[g]);
      if (!sc) throw Failure(g_err);
    }
  }
  ctx->launches = 0;
  if (count == 0) return;
  const long long chunk = opts.shard_chunk > 0 ? opts.shard_chunk
                                               : std::max<long long>(1, (count + 16LL * G - 1) / (16LL * G));
  const int ncell = cell_count(grid_bound(call.n, par->alpha));
  std::atomic<long long> cursor{0};
  std::atomic<long long> launches{0};
  std::exception_ptr failure;
  std::mutex failure_mu;
  auto worker = [&](int g) {
    try {
      mine_b200_ctx* sc = ctx->shards[g];
      std::lock_guard<std::mutex> lk(sc->mu);
      bool prepared = false;
      for (;;) {
        const long long c0 = cursor.fetch_add(chunk);
        if (c0 >= count) break;
        const long long cn = std::min(chunk, count - c0);
        mine_b200_opts o{};
        o.first = first + c0;
        o.count = cn;
        o.tier = opts.tier;
        o.reuse_vars = prepared;
        mine_stats_out so = *out;
        double** f[] = {&so.mic, &so.mas, &so.mev, &so.mcn, &so.mic_e, &so.tic, &so.pearson_r,
                        &so.nonlinearity};
        for (double** q : f)
          if (*q) *q += c0;
        if (so.cells) so.cells += (size_t)c0 * 2 * ncell;
        run_call(sc, call, par, &o, &so);
        launches += sc->launches;
        prepared = true;
      }
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> lk(failure_mu);
      if (!failure) failure = std::make_exception_ptr(Failure(e.what()));
    }
  };
  std::vector<std::thread> th;
  for (int g = 0; g < G; ++g) th.emplace_back(worker, g);
  for (auto& t : th) t.join();
  ctx->launches = launches;
  if (failure) std::rethrow_exception(failure);
}

void dispatch(mine_b200_ctx* ctx, const Call& call, const mine_parameter* par,
              const mine_b200_opts* opts, mine_stats_out* out) {
  if (opts && opts->ndevices > 1)
    run_sharded(ctx, call, par, *opts, out);
  else
    run_call(ctx, call, par, opts, out);
}

mine_b200_ctx* default_ctx() {
  thread_local std::unique_ptr<mine_b200_ctx, void (*)(mine_b200_ctx*)> ctx(nullptr, mine_b200_destroy);
  if (!ctx) {
    const char* env = std::getenv("MINE_B200_DEVICE");
    mine_b200_ctx* c = mine_b200_create(env ? std::atoi(env) : 0);
    if (!c) throw Failure(g_err);
    ctx.reset(c);
  }
  return ctx.get();
}

}  // namespace

// ===========================================================================
namespace mb200 {
// for the host front end (records.cpp): the thread-local message the C ABI
// reports through mine_b200_last_error
void set_last_error(const std::string& msg) { g_err = msg; }
int ctx_device(const mine_b200_ctx* ctx) { return ctx->device; }
}  // namespace mb200

extern "C" {

const char* mine_b200_last_error(void) { return g_err.c_str(); }
int mine_b200_version(void) { return MINE_B200_VERSION; }
int mine_b200_grid_bound(long long n, double alpha) { return grid_bound(n, alpha); }
int mine_b200_cell_count(int bound) { return cell_count(bound); }
long long mine_b200_last_launches(mine_b200_ctx* ctx) { return ctx ? ctx->launches : 0; }

int mine_b200_sync(mine_b200_ctx* ctx) {
  return guarded([&] {
    if (!ctx) throw Failure("mine_b200: null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    CK(cudaSetDevice(ctx->device));
    if (ctx->last_recorded) CK(cudaEventSynchronize(ctx->last_done));
    if (ctx->async_pending) {
      ctx->async_pending = false;
      int h_flag = 0;
      CK(cudaMemcpy(&h_flag, ctx->flag.as<int>(), sizeof(int), cudaMemcpyDeviceToHost));
      if (h_flag) throw Failure("compute_score: inputs must be finite");
    }
  });
}

mine_b200_ctx* mine_b200_create(int device) {
  mine_b200_ctx* ctx = nullptr;
  const int rc = guarded([&] {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw Failure("mine_b200: no such CUDA device");
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) throw Failure("mine_b200: needs an sm_100 (Blackwell) GPU");
    CK(cudaSetDevice(device));
    {
      static std::mutex init_mu;
      static std::vector<int> inited;
      std::lock_guard<std::mutex> lk(init_mu);
      if (std::find(inited.begin(), inited.end(), device) == inited.end()) {
        CK(init_kernel_attributes(device));
        CK(init_general_attributes(device));
        inited.push_back(device);
      }
    }
    std::unique_ptr<mine_b200_ctx> c(new mine_b200_ctx());
    c->device = device;
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->last_done, cudaEventDisableTiming));
    c->sms = prop.multiProcessorCount;
    ctx = c.release();
  });
  return rc ? nullptr : ctx;
}

void mine_b200_destroy(mine_b200_ctx* ctx) {
  if (!ctx) return;
  for (auto* sc : ctx->shards) mine_b200_destroy(sc);
  cudaSetDevice(ctx->device);
  for (auto e : ctx->events) cudaEventDestroy(e);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->copy) cudaStreamDestroy(ctx->copy);
  if (ctx->last_done) {
    cudaEventSynchronize(ctx->last_done);
    cudaEventDestroy(ctx->last_done);
  }
  for (auto& L : ctx->glane) {
    if (L.s) cudaStreamDestroy(L.s);
    for (auto sd : L.side)
      if (sd) cudaStreamDestroy(sd);
    for (auto e : L.ev)
      if (e) cudaEventDestroy(e);
  }
  delete ctx;
}

int mine_b200_pairwise(mine_b200_ctx* ctx, const double* vars, int p, int n,
                       const mine_parameter* param, const mine_b200_opts* opts,
                       mine_stats_out* out) {
  return guarded([&] {
    if (!ctx) throw Failure("mine_b200: null context");
    if (p < 0) throw Failure("mine_b200: negative variable count");
    std::lock_guard<std::mutex> lk(ctx->mu);
    Call call{kPairwise, vars, nullptr, p, 0, n, nullptr, nullptr, (long long)p * (p - 1) / 2};
    if (p < 2) call.total = 0;
    dispatch(ctx, call, param, opts, out);
  });
}

int mine_b200_cross(mine_b200_ctx* ctx, const double* X, int px, const double* Y, int py, int n,
                    const mine_parameter* param, const mine_b200_opts* opts,
                    mine_stats_out* out) {
  return guarded([&] {
    if (!ctx) throw Failure("mine_b200: null context");
    if (px < 0 || py < 0) throw Failure("mine_b200: negative variable count");
    std::lock_guard<std::mutex> lk(ctx->mu);
    Call call{kCross, X, Y, px, py, n, nullptr, nullptr, (long long)px * py};
    dispatch(ctx, call, param, opts, out);
  });
}

int mine_b200_pairs(mine_b200_ctx* ctx, const double* vars, int nvars, int n, const int* xi,
                    const int* yi, long long npairs, const mine_parameter* param,
                    const mine_b200_opts* opts, mine_stats_out* out) {
  return guarded([&] {
    if (!ctx) throw Failure("mine_b200: null context");
    if (npairs < 0 || nvars < 0) throw Failure("mine_b200: negative size");
    std::lock_guard<std::mutex> lk(ctx->mu);
    Call call{kList, vars, nullptr, nvars, 0, n, xi, yi, npairs};
    dispatch(ctx, call, param, opts, out);
  });
}

int mine_b200_variances(mine_b200_ctx* ctx, const double* vars, int p, int n, double* var_out) {
  return guarded([&] {
    if (!ctx) throw Failure("mine_b200: null context");
    if (p < 0 || n < 2) throw Failure("mine_b200_variances: need p >= 0 and n >= 2");
    if (p == 0) return;
    std::lock_guard<std::mutex> lk(ctx->mu);
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    order_after_last_call(ctx, s);
    ctx->prep.valid = false;  // the variable buffers are reused below
    VarSet vs;
    vs.V = p;
    vs.n = n;
    double* d = static_cast<double*>(ctx->vals.ensure(sizeof(double) * (size_t)p * n));
    CK(cudaMemcpyAsync(d, vars, sizeof(double) * (size_t)p * n, cudaMemcpyHostToDevice, s));
    vs.vals = d;
    vs.dx = static_cast<double*>(ctx->dx.ensure(sizeof(double) * (size_t)p * n));
    vs.sxx = static_cast<double*>(ctx->sxx.ensure(sizeof(double) * (size_t)p));
    double* var = static_cast<double*>(ctx->micscr.ensure(sizeof(double) * (size_t)p));
    launch_center_vars(vs, s);
    launch_variances(vs, var, s);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(var_out, var, sizeof(double) * (size_t)p, cudaMemcpyDeviceToHost, s));
    mark_call_done(ctx, s);
    CK(cudaStreamSynchronize(s));
  });
}

int mine_b200_debug_subproblem(mine_b200_ctx* ctx, int n, const double* col_var,
                               const double* row_var, int y_target, int x_max, int k_hat,
                               int* row_count, int* q_x, int* raw_k, int* k, int* bounds,
                               double* h_q, double* values) {
  return guarded([&] {
    if (!ctx) throw Failure("mine_b200: null context");
    if (n < 2) throw Failure("equipartition_y_axis: need at least 2 points");
    if (y_target < 2) throw Failure("equipartition_y_axis: row target must be >= 2");
    if (k_hat < 1) throw Failure("get_superclumps_partition: clump budget must be >= 1");
    if (x_max < 2) throw Failure("optimize_x_axis: column target must be >= 2");
    std::lock_guard<std::mutex> lk(ctx->mu);
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    order_after_last_call(ctx, s);
    // the per-variable buffers (vals, perm, runid, q, yhat, hq, ...) are
    // overwritten below: a following reuse_vars call must not trust them
    ctx->prep.valid = false;
    const int B = x_max * y_target;  // admits (x_max, y_target) and rows up to y_target
    ctx->tables.build(n, B, s);
    const Tables tb = ctx->tables.view();
    VarSet vs;
    vs.V = 2;
    vs.n = n;
    vs.ny = B / 2 - 1;
    double* d = static_cast<double*>(ctx->vals.ensure(sizeof(double) * 2 * n));
    CK(cudaMemcpyAsync(d, col_var, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d + n, row_var, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    vs.vals = d;
    vs.perm = static_cast<int*>(ctx->perm.ensure(sizeof(int) * 2 * n));
    vs.runid = static_cast<int*>(ctx->runid.ensure(sizeof(int) * 2 * n));
    vs.runstart = static_cast<int*>(ctx->runstart.ensure(sizeof(int) * 2 * (n + 1)));
    vs.nruns = static_cast<int*>(ctx->nruns.ensure(sizeof(int) * 2));
    vs.q = static_cast<uint16_t*>(ctx->q.ensure(sizeof(uint16_t) * 2 * vs.ny * n));
    vs.yhat = static_cast<int*>(ctx->yhat.ensure(sizeof(int) * 2 * vs.ny));
    vs.hq = static_cast<double*>(ctx->hq.ensure(sizeof(double) * 2 * vs.ny));
    CK(launch_sort_vars(vs, ctx->sortscr.ensure(sort_scratch_bytes(2, n)), s));
    launch_equipartition(vs, tb, s);
    int hidx[2] = {0, 1};
    int* didx = static_cast<int*>(ctx->idx.ensure(sizeof(int) * 2));
    CK(cudaMemcpyAsync(didx, hidx, sizeof(hidx), cudaMemcpyHostToDevice, s));
    PairSpace ps;
    ps.kind = kList;
    ps.first = 0;
    ps.count = 1;
    ps.xi = didx;
    ps.yi = didx + 1;
    YParams yp{y_target, y_target - 2, x_max, k_hat};
    if (gen_pf_smem(n, yp) > 227 * 1024 || gen_dp_smem(n, yp) > 227 * 1024)
      throw Failure("mine_b200: subproblem too large for the general tier");
    // debug outputs in one device block
    const size_t ints = 3 + (size_t)n + (n + 1);
    const size_t bytes = sizeof(double) * (1 + x_max) + sizeof(int) * ints;
    char* dd = static_cast<char*>(ctx->stats.ensure(bytes));
    SubDebug dbg;
    dbg.h_q = reinterpret_cast<double*>(dd);
    dbg.values = dbg.h_q + 1;
    int* ib = reinterpret_cast<int*>(dbg.values + x_max);
    dbg.row_count = ib;
    dbg.raw_k = ib + 1;
    dbg.k = ib + 2;
    dbg.q_x = ib + 3;
    dbg.bounds = ib + 3 + n;
    double* oc = static_cast<double*>(ctx->ocells.ensure(sizeof(double) * 2 * tb.ncell));
    run_gen_group(ctx, vs, tb, ps, 1, &yp, 1, oc, &dbg, 0, nullptr, s);
    std::vector<char> h(bytes);
    CK(cudaMemcpyAsync(h.data(), dd, bytes, cudaMemcpyDeviceToHost, s));
    mark_call_done(ctx, s);
    CK(cudaStreamSynchronize(s));
    const double* hd = reinterpret_cast<const double*>(h.data());
    const int* hi = reinterpret_cast<const int*>(hd + 1 + x_max);
    *h_q = hd[0];
    for (int l = 0; l < x_max - 1; ++l) values[l] = hd[1 + l];
    *row_count = hi[0];
    *raw_k = hi[1];
    *k = hi[2];
    for (int i = 0; i < n; ++i) q_x[i] = hi[3 + i];
    for (int j = 0; j <= hi[2]; ++j) bounds[j] = hi[3 + n + j];
  });
}

// ---- minepy-compatible API -------------------------------------------------
char* mine_check_parameter(mine_parameter* param) {
  static char bad_alpha[] = "alpha must be in (0, 1]";
  static char bad_c[] = "c must be > 0";
  static char bad_est[] = "est must be MINE_EST_MIC_APPROX or MINE_EST_MIC_E";
  if (!param || !(param->alpha > 0.0) || param->alpha > 1.0) return bad_alpha;
  if (!(param->c > 0.0)) return bad_c;
  if (param->est != MINE_EST_MIC_APPROX && param->est != MINE_EST_MIC_E) return bad_est;
  return nullptr;
}

mine_score* mine_compute_score(mine_problem* prob, mine_parameter* param) {
  mine_score* score = nullptr;
  const int rc = guarded([&] {
    if (!prob || !prob->x || !prob->y) throw Failure("compute_score: null problem");
    validate_param(param);
    const int n = prob->n;
    if (n < 2) throw Failure("compute_score: need at least 2 samples");
    const int B = grid_bound(n, param->alpha);
    const int nc = cell_count(B);
    std::vector<double> vars(2 * (size_t)n), cells(2 * (size_t)nc);
    std::memcpy(vars.data(), prob->x, sizeof(double) * n);
    std::memcpy(vars.data() + n, prob->y, sizeof(double) * n);
    int xi = 0, yi = 1;
    mine_stats_out out{};
    double dummy = 0;
    out.mic = &dummy;
    out.cells = cells.data();
    mine_b200_ctx* ctx = default_ctx();
    {
      std::lock_guard<std::mutex> lk(ctx->mu);
      Call call{kList, vars.data(), nullptr, 2, 0, n, &xi, &yi, 1};
      run_call(ctx, call, param, nullptr, &out);
    }
    score = static_cast<mine_score*>(std::calloc(1, sizeof(mine_score)));
    score->n = B / 2 - 1;
    score->B = B;
    score->est = param->est;
    score->m = static_cast<int*>(std::malloc(sizeof(int) * std::max(score->n, 1)));
    double** ma = static_cast<double**>(std::malloc(sizeof(double*) * std::max(score->n, 1)));
    double** me = static_cast<double**>(std::malloc(sizeof(double*) * std::max(score->n, 1)));
    int c = 0;
    for (int i = 0; i < score->n; ++i) {
      const int y = i + 2;
      score->m[i] = B / y - 1;
      ma[i] = static_cast<double*>(std::malloc(sizeof(double) * score->m[i]));
      me[i] = static_cast<double*>(std::malloc(sizeof(double) * score->m[i]));
      for (int j = 0; j < score->m[i]; ++j, ++c) {
        const int x = j + 2;
        const double a = cells[c], b = cells[nc + c];
        const double m = b > a ? b : a;  // update_max of orientation 2 over 1
        ma[i][j] = m;
        me[i][j] = x < y ? a : (x > y ? b : m);
      }
    }
    score->M = param->est == MINE_EST_MIC_E ? me : ma;
    score->M_e = me;
    if (param->est == MINE_EST_MIC_E) {
      for (int i = 0; i < score->n; ++i) std::free(ma[i]);
      std::free(ma);
    }
  });
  return rc ? nullptr : score;
}

void mine_free_score(mine_score** score) {
  if (!score || !*score) return;
  mine_score* s = *score;
  const bool shared = s->M == s->M_e;
  for (int i = 0; i < s->n; ++i) {
    if (!shared) std::free(s->M[i]);
    std::free(s->M_e[i]);
  }
  if (!shared) std::free(s->M);
  std::free(s->M_e);
  std::free(s->m);
  std::free(s);
  *score = nullptr;
}

static double score_max(double** M, const mine_score* s) {
  double best = 0.0;
  for (int i = 0; i < s->n; ++i)
    for (int j = 0; j < s->m[i]; ++j) best = best < M[i][j] ? M[i][j] : best;
  return best;
}

double mine_mic(mine_score* s) { return s ? score_max(s->M, s) : NAN; }
double mine_mic_e(mine_score* s) { return s ? score_max(s->M_e, s) : NAN; }

double mine_mas(mine_score* s) {  // statistics.cpp:16-20
  if (!s) return NAN;
  double best = 0.0;
  for (int i = 0; i < s->n; ++i)
    for (int j = 0; j < s->m[i]; ++j) {
      const int x = j + 2, y = i + 2;  // M(y, x) lives in row x-2, column y-2
      const double d = std::fabs(s->M[i][j] - s->M[x - 2][y - 2]);
      best = best < d ? d : best;
    }
  return best;
}

double mine_mev(mine_score* s) {  // statistics.cpp:22-28
  if (!s) return NAN;
  double best = 0.0;
  for (int i = 0; i < s->n; ++i)
    for (int j = 0; j < s->m[i]; ++j)
      if (i == 0 || j == 0) best = best < s->M[i][j] ? s->M[i][j] : best;
  return best;
}

double mine_mcn(mine_score* s, double eps) {  // statistics.cpp:30-37 (eps = 0)
  if (!s) return NAN;
  const double top = mine_mic(s);
  long best = LONG_MAX;
  for (int i = 0; i < s->n; ++i)
    for (int j = 0; j < s->m[i]; ++j) {
      const bool hit = eps == 0.0 ? s->M[i][j] == top : s->M[i][j] >= (1.0 - eps) * top;
      if (hit) best = std::min(best, static_cast<long>(i + 2) * (j + 2));
    }
  return std::log2(static_cast<double>(best));
}

double mine_mcn_general(mine_score* s) { return s ? mine_mcn(s, 1.0 - mine_mic(s)) : NAN; }

double mine_tic(mine_score* s, int norm) {
  if (!s) return NAN;
  double tic = 0.0;
  long cnt = 0;
  for (int i = 0; i < s->n; ++i)
    for (int j = 0; j < s->m[i]; ++j, ++cnt) tic += s->M[i][j];
  return norm ? tic / static_cast<double>(cnt) : tic;
}

mine_pstats* mine_compute_pstats(mine_matrix* X, mine_parameter* param) {
  mine_pstats* ps = nullptr;
  const int rc = guarded([&] {
    if (!X || !X->data) throw Failure("mine_compute_pstats: null matrix");
    const long long total = X->n >= 2 ? (long long)X->n * (X->n - 1) / 2 : 0;
    std::unique_ptr<mine_pstats, void (*)(mine_pstats*)> r(
        static_cast<mine_pstats*>(std::calloc(1, sizeof(mine_pstats))),
        [](mine_pstats* p) { mine_free_pstats(&p); });
    r->n = total;
    r->mic = static_cast<double*>(std::malloc(sizeof(double) * std::max<long long>(total, 1)));
    r->tic = static_cast<double*>(std::malloc(sizeof(double) * std::max<long long>(total, 1)));
    mine_stats_out out{};
    out.mic = r->mic;
    out.tic = r->tic;
    mine_b200_ctx* ctx = default_ctx();
    std::lock_guard<std::mutex> lk(ctx->mu);
    Call call{kPairwise, X->data, nullptr, X->n, 0, X->m, nullptr, nullptr, total};
    run_call(ctx, call, param, nullptr, &out);
    ps = r.release();
  });
  return rc ? nullptr : ps;
}

mine_cstats* mine_compute_cstats(mine_matrix* X, mine_matrix* Y, mine_parameter* param) {
  mine_cstats* cs = nullptr;
  const int rc = guarded([&] {
    if (!X || !Y || !X->data || !Y->data) throw Failure("mine_compute_cstats: null matrix");
    if (X->m != Y->m) throw Failure("compute_score: input lengths differ");
    const long long total = (long long)X->n * Y->n;
    std::unique_ptr<mine_cstats, void (*)(mine_cstats*)> r(
        static_cast<mine_cstats*>(std::calloc(1, sizeof(mine_cstats))),
        [](mine_cstats* p) { mine_free_cstats(&p); });
    r->n = X->n;
    r->m = Y->n;
    r->mic = static_cast<double*>(std::malloc(sizeof(double) * std::max<long long>(total, 1)));
    r->tic = static_cast<double*>(std::malloc(sizeof(double) * std::max<long long>(total, 1)));
    mine_stats_out out{};
    out.mic = r->mic;
    out.tic = r->tic;
    mine_b200_ctx* ctx = default_ctx();
    std::lock_guard<std::mutex> lk(ctx->mu);
    Call call{kCross, X->data, Y->data, X->n, Y->n, X->m, nullptr, nullptr, total};
    run_call(ctx, call, param, nullptr, &out);
    cs = r.release();
  });
  return rc ? nullptr : cs;
}

void mine_free_pstats(mine_pstats** p) {
  if (!p || !*p) return;
  std::free((*p)->mic);
  std::free((*p)->tic);
  std::free(*p);
  *p = nullptr;
}

void mine_free_cstats(mine_cstats** c) {
  if (!c || !*c) return;
  std::free((*c)->mic);
  std::free((*c)->tic);
  std::free(*c);
  *c = nullptr;
}

}  // extern "C"
