// General tier of the MINE engine (any n, any B): two kernels per row target y.
//
//   k_part_f2  one CTA per (pair, orientation) subproblem: labels in x order,
//              Alg. 1 clumps (partition.cpp:108-146), Alg. 2 superclumps
//              (:148-165), the cumulative cell counts (mutual_info.cpp:9-24)
//              and the whole first DP level F(t,2) (mutual_info.cpp:47-56),
//              which has no sequential dependency: warps over t, lanes over s.
//              Subproblems that need no further level (l_max <= 2) finish here.
//   k_dp       persistent CTAs pulling subproblems from an atomic queue: the
//              levels l >= 3 (mutual_info.cpp:57-66) with the reference's exact
//              F-form arithmetic, tiled over (t-tile x level-tile).  For a tile
//              the candidates from every earlier s (the bulk of the work) are
//              independent of each other: the span terms
//                A(s,t) = c_s/c_t,  W(s,t) = ((c_t - c_s)/c_t) h_span(s,t)
//              are computed once per (s-chunk, t-tile) into shared memory and
//              consumed by register-blocked accumulators for all (t, l) cells;
//              only the s inside the tile is sequential (one step per t).  The F
//              table lives in shared memory when it fits, else in a per-CTA HBM
//              slot (c4: 7.5k x 500 f64 at y = 2).
// Compiled with -fmad=false; every FP64 op rounds like the reference's.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "device_common.cuh"
#include "mine_kernels.h"
#include "plog.cuh"

namespace mb200 {

namespace {

// k_part_f2 runs 256 threads per subproblem when the F(t,2) level is heavy
// (x_max >= 3: every t), 128 when only F(k,2) is needed
#ifndef KDP_THREADS
#define KDP_THREADS 256
#endif
// KDP_PREFETCH: F rows staged by cp.async under the span terms' gathers
// (c4 +47%); KDP_SPAN2: span-term gathers of two rows in flight together
#ifndef KDP_PREFETCH
#define KDP_PREFETCH 1
#endif
#ifndef KDP_SPAN2
#define KDP_SPAN2 1
#endif
#ifndef KDP_WIDE_SHARED_ACC
#define KDP_WIDE_SHARED_ACC 1  // c4 -10.8%: 51 KB per CTA, 3 CTAs per SM at the 58% carveout
#endif
#ifndef KDP_TILE
#define KDP_TILE 32
#endif
constexpr int kDpThreads = KDP_THREADS;
constexpr int kMaxTile = KDP_TILE;  // t-tile / s-chunk edge
#ifndef KDP_SUBTILE
#define KDP_SUBTILE 8
#endif
constexpr int kSubTile = KDP_SUBTILE;  // k_dp inner part: rows per sequential sub-tile
// Levels per thread in k_dp's register tile (2 adjacent t x GL consecutive
// levels): 4 or 8, per variant.  Every operand of the tile comes from shared
// memory by 16-byte loads, which cost 4 wavefronts per warp whatever the
// lanes share, so the loop runs at 16 GL / (4 + GL) candidates per wavefront:
// 16 at GL = 4, 21.3 at GL = 8 (the L1 pipe is k_dp's busiest, ncu).
#ifndef KDP_GL_LEAN
#define KDP_GL_LEAN 4
#endif
#ifndef KDP_GL_WIDE
#define KDP_GL_WIDE 4
#endif
__host__ __device__ constexpr int dp_gl(bool lean) { return lean ? KDP_GL_LEAN : KDP_GL_WIDE; }
// doubles per thread in the accumulator hand-over (odd: no bank conflicts)
__host__ __device__ constexpr int dp_acc_stride(bool lean) { return 2 * dp_gl(lean) + 1; }

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

struct PfLayout {
  size_t lab, fused, cl, cb, pts, cnt, misc, total;
};

// The per-point arrays (labels, fused flags, clump ids, clump bounds: 11n
// bytes) sit in shared memory up to n ~ 19000 (alpha 0.6).  Above that they go
// to a per-subproblem slot in HBM (pts bytes each; kPtsGlobal), and only the
// cumulative table and the scan scratch stay on chip.  When even the
// cumulative table y (kc+1) ints is too big (c B large), it is built in place
// in the subproblem's GenScratch slot (kCumGlobal, which implies kPtsGlobal).
// total: shared bytes.
__host__ __device__ inline PfLayout pf_layout(int n, int y, int kc, bool pts_global,
                                              bool cum_global = false) {
  PfLayout L;
  size_t o = 0;
  L.lab = o;
  o += al16(sizeof(uint16_t) * n);
  L.fused = o;
  o += al16(n);
  L.cl = o;
  o += al16(sizeof(int) * n);
  L.cb = o;
  o += al16(sizeof(int) * (n + 1));
  L.pts = o;
  if (pts_global) o = 0;
  L.cnt = o;
  if (!cum_global) o += al16(sizeof(int) * (size_t)y * (kc + 1));
  L.misc = o;
  o += al16(sizeof(double) * 40);
  L.total = o;
  return L;
}

// The device view of row target Y's scratch.
__device__ __forceinline__ GenScratch scratch_of(const GenY& Y, long long nsub) {
  GenScratch g;
  g.desc = Y.desc;
  g.cb = Y.cb;
  g.cum = Y.cum;
  g.f2 = Y.f2;
  g.nsub = nsub;
  g.kc = Y.kc;
  g.cum_stride = Y.cum_stride;
  g.small_ok = Y.small_ok;
  g.pts = Y.pts;
  g.tables_global = Y.tables_global;
  return g;
}

__device__ __forceinline__ void sub_vars(const PairSpace& ps, long long pl, int orient, int& X,
                                         int& Y) {
  int va, vb;
  pair_vars(ps, ps.first + pl, va, vb);
  X = orient ? vb : va;
  Y = orient ? va : vb;
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Row-map dedup (k_row_same): the group index of the smallest row target
// whose row map equals row target gi's for row variable Yv, or gi itself.
// Only y's of this group count (their descriptors are live).
__device__ __forceinline__ int canonical_gi(const VarSet& vs, const GenGroup& grp, int gi, int Yv) {
  const int yi = grp.ys[gi].yp.yi;
  const int yc = vs.qsame[(size_t)Yv * vs.ny + yi];
  if (yc == yi) return gi;
  const int gc = gi - (yi - yc);  // the group's y's are consecutive
  return gc >= 0 && grp.ys[gc].yp.yi == yc ? gc : gi;
}

// Writes the normalised cells of one orientation / row target (char_matrix.cpp:
// 57-64); I(l) gives the unnormalised I_l.
template <typename IFn>
__device__ void write_cells(const Tables& tb, double* ocells, long long pl, int orient, int y,
                            int x_max, int rows, IFn I, const SubDebug& dbg, bool has_dbg) {
  double* oc = ocells + (size_t)pl * 2 * tb.ncell + (size_t)orient * tb.ncell;
  const double logy = tb.logi[rows];
  for (int l = 2 + threadIdx.x; l <= x_max; l += blockDim.x) {
    const double v = I(l);
    if (has_dbg) dbg.values[l - 2] = v;
    const int cell = orient ? tb.cell_off[l] + (y - 2) : tb.cell_off[y] + (l - 2);
    oc[cell] = norm_cell(v, tb.logi[l], logy);
  }
}

// ---------------------------------------------------------------------------
// Grid: nsub x (the group's y's gi0 .. gi0 + gridDim.x / nsub - 1), y-major.
#ifndef PF_MINB_THREADS
#define PF_MINB_THREADS 1536  // resident threads per SM the register budget is set for (40 regs: -0.6% vs 32)
#endif
template <int kPfThreads, bool kPtsGlobal, bool kCumGlobal>
__global__ void __launch_bounds__(kPfThreads, PF_MINB_THREADS / kPfThreads) k_part_f2(VarSet vs, Tables tb, PairSpace ps,
                                                        long long base, GenGroup grp, int gi0,
                                                        double* __restrict__ ocells, SubDebug dbg,
                                                        int has_dbg, int orient_only,
                                                        unsigned long long* counters) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = vs.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int norient = orient_only >= 0 ? 1 : 2;
  const int gi = gi0 + (int)(blockIdx.x / grp.nsub);
  const long long sub = (long long)(blockIdx.x % grp.nsub);  // index inside this y's scratch
  const GenY& GY = grp.ys[gi];
  const YParams yp = GY.yp;
  const GenScratch gs = scratch_of(GY, grp.nsub);
  const long long pl = base + sub / norient;
  const int orient = orient_only >= 0 ? orient_only : (int)(sub % 2);
  // the pair's variables: one thread inverts the condensed index
  __shared__ int s_xy[2];
  if (tid == 0) sub_vars(ps, pl, orient, s_xy[0], s_xy[1]);
  __syncthreads();
  const int X = s_xy[0], Y = s_xy[1];
  const int y = yp.y, yi = yp.yi, x_max = yp.x_max, k_hat = yp.k_hat, kc = gs.kc;

  const PfLayout L = pf_layout(n, y, kc, kPtsGlobal, kCumGlobal);
  unsigned char* pts = kPtsGlobal ? gs.pts + (size_t)sub * L.pts : smem;
  uint16_t* lab = reinterpret_cast<uint16_t*>(pts + L.lab);
  uint8_t* fused = pts + L.fused;
  int* cl = reinterpret_cast<int*>(pts + L.cl);
  int* cb = reinterpret_cast<int*>(pts + L.cb);
  int* cum = kCumGlobal ? gs.cum + (size_t)sub * gs.cum_stride
                        : reinterpret_cast<int*>(smem + L.cnt);
  int* misc = reinterpret_cast<int*>(smem + L.misc);
  double* dmisc = reinterpret_cast<double*>(smem + L.misc) + 30;  // ints 0..59 are scan / k scratch

  const int* permX = vs.perm + (size_t)X * n;
  const int* ridX = vs.runid + (size_t)X * n;
  const uint16_t* qY = vs.q + ((size_t)Y * vs.ny + yi) * n;
  const int rows = vs.yhat[(size_t)Y * vs.ny + yi];
  const double hq = vs.hq[(size_t)Y * vs.ny + yi];

  // --- row-map dedup: when a smaller y of this group has the same row map
  // (ties saturate the equipartition), the raw clumps are that y's too; if
  // they do not superclump here (raw k <= k_hat <= that y's k_hat) the
  // partition, and so every F(t, l) with l <= min(x_max, k), is that y's, and
  // so are the cells (l, y), l <= x_max (mutual_info.cpp:68-70 repeats I_k
  // beyond k in both).  The canonical subproblem has a lower block index (the
  // grid is y-major) or ran in an earlier launch; its raw k is published in
  // its descriptor (zeroed per group).  The wait is bounded: on a timeout
  // the subproblem is computed here, so the result never depends on it.
  if (vs.qsame && !has_dbg) {
    if (tid == 0) {
      int kr = 0;
      const int gc = canonical_gi(vs, grp, gi, Y);
      if (gc != gi) {
        const int* dz = grp.ys[gc].desc + 4 * sub + 2;
        for (int it = 0; it < 4096 && (kr = ld_relaxed(dz)) == 0; ++it) __nanosleep(128);
        if (kr > 0 && kr <= k_hat) {
          reinterpret_cast<int4*>(gs.desc)[sub] = make_int4(kr, rows, gc, -1);  // l_max -1: copy
          if (counters) {
            unsigned long long w[kNumCounters] = {};
            subproblem_work(rows, kr, x_max, n, w);
            for (int i = 0; i < kNumCounters; ++i)
              if (w[i]) atomicAdd(counters + i, w[i]);
          }
        } else {
          kr = 0;
        }
      }
      misc[0] = kr;
    }
    __syncthreads();
    if (misc[0] != 0) return;
    __syncthreads();  // misc is scan scratch below
  }

  // --- row labels in x order (reindex_to_first_order, partition.cpp:94-106)
  for (int t = tid; t < n; t += kPfThreads) {
    lab[t] = qY[permX[t]];
    fused[t] = 0;
  }
  __syncthreads();
  // --- Alg. 1 (partition.cpp:116-133): an x tie run whose labels change is fused
  for (int t = tid + 1; t < n; t += kPfThreads)
    if (ridX[t] == ridX[t - 1] && lab[t] != lab[t - 1]) fused[ridX[t]] = 1;
  __syncthreads();
  // --- clump starts (:135-144): label change at a run start, or either run fused
  for (int t = tid; t < n; t += kPfThreads) {
    int f = 0;
    if (t > 0) {
      const int a = ridX[t], b = ridX[t - 1];
      f = a != b && (fused[a] || fused[b] || lab[t] != lab[t - 1]);
    }
    cl[t] = f;
  }
  __syncthreads();
  const int kraw = block_incl_scan(cl, n, misc) + 1;  // cl[t]: clump of position t
  if (vs.qsame && tid == 0) {  // for the row-map dedup of larger y's (above)
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(gs.desc + 4 * sub + 2), "r"(kraw) : "memory");
  }
  for (int t = tid + 1; t < n; t += kPfThreads)
    if (cl[t] != cl[t - 1]) cb[cl[t]] = t;
  if (tid == 0) {
    cb[0] = 0;
    cb[kraw] = n;
  }
  __syncthreads();
  // --- Alg. 2 (partition.cpp:148-165): equipartition the clump ordinals.
  // The greedy scan (equipartition_runs, partition.cpp:42-67) closes the
  // current group before clump j iff |in_row + run_j - desired| >=
  // |in_row - desired|.  For a group starting at clump i0, in_row = cb[j] -
  // cb[i0] grows with j, so that test is false ... false, true ... true
  // (also in FP64: the integers are exact and rounding is monotone).  Warp 0
  // therefore tests 32 clumps per step and takes the first true one (ballot):
  // the same group boundaries as the sequential scan, in ~k/32 + groups steps.
  int k = kraw;
  if (kraw > k_hat) {
    if (warp == 0) {
      double desired = (double)n / (double)k_hat;
      int curr = 1, i0 = 0, j = 1;
      while (j < kraw) {
        const int jj = j + lane;
        bool close = false;
        if (jj < kraw) {
          const int in_row = cb[jj] - cb[i0], run = cb[jj + 1] - cb[jj];
          close = fabs((double)(in_row + run) - desired) >= fabs((double)in_row - desired);
        }
        const unsigned m = __ballot_sync(0xffffffffu, close);
        if (m) {
          const int jc = j + __ffs(m) - 1;  // the next group starts at clump jc
          const int i = cb[jc];
          ++curr;
          desired = (double)(n - i) / (double)(k_hat - curr + 1);
          __syncwarp();
          if (lane == 0) cb[curr - 1] = i;  // in place: curr - 1 <= jc, and cb[jc] keeps its value
          __syncwarp();
          i0 = jc;
          j = jc + 1;
        } else {
          j += 32;
        }
      }
      if (lane == 0) {
        cb[curr] = n;
        misc[40] = curr;
      }
    }
    __syncthreads();
    k = misc[40];
    // superclump of every position, by a scan over superclump starts
    for (int t = tid; t < n; t += kPfThreads) cl[t] = 0;
    __syncthreads();
    for (int j = 1 + tid; j < k; j += kPfThreads) cl[cb[j]] = 1;
    __syncthreads();
    block_incl_scan(cl, n, misc);
  }
  // --- cell counts and cumulative table (mutual_info.cpp:9-24): cum[r][j]
  const int kk = k + 1;
  for (int i = tid; i < rows * kk; i += kPfThreads) cum[i] = 0;
  __syncthreads();
  for (int t = tid; t < n; t += kPfThreads) atomicAdd(&cum[(lab[t] - 1) * kk + cl[t] + 1], 1);
  __syncthreads();
  for (int r = warp; r < rows; r += (kPfThreads / 32)) {
    int carry = 0;
    for (int j0 = 1; j0 <= k; j0 += 32) {
      const int j = j0 + lane;
      int v = j <= k ? cum[r * kk + j] : 0;
      v = warp_incl_scan(v) + carry;
      if (j <= k) cum[r * kk + j] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();

  const int l_max = min(x_max, k);
  MB_CHECK(k >= 1 && k <= kc && kraw <= n && rows >= 1 && rows <= y && sub < grp.nsub);
  MB_CHECK(kCumGlobal || L.total <= 227 * 1024);
  if (counters && tid == 0) {
    unsigned long long w[kNumCounters] = {};
    subproblem_work(rows, k, x_max, n, w);
    for (int i = 0; i < kNumCounters; ++i)
      if (w[i]) atomicAdd(counters + i, w[i]);
  }
  if (has_dbg && tid == 0) {
    *dbg.row_count = rows;
    *dbg.raw_k = kraw;
    *dbg.k = k;
    *dbg.h_q = hq;
  }
  if (has_dbg) {
    for (int t = tid; t < n; t += kPfThreads) dbg.q_x[t] = lab[t];
    for (int j = tid; j <= k; j += kPfThreads) dbg.bounds[j] = cb[j];
  }
  // hand the partition to k_dp_warp (k <= kSmallK) or k_dp
  if (l_max >= 3) {
    if (tid == 0) {
      int4 d;
      d.x = k;
      d.y = rows;
      d.z = kraw;
      d.w = l_max;
      reinterpret_cast<int4*>(gs.desc)[sub] = d;
      if (gs.small_ok && k <= kSmallK) {
        const unsigned long long q = atomicAdd(grp.cnt + gi, 1ull);
        MB_CHECK(q < (unsigned long long)grp.nsub);
        GY.small_list[q] = sub;
      } else {
        const unsigned long long q = atomicAdd(grp.cnt + grp.ny + gi, 1ull);
        MB_CHECK(q < (unsigned long long)grp.nsub);
        GY.big_list[q] = sub;
      }
    }
    int* gcb = gs.cb + (size_t)sub * (kc + 1);
    int* gcum = gs.cum + (size_t)sub * gs.cum_stride;
    for (int j = tid; j <= k; j += kPfThreads) gcb[j] = cb[j];
    if (!kCumGlobal)
      for (int i = tid; i < rows * kk; i += kPfThreads) gcum[i] = cum[i];
  } else if (tid == 0) {
    int4 d;
    d.x = k;
    d.y = rows;
    d.z = kraw;
    d.w = l_max;
    reinterpret_cast<int4*>(gs.desc)[sub] = d;
  }

  // --- first DP level F(t,2) = max_s H(P) - H(P,Q) (mutual_info.cpp:47-56):
  // every t is independent; warps over t, lanes over s, all p*log(p) terms
  // from row c_t of the table.
  double* gf2 = gs.f2 + (size_t)sub * (kc + 1);
  // max over s in [1, t) of one t's candidates, by the lanes hl = 0 .. W-1
  // of a W-lane segment (W = 32: a warp; W = 16: a half-warp)
  auto f2_best = [&](int t, int hl, int W) {
    const int ct = cb[t];
    // p*log(p) row c_t as a 32-bit index base: tri(65535) + 65535 < 2^32, so
    // every lookup is one IADD + IMAD.WIDE.U32 (64-bit pointer sums cost four)
    const double* __restrict__ pl = tb.pl;
    const unsigned plt = tri(ct);
    double best = kLowest;
    if (rows == 2) {
      // two rows (y = 2, the heaviest level): all six gathers of a
      // candidate are issued before its adds; unsigned offsets from the
      // row base (one IMAD.WIDE.U32 per address)
      const unsigned uct = ct, ct0 = cum[t], ct1 = cum[kk + t];
      for (int s = 1 + hl; s < t; s += W) {
        const unsigned cs = cb[s], a0 = cum[s], a1 = cum[kk + s];
        // H(P) = entropy of (c_s, c_t - c_s): pl + pl, or one H2 gather
        const double acc2 = tb.h2 ? h2_at(tb.h2, uct, cs)
                                  : __dadd_rn(__ldg(pl + (plt + cs)), __ldg(pl + (plt + (uct - cs))));
        const double j0 = __ldg(pl + (plt + a0)), j1 = __ldg(pl + (plt + a1));
        const double j2 = __ldg(pl + (plt + (ct0 - a0))), j3 = __ldg(pl + (plt + (ct1 - a1)));
        const double accj = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(0.0, j0), j1), j2), j3);
        best = dmax(best, __dsub_rn(-acc2, -accj));
      }
    } else {
      const unsigned uct = ct;
      for (int s = 1 + hl; s < t; s += W) {
        const unsigned cs = cb[s];
        const double acc2 = tb.h2 ? h2_at(tb.h2, uct, cs)
                                  : __dadd_rn(__ldg(pl + (plt + cs)), __ldg(pl + (plt + (uct - cs))));
        double accj = 0.0;
        // columns s and t of cum walked by pointer (stride kk): one IADD per
        // row instead of re-deriving r * kk + s
        const int* cps = cum + s;
        for (int r = 0; r < rows; ++r, cps += kk) accj = __dadd_rn(accj, __ldg(pl + (plt + (unsigned)*cps)));
        const int* cpt = cum + t;
        cps = cum + s;
        for (int r = 0; r < rows; ++r, cps += kk, cpt += kk)
          accj = __dadd_rn(accj, __ldg(pl + (plt + ((unsigned)*cpt - (unsigned)*cps))));
        best = dmax(best, __dsub_rn(-acc2, -accj));
      }
    }
    return best;
  };
  auto f2_store = [&](int t, double best) {
    if (l_max >= 3) gf2[t] = best;
    if (t == k) dmisc[0] = best;
  };
  if (k >= 2) {
    constexpr int nw = kPfThreads / 32;
    const int t_lo = l_max >= 3 ? 2 : k;
    // t <= 17 (at most 16 candidates): two t's per warp, a half-warp each --
    // small-k subproblems (ties, large y) would leave most lanes idle
    const int t_mid = min(k, 17);
    for (int t2 = t_lo + 2 * warp; t2 <= t_mid; t2 += 2 * nw) {
      const int half = lane >> 4, t = t2 + half;
      const bool ok = t <= t_mid;
      double best = ok ? f2_best(t, lane & 15, 16) : kLowest;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) best = dmax(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (ok && (lane & 15) == 0) f2_store(t, best);
    }
    for (int t = max(t_lo, t_mid + 1) + warp; t <= k; t += nw) {
      const double best = warp_max(f2_best(t, lane, 32));
      if (lane == 0) f2_store(t, best);
    }
  }
  __syncthreads();
  if (l_max <= 2) {  // done: I_l = I_2 for every l (mutual_info.cpp:68-70)
    const double i2 = k >= 2 ? dmax(0.0, __dadd_rn(hq, dmisc[0])) : 0.0;
    write_cells(tb, ocells, pl, orient, y, x_max, rows, [&](int) { return i2; }, dbg, has_dbg != 0);
  }
}

// ---------------------------------------------------------------------------
// Warp partition path (n <= kWarpPartMaxN, per-point arrays on chip): the
// same partition, cell counts and F(t,2) level as k_part_f2, but one WARP per
// (y, subproblem) with no block barrier.  A subproblem at n = 500 is ~16
// chunks of 32 x-sorted positions per pass; in a 128-thread CTA its ~10 block
// barriers, block scans and per-CTA setup cost more than the partition
// itself (c2: every pair has 38 such subproblems).  Here the passes run over
// 32-position chunks with ballots:
//   1. labels in x order (partition.cpp:94-106), label changes inside an x
//      tie run mark the run fused (Alg. 1, :116-133) in a bitmask by run;
//   2. clump starts (:135-144) as one ballot word per chunk; the boundaries
//      by popcount prefix;
//   3. superclumps (Alg. 2) by the ballot greedy of k_part_f2, their starts
//      re-marked in the start mask;
//   4. cell counts: clump of a position = popcount prefix of the start mask,
//      shared atomics, then a warp scan per row (mutual_info.cpp:9-24);
//   5. F(t,2) (mutual_info.cpp:47-56), half-warps or the warp per t.
constexpr int kWarpPartMaxN = 1024;
constexpr int kWpWarps = 8;  // warps per CTA

struct WpLayout {
  size_t lab, rid, fm, sm, cb, cum, per_warp;
};
__host__ __device__ inline WpLayout wp_layout(int n, size_t cum_ints) {
  WpLayout L;
  size_t o = 0;
  const size_t nw = (size_t)(n + 31) >> 5;
  L.lab = o;
  o += al16(sizeof(uint16_t) * n);
  L.rid = o;  // x tie-run ordinal per position (< n <= 1024)
  o += al16(sizeof(uint16_t) * n);
  L.fm = o;  // fused runs, by run ordinal
  o += al16(4 * nw);
  L.sm = o;  // (super)clump starts, by position
  o += al16(4 * nw);
  L.cb = o;
  o += al16(sizeof(int) * (n + 1));
  L.cum = o;
  o += al16(sizeof(int) * cum_ints);
  L.per_warp = o;
  return L;
}

__device__ __forceinline__ void part_warp_item(const VarSet& vs, const Tables& tb, const PairSpace& ps,
                                               long long base, const GenGroup& grp, int gi, long long sub,
                                               int per_warp, double* __restrict__ ocells, int orient_only,
                                               unsigned long long* counters, unsigned char* wb) {
  const int lane = threadIdx.x & 31;
  const int n = vs.n, nwd = (n + 31) >> 5;
  const GenY& GY = grp.ys[gi];
  const YParams yp = GY.yp;
  const GenScratch gs = scratch_of(GY, grp.nsub);
  const int norient = orient_only >= 0 ? 1 : 2;
  const long long pl = base + sub / norient;
  const int orient = orient_only >= 0 ? orient_only : (int)(sub % 2);
  int X = 0, Y = 0;
  if (lane == 0) sub_vars(ps, pl, orient, X, Y);
  X = __shfl_sync(0xffffffffu, X, 0);
  Y = __shfl_sync(0xffffffffu, Y, 0);
  const int y = yp.y, yi = yp.yi, x_max = yp.x_max, k_hat = yp.k_hat, kc = gs.kc;
  const int rows = vs.yhat[(size_t)Y * vs.ny + yi];
  const double hq = vs.hq[(size_t)Y * vs.ny + yi];
  const WpLayout L = wp_layout(n, (size_t)y * (kc + 1));
  uint16_t* lab = reinterpret_cast<uint16_t*>(wb + L.lab);
  uint16_t* rid = reinterpret_cast<uint16_t*>(wb + L.rid);
  uint32_t* fm = reinterpret_cast<uint32_t*>(wb + L.fm);
  uint32_t* sm = reinterpret_cast<uint32_t*>(wb + L.sm);
  int* cb = reinterpret_cast<int*>(wb + L.cb);
  int* cum = reinterpret_cast<int*>(wb + L.cum);
  MB_CHECK(L.per_warp <= (size_t)per_warp && n <= kWarpPartMaxN);

  // --- row-map dedup (as in k_part_f2): a smaller y of this group with the
  // same row map whose raw clumps do not superclump here gives the cells
  if (vs.qsame) {
    int kr = 0;
    if (lane == 0) {
      const int gc = canonical_gi(vs, grp, gi, Y);
      if (gc != gi) {
        const int* dz = grp.ys[gc].desc + 4 * sub + 2;
        for (int it = 0; it < 4096 && (kr = ld_relaxed(dz)) == 0; ++it) __nanosleep(128);
        if (kr > 0 && kr <= k_hat) {
          reinterpret_cast<int4*>(gs.desc)[sub] = make_int4(kr, rows, gc, -1);
          if (counters) {
            unsigned long long w[kNumCounters] = {};
            subproblem_work(rows, kr, x_max, n, w);
            for (int i = 0; i < kNumCounters; ++i)
              if (w[i]) atomicAdd(counters + i, w[i]);
          }
        } else {
          kr = 0;
        }
      }
    }
    if (__shfl_sync(0xffffffffu, kr, 0) != 0) return;
  }

  const int* permX = vs.perm + (size_t)X * n;
  const int* ridX = vs.runid + (size_t)X * n;
  const uint16_t* qY = vs.q + ((size_t)Y * vs.ny + yi) * n;
  const unsigned lt = (1u << lane) - 1u;

  // --- pass 0: labels in x order (the dependent gathers of every chunk in
  // flight together) and the x tie-run ordinals, into this warp's slice
  for (int w = lane; w < nwd; w += 32) fm[w] = 0u;
#pragma unroll 4
  for (int t = lane; t < n; t += 32) {
    lab[t] = qY[__ldg(permX + t)];
    rid[t] = (uint16_t)__ldg(ridX + t);
  }
  __syncwarp();
  // --- pass 1: a label change inside an x tie run fuses the run
#pragma unroll 4
  for (int t = 1 + lane; t < n; t += 32) {
    const int rd = rid[t];
    if (rd == rid[t - 1] && lab[t] != lab[t - 1]) atomicOr(fm + (rd >> 5), 1u << (rd & 31));
  }
  __syncwarp();
  // --- pass 2: clump starts (a run start whose run or predecessor run is
  // fused, or whose label changes); boundaries by popcount prefix
  int kraw;
  {
    int cnt = 0;
    for (int t0 = 0, c = 0; t0 < n; t0 += 32, ++c) {
      const int t = t0 + lane;
      bool st = false;
      if (t < n && t > 0) {
        const int rd = rid[t], rd1 = rid[t - 1];
        if (rd != rd1)
          st = ((fm[rd >> 5] >> (rd & 31)) & 1u) || ((fm[rd1 >> 5] >> (rd1 & 31)) & 1u) || lab[t] != lab[t - 1];
      }
      const uint32_t m = __ballot_sync(0xffffffffu, st);
      if (lane == 0) sm[c] = m;
      if (st) cb[cnt + __popc(m & lt) + 1] = t;
      cnt += __popc(m);
    }
    kraw = cnt + 1;
  }
  if (vs.qsame && lane == 0)  // for the row-map dedup of larger y's
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(gs.desc + 4 * sub + 2), "r"(kraw) : "memory");
  if (lane == 0) {
    cb[0] = 0;
    cb[kraw] = n;
  }
  __syncwarp();
  // --- superclumps (Alg. 2, partition.cpp:148-165): the ballot greedy of
  // k_part_f2, then the start mask rebuilt from the group starts
  int k = kraw;
  if (kraw > k_hat) {
    double desired = (double)n / (double)k_hat;
    int curr = 1, i0 = 0, j = 1;
    while (j < kraw) {
      const int jj = j + lane;
      bool close = false;
      if (jj < kraw) {
        const int in_row = cb[jj] - cb[i0], run = cb[jj + 1] - cb[jj];
        close = fabs((double)(in_row + run) - desired) >= fabs((double)in_row - desired);
      }
      const unsigned m = __ballot_sync(0xffffffffu, close);
      if (m) {
        const int jc = j + __ffs(m) - 1;
        const int i = cb[jc];
        ++curr;
        desired = (double)(n - i) / (double)(k_hat - curr + 1);
        __syncwarp();
        if (lane == 0) cb[curr - 1] = i;
        __syncwarp();
        i0 = jc;
        j = jc + 1;
      } else {
        j += 32;
      }
    }
    k = curr;
    __syncwarp();
    if (lane == 0) cb[k] = n;
    for (int w = lane; w < nwd; w += 32) sm[w] = 0u;
    __syncwarp();
    for (int jj = 1 + lane; jj < k; jj += 32) atomicOr(sm + (cb[jj] >> 5), 1u << (cb[jj] & 31));
    __syncwarp();
  }
  // --- cell counts and the cumulative table cum[r][j] (mutual_info.cpp:9-24)
  const int kk = k + 1;
  MB_CHECK(k >= 1 && k <= kc && rows >= 1 && rows <= y && (size_t)rows * kk <= (size_t)y * (kc + 1));
  for (int i = lane; i < rows * kk; i += 32) cum[i] = 0;
  __syncwarp();
  {
    int cl0 = 0;  // starts before this chunk
    for (int t0 = 0, c = 0; t0 < n; t0 += 32, ++c) {
      const int t = t0 + lane;
      const uint32_t m = sm[c];
      if (t < n) atomicAdd(cum + (lab[t] - 1) * kk + cl0 + __popc(m & (lt | (1u << lane))) + 1, 1);
      cl0 += __popc(m);
    }
  }
  __syncwarp();
  for (int r = 0; r < rows; ++r) {
    int carry = 0;
    for (int j0 = 1; j0 <= k; j0 += 32) {
      const int j = j0 + lane;
      int v = j <= k ? cum[r * kk + j] : 0;
      v = warp_incl_scan(v) + carry;
      if (j <= k) cum[r * kk + j] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncwarp();

  const int l_max = min(x_max, k);
  if (counters && lane == 0) {
    unsigned long long w[kNumCounters] = {};
    subproblem_work(rows, k, x_max, n, w);
    for (int i = 0; i < kNumCounters; ++i)
      if (w[i]) atomicAdd(counters + i, w[i]);
  }
  // hand the partition to k_dp_warp (k <= kSmallK) or k_dp
  if (lane == 0) {
    reinterpret_cast<int4*>(gs.desc)[sub] = make_int4(k, rows, kraw, l_max);
    if (l_max >= 3) {
      if (gs.small_ok && k <= kSmallK) {
        const unsigned long long q = atomicAdd(grp.cnt + gi, 1ull);
        MB_CHECK(q < (unsigned long long)grp.nsub);
        GY.small_list[q] = sub;
      } else {
        const unsigned long long q = atomicAdd(grp.cnt + grp.ny + gi, 1ull);
        MB_CHECK(q < (unsigned long long)grp.nsub);
        GY.big_list[q] = sub;
      }
    }
  }
  if (l_max >= 3) {
    int* gcb = gs.cb + (size_t)sub * (kc + 1);
    int* gcum = gs.cum + (size_t)sub * gs.cum_stride;
    for (int j = lane; j <= k; j += 32) gcb[j] = cb[j];
    for (int i = lane; i < rows * kk; i += 32) gcum[i] = cum[i];
  }
  // --- F(t,2) = max_s H(P) - H(P,Q) (mutual_info.cpp:47-56): half-warps per
  // t up to 16 candidates, then the warp per t; the p*log(p) terms from row
  // c_t of the table, in the reference's order
  double* gf2 = gs.f2 + (size_t)sub * (kc + 1);
  auto f2_best = [&](int t, int hl, int W) {
    const int ct = cb[t];
    // p*log(p) row c_t as a 32-bit index base: tri(65535) + 65535 < 2^32, so
    // every lookup is one IADD + IMAD.WIDE.U32 (64-bit pointer sums cost four)
    const double* __restrict__ pl = tb.pl;
    const unsigned plt = tri(ct);
    double best = kLowest;
    if (rows == 2) {
      const unsigned uct = ct, ct0 = cum[t], ct1 = cum[kk + t];
      for (int s = 1 + hl; s < t; s += W) {
        const unsigned cs = cb[s], a0 = cum[s], a1 = cum[kk + s];
        const double acc2 = tb.h2 ? h2_at(tb.h2, uct, cs)
                                  : __dadd_rn(__ldg(pl + (plt + cs)), __ldg(pl + (plt + (uct - cs))));
        const double j0 = __ldg(pl + (plt + a0)), j1 = __ldg(pl + (plt + a1));
        const double j2 = __ldg(pl + (plt + (ct0 - a0))), j3 = __ldg(pl + (plt + (ct1 - a1)));
        const double accj = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(0.0, j0), j1), j2), j3);
        best = dmax(best, __dsub_rn(-acc2, -accj));
      }
    } else {
      const unsigned uct = ct;
      for (int s = 1 + hl; s < t; s += W) {
        const unsigned cs = cb[s];
        const double acc2 = tb.h2 ? h2_at(tb.h2, uct, cs)
                                  : __dadd_rn(__ldg(pl + (plt + cs)), __ldg(pl + (plt + (uct - cs))));
        double accj = 0.0;
        // columns s and t of cum walked by pointer (stride kk): one IADD per
        // row instead of re-deriving r * kk + s
        const int* cps = cum + s;
        for (int r = 0; r < rows; ++r, cps += kk) accj = __dadd_rn(accj, __ldg(pl + (plt + (unsigned)*cps)));
        const int* cpt = cum + t;
        cps = cum + s;
        for (int r = 0; r < rows; ++r, cps += kk, cpt += kk)
          accj = __dadd_rn(accj, __ldg(pl + (plt + ((unsigned)*cpt - (unsigned)*cps))));
        best = dmax(best, __dsub_rn(-acc2, -accj));
      }
    }
    return best;
  };
  double f2k = 0.0;  // F(k, 2), held by the lanes that computed it
  bool has_k = false;
  if (k >= 2) {
    const int t_lo = l_max >= 3 ? 2 : k;
    const int t_mid = min(k, 17);
    for (int t2 = t_lo; t2 <= t_mid; t2 += 2) {
      const int half = lane >> 4, t = t2 + half;
      const bool ok = t <= t_mid;
      double best = ok ? f2_best(t, lane & 15, 16) : kLowest;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) best = dmax(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (ok && (lane & 15) == 0 && l_max >= 3) gf2[t] = best;
      if (ok && t == k) {
        f2k = best;
        has_k = true;
      }
    }
    for (int t = max(t_lo, t_mid + 1); t <= k; ++t) {
      const double best = warp_max(f2_best(t, lane, 32));
      if (lane == 0 && l_max >= 3) gf2[t] = best;
      if (t == k) {
        f2k = best;
        has_k = true;
      }
    }
  }
  {
    const unsigned hm = __ballot_sync(0xffffffffu, has_k);
    if (hm) f2k = __shfl_sync(0xffffffffu, f2k, __ffs(hm) - 1);
  }
  if (l_max <= 2) {  // done: I_l = I_2 for every l (mutual_info.cpp:68-70)
    const double i2 = k >= 2 ? dmax(0.0, __dadd_rn(hq, f2k)) : 0.0;
    double* oc = ocells + (size_t)pl * 2 * tb.ncell + (size_t)orient * tb.ncell;
    const double logy = tb.logi[rows];
    for (int l = 2 + lane; l <= x_max; l += 32) {
      const int cell = orient ? tb.cell_off[l] + (y - 2) : tb.cell_off[y] + (l - 2);
      oc[cell] = norm_cell(i2, tb.logi[l], logy);
    }
  }
}

#ifndef WP_MIN_BLOCKS
#define WP_MIN_BLOCKS 4  // 64 registers: 4 CTAs of 8 warps per SM (c2 -2% against 79 registers)
#endif
__global__ void __launch_bounds__(kWpWarps * 32, WP_MIN_BLOCKS) k_part_warp(VarSet vs, Tables tb, PairSpace ps,
                                                            long long base, GenGroup grp, int gi0,
                                                            int gcount, int per_warp,
                                                            double* __restrict__ ocells,
                                                            int orient_only,
                                                            unsigned long long* counters) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // persistent warps: items in y-major order from a ticket (grp.cnt[4 ny]),
  // so a smaller y's subproblem is always taken before (the dedup wait)
  for (;;) {
    long long wg = 0;
    if (lane == 0) wg = (long long)atomicAdd(grp.cnt + 4 * grp.ny, 1ull);
    wg = __shfl_sync(0xffffffffu, wg, 0);
    if (wg >= grp.nsub * gcount) return;
    part_warp_item(vs, tb, ps, base, grp, gi0 + (int)(wg / grp.nsub), wg % grp.nsub, per_warp, ocells,
                   orient_only, counters, smem + (size_t)wib * per_warp);
  }
}

// ---------------------------------------------------------------------------
constexpr int kFRing = 128;  // F row ring width above 128 levels (power of two >= 65)
__host__ __device__ inline int fring_width(int LW) { return LW > kFRing ? kFRing : LW; }
// Rows 0 .. kc of F, then the row fk of F(k, .) that the ring variants keep
// (always reserved: the global-table variant runs the ring code at any width).
__host__ __device__ inline size_t fslot_doubles(int kc, int LW) {
  return (size_t)(kc + 1) * fring_width(LW) + LW;
}

struct DpLayout {
  size_t cb, cum, A, W, acc, fs, ft, total;
  int fsw, ftw;  // staged / tile F row widths (doubles)
};

// Staged F rows (levels l0-1 .. l1-1) are GL ngc doubles wide, ngc = the
// level groups (GL levels each, dp_gl) of the widest level tile (nlc =
// min(64, x_max - 2) levels).  Level offset j = GL g + i (g: the consumer's
// group) sits at (i / 2) fo + 2 g + (i & 1), fo = 2 ng (ng: this tile's
// groups; 64 / GL in the 64-wide rows of the wide variants), so the 16-byte
// loads of consecutive groups are contiguous (no bank conflicts).
template <int GL>
__host__ __device__ inline int fs_col(int j, int fo) {  // fo: offset between level pairs (2 ng)
  const int g = j / GL, i = j % GL;
  return (i >> 1) * fo + 2 * g + (i & 1);
}
#ifndef KDP_LEAN_XMAX
#define KDP_LEAN_XMAX 64
#endif
constexpr int kLeanXMax = KDP_LEAN_XMAX;
#ifndef DP_COMPACT
#define DP_COMPACT 1
#endif
__host__ __device__ inline int dp_nlc(int x_max) { return !DP_COMPACT || x_max - 2 >= 64 ? 64 : x_max - 2; }
__host__ __device__ inline int dp_ngc(int x_max, int gl) { return (dp_nlc(x_max) + gl - 1) / gl; }

// kGlobalTables: cb and cum are read in place from the subproblem's
// GenScratch slot instead of being staged (for c B too large for the chip).
// The staged F rows (fs) and the accumulator hand-over (acc, the owners'
// cells only) share one region: acc is written after a tile's last chunk and
// read by its inner part, fs only by the chunks.
__host__ __device__ inline DpLayout dp_layout(int y, int kc, int x_max, bool global_tables,
                                              bool lean) {
  DpLayout L;
  size_t o = 0;
  L.cb = o;
  if (!global_tables) o += al16(sizeof(int) * (kc + 1));
  L.cum = o;
  if (!global_tables) o += al16(sizeof(int) * (size_t)y * (kc + 1));
  L.A = o;
  o += al16(sizeof(double) * kMaxTile * kMaxTile);
  L.W = o;  // = L.A + kMaxTile^2 doubles (the accumulation loop relies on it)
  o += al16(sizeof(double) * kMaxTile * kMaxTile);
  // compact widths for the lean variant only (gen_dp_lean); the others use
  // 64 / 65
  const int gl = dp_gl(lean), kAccStride = dp_acc_stride(lean);
  const int ngc = lean ? dp_ngc(x_max, gl) : 64 / gl;
  L.fsw = gl * ngc;
  L.ftw = lean ? dp_nlc(x_max) + 1 : 65;
  const size_t acc_b = sizeof(double) * (size_t)(kMaxTile / 2) * ngc * kAccStride;
  const size_t fs_b = sizeof(double) * (size_t)kMaxTile * L.fsw;
  L.acc = o;
  if (!lean && !KDP_WIDE_SHARED_ACC) {  // wide variants: separate regions, as sized before the lean variant
    o += al16(acc_b);
    L.fs = o;
    o += al16(fs_b);
  } else if (!lean) {  // wide, shared: the hand-over (inner part) and the staged rows (chunks) alternate
    L.fs = o;
    o += al16(acc_b > fs_b ? acc_b : fs_b);
  } else {
    L.fs = o;
    o += al16(acc_b > fs_b ? acc_b : fs_b);
  }
  L.ft = o;
  o += al16(sizeof(double) * (size_t)kMaxTile * L.ftw);
  L.total = o;
  return L;
}

// Span terms for s in [s0, s0+ns) x t in [t0, t0+nt) (mutual_info.cpp:39-41,
// 62): A = c_s/c_t, W = ((c_t - c_s)/c_t) h_span(s,t), h by the reference's
// sequential row sum.  The two quotients come from the exact c_s/c_t table
// when it exists (same IEEE quotient, no DDIV).  Entries with s >= t or t > k
// are left undefined.
__device__ __forceinline__ void span_terms(const Tables& tb, const int* cb, const int* cum, int kk,
                                           int rows, int k, int s0, int ns, int t0, int nt,
                                           double* A, double* W) {
  // k_dp's block size is a compile-time constant: no blockDim reads (the
  // compiler rematerialises the index math under k_dp's register budget)
  constexpr int nw = kDpThreads >> 5;
  const int lane = threadIdx.x & 31;
  // a lane keeps one t (nt <= 32): c_t and its reciprocal once per call
  const int tl = lane, t = t0 + tl;
  if (tl >= nt || t > k) return;
  const int ct = cb[t];
  const double dct = (double)ct, rct = __drcp_rn(dct);
  // four rows s per pass with interleaved row sums: their L2 gathers of the
  // p*log(p) table are in flight together (each sum keeps the reference's
  // row order)
  const int w0 = threadIdx.x >> 5;
  for (int base = 0; base < ns; base += 4 * nw) {
    int cs[4];
    unsigned plm[4];  // 32-bit row bases (one IMAD.WIDE.U32 per lookup)
    const double* __restrict__ pl = tb.pl;
    bool ok[4];
    double acch[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int sl = base + w0 + e * nw, s = s0 + sl;
      ok[e] = sl < ns && s < t;
      cs[e] = ok[e] ? cb[s] : ct;
      plm[e] = tri(ct - cs[e]);
      acch[e] = 0.0;
    }
    int r = 0;
    if (rows == 2 && tb.h2) {
      // two rows: the span's sum pl(m, w0) + pl(m, m - w0) is one H2 gather
      const unsigned ct0 = cum[t];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int s = s0 + base + w0 + e * nw;
        acch[e] = ok[e] ? h2_at(tb.h2, (unsigned)(ct - cs[e]), ct0 - (unsigned)cum[s]) : 0.0;
      }
      r = rows;
    }
#if MB_HAVE_LOGDATA
    if (r < rows && tb.span_log) {
      // three or more rows: p*log(p) computed (plog.cuh), no table gathers;
      // each entry's sum still runs in row order
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (!ok[e]) continue;
        const int s = s0 + base + w0 + e * nw;
        const unsigned m = (unsigned)(ct - cs[e]);
        const double rm = __drcp_rn((double)m);
        double a = 0.0;
        for (int rr = 0; rr < rows; ++rr)
          a = __dadd_rn(a, plog_dev((unsigned)cum[rr * kk + t] - (unsigned)cum[rr * kk + s], m, rm));
        acch[e] = a;
      }
      r = rows;
    }
#endif
    // unsigned offsets from the row base (one IMAD.WIDE.U32 per address)
#if KDP_SPAN2
    // two rows per step: all eight gathers are issued before the adds (each
    // sum still runs in row order)
    for (; r + 2 <= rows; r += 2) {
      const unsigned ctr0 = cum[r * kk + t], ctr1 = cum[(r + 1) * kk + t];
      double v[2][4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int s = s0 + base + w0 + e * nw;
        v[0][e] = ok[e] ? __ldg(pl + (plm[e] + (ctr0 - (unsigned)cum[r * kk + s]))) : 0.0;
        v[1][e] = ok[e] ? __ldg(pl + (plm[e] + (ctr1 - (unsigned)cum[(r + 1) * kk + s]))) : 0.0;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) acch[e] = __dadd_rn(__dadd_rn(acch[e], v[0][e]), v[1][e]);
    }
#endif
    for (; r < rows; ++r) {
      const unsigned ctr = cum[r * kk + t];
      double v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int s = s0 + base + w0 + e * nw;
        v[e] = ok[e] ? __ldg(pl + (plm[e] + (ctr - (unsigned)cum[r * kk + s]))) : 0.0;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) acch[e] = __dadd_rn(acch[e], v[e]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (!ok[e]) continue;
      const int sl = base + w0 + e * nw;
      double a, q;
      if (tb.div) {
        const double* dr = tb.div + tri(ct);
        a = __ldg(dr + cs[e]);
        q = __ldg(dr + (ct - cs[e]));
      } else {
        const double dcs = (double)cs[e];
        a = int_quot(dcs, dct, rct);
        q = int_quot(__dsub_rn(dct, dcs), dct, rct);
      }
      A[sl * kMaxTile + tl] = a;
      W[sl * kMaxTile + tl] = __dmul_rn(q, -acch[e]);
    }
  }
}

// 8-byte global -> shared copy that does not occupy registers until the wait
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// F lives in a per-CTA HBM slot (L2-resident for typical sizes); each outer
// s-chunk's rows are staged into shared memory with coalesced loads, and the
// current t-tile's rows are kept in shared memory while its inner part runs.
#ifndef KDP_MIN_BLOCKS
#define KDP_MIN_BLOCKS 4
#endif
#ifndef KDP_WIDE_MIN_BLOCKS
#define KDP_WIDE_MIN_BLOCKS 3
#endif
#ifndef KDP_CTAS_PER_SM
#define KDP_CTAS_PER_SM 4
#endif
// kLean: x_max <= kLeanXMax (one level tile of <= 62 levels): compiled for 64
// registers so 4 CTAs share an SM; the wider variants keep 80 (3 per SM).

// Persistent: each CTA pulls subproblems from the big lists of the y's
// gi0 .. gi0 + gcount - 1 in ascending y (the heaviest first).  The layout is
// set up per item (the launch's shared memory is the maximum over its y's);
// F lives in this CTA's HBM slot of fslot_stride doubles.
template <bool kGlobalTables, bool kRing, bool kLean>
__global__ void __launch_bounds__(kDpThreads, kLean ? KDP_MIN_BLOCKS : KDP_WIDE_MIN_BLOCKS) k_dp(VarSet vs, Tables tb, PairSpace ps,
                                                      long long base, GenGroup grp, int gi0,
                                                      int gcount, double* __restrict__ fslots,
                                                      unsigned long long fslot_stride,
                                                      double* __restrict__ ocells,
                                                      SubDebug dbg, int has_dbg, int orient_only) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ long long s_sub;
  __shared__ int s_gi;
  const int tid = threadIdx.x;
  const int norient = orient_only >= 0 ? 1 : 2;
  if (tid == 0) s_gi = gi0;
  double* const F = fslots + (size_t)blockIdx.x * fslot_stride;

  for (;;) {
    __syncthreads();
    if (tid == 0) {
      long long got = -1;
      int gi = s_gi;
      for (; gi < gi0 + gcount; ++gi) {  // ascending y: drain y's list, then move on
        const unsigned long long i = atomicAdd(grp.cnt + 2 * grp.ny + gi, 1ull);
        if (i < grp.cnt[grp.ny + gi]) {
          got = grp.ys[gi].big_list[i];
          break;
        }
      }
      s_gi = gi;
      s_sub = got;
    }
    __syncthreads();
    const long long sub = s_sub;
    if (sub < 0) break;
    const GenY& GY = grp.ys[s_gi];
    const YParams yp = GY.yp;
    const GenScratch gs = scratch_of(GY, grp.nsub);
    const int y = yp.y, x_max = yp.x_max, kc = gs.kc, LW = x_max - 1;
    const DpLayout L = dp_layout(y, kc, x_max, kGlobalTables, kLean);
    // row widths: compile-time for the wide variants (x_max > 64: 64 / 65)
    const int fsw = kLean ? L.fsw : 64, ftw = kLean ? L.ftw : 65;
    constexpr int GL = dp_gl(kLean), kAccStride = dp_acc_stride(kLean);
    int* cb = reinterpret_cast<int*>(smem + L.cb);
    int* cum = reinterpret_cast<int*>(smem + L.cum);
    double* A = reinterpret_cast<double*>(smem + L.A);
    double* W = reinterpret_cast<double*>(smem + L.W);
    double* accS = reinterpret_cast<double*>(smem + L.acc);
    double* fs = reinterpret_cast<double*>(smem + L.fs);
    double* ft = reinterpret_cast<double*>(smem + L.ft);
    // F(t, l) at column l - 2 of row t; above 128 levels the row is a ring of
    // 128 columns (a level tile reads l0-1 .. l1-1 and writes l0 .. l1, 65
    // columns), and F(k, .) -- all of which I_l needs -- is kept in its own row fk
    // (kRing: x_max > 129 only).
    const int RW = kRing ? fring_width(LW) : LW, cm = kRing ? kFRing - 1 : 0x7fffffff;
    double* fk = F + (size_t)(kc + 1) * RW;
    const int4 d = reinterpret_cast<const int4*>(gs.desc)[sub];
    const int k = d.x, rows = d.y, l_max = d.w, kk = k + 1;
    if (l_max < 3) continue;  // finished by k_part_f2
    MB_CHECK(k <= kc && rows <= y && l_max <= x_max && sub < grp.nsub);
    MB_CHECK((size_t)(kc + 1) * RW + LW <= fslot_stride);  // F rows + the fk row inside this CTA's slot
    MB_CHECK(L.total <= 227 * 1024);
    const long long pl = base + sub / norient;
    const int orient = orient_only >= 0 ? orient_only : (int)(sub % 2);
    {
      const int* gcb = gs.cb + (size_t)sub * (kc + 1);
      const int* gcum = gs.cum + (size_t)sub * gs.cum_stride;
      const double* gf2 = gs.f2 + (size_t)sub * (kc + 1);
      if (kGlobalTables) {
        cb = const_cast<int*>(gcb);
        cum = const_cast<int*>(gcum);
      } else {
        for (int j = tid; j <= k; j += kDpThreads) cb[j] = gcb[j];
        for (int i = tid; i < rows * kk; i += kDpThreads) cum[i] = gcum[i];
      }
      for (int t = 2 + tid; t <= k; t += kDpThreads) F[(size_t)t * RW] = gf2[t];
      if (kRing && tid == 0) fk[0] = gf2[k];
    }
    __syncthreads();

    // Level tiles of <= 64 levels.  A thread owns 2 GL cells: two adjacent t
    // (t0 + 2p, t0 + 2p + 1) x a group of GL consecutive levels, so each s
    // costs one 16-byte load for both A, one for both W and GL / 2 for the F
    // values, feeding 2 GL independent max chains.  (T/2) * groups <= 256.
    // (Splitting a chunk's rows over several owner sets when the level tile
    // is narrow was measured: no gain, and the larger hand-over region cost
    // L1 capacity -- c3 -13%.)
    for (int l0 = 3; l0 <= l_max; l0 += 64) {
      const int l1 = min(l0 + 63, l_max), nl = l1 - l0 + 1;
      const int ng = (nl + GL - 1) / GL;
      const int fo = kLean ? 2 * ng : 128 / GL;  // staged row offset between a group's level pairs
      // this thread's first staged element and its stride in (row, level)
      const int st_sl = tid / nl, st_j = tid - st_sl * nl;
      const int st_dsl = kDpThreads / nl, st_dj = kDpThreads - st_dsl * nl;
      const int T = max(2, min(kMaxTile, 2 * (kDpThreads / ng)));
      const int t_lo = (l0 == l_max) ? k : l0;  // level l_max is needed at t = k only
      const int my_tp = tid / ng, my_g = tid - my_tp * ng;
      const int my_l = l0 + GL * my_g;  // first of my GL levels
      const int my_tl = 2 * my_tp;     // first of my 2 t's (tile-local)
      const int inner_threads = ((nl + 31) >> 5) << 5;
      for (int t0 = t_lo; t0 <= k; t0 += T) {
        const int nt = min(T, k - t0 + 1);
        const bool owner = my_tl < nt;
        double acc[2 * GL];
#pragma unroll
        for (int i = 0; i < 2 * GL; ++i) acc[i] = kLowest;
        // ---- outer part: every s < t0 (independent candidates)
        for (int s0 = max(2, l0 - 1); s0 < t0; s0 += T) {
          const int ns = min(T, t0 - s0);
#if KDP_PREFETCH
          // stage F(s, l0-1 .. l1-1) by cp.async, in flight while the span
          // terms' gathers run; no registers are held across span_terms
          // element i = tid + 256 u of the (row, level) grid, walked without
          // a division per element
          for (int sl = st_sl, j = st_j; sl < ns;) {
            cp_async8(fs + sl * fsw + fs_col<GL>(j, fo), F + (size_t)(s0 + sl) * RW + (((l0 - 3) + j) & cm));
            sl += st_dsl;
            j += st_dj;
            if (j >= nl) {
              j -= nl;
              ++sl;
            }
          }
          span_terms(tb, cb, cum, kk, rows, k, s0, ns, t0, nt, A, W);
          cp_async_wait_all();
#else
          span_terms(tb, cb, cum, kk, rows, k, s0, ns, t0, nt, A, W);
          for (int i = tid; i < ns * nl; i += kDpThreads) {  // stage F(s, l0-1 .. l1-1)
            const int sl = i / nl, j = i - sl * nl;
            fs[sl * fsw + fs_col<GL>(j, fo)] = F[(size_t)(s0 + sl) * RW + (((l0 - 3) + j) & cm)];
          }
#endif
          __syncthreads();
          if (owner) {
            // s >= l - 1 holds for all GL levels once s >= my_l + GL - 2; only
            // the chunk(s) near the diagonal need the per-level test.  Cells
            // that are not valid accumulate garbage that is never read.
            const double* fr = fs + 2 * my_g;
            int sl = 0;
            for (; sl < ns && s0 + sl < my_l + GL - 2; ++sl) {
              const int s = s0 + sl;
              const double2 a = *reinterpret_cast<const double2*>(A + sl * kMaxTile + my_tl);
              const double2 w = *reinterpret_cast<const double2*>(W + sl * kMaxTile + my_tl);
#pragma unroll
              for (int i = 0; i < GL; ++i)
                if (s >= my_l + i - 1) {
                  const double f = fr[sl * fsw + (i >> 1) * fo + (i & 1)];
                  acc[i] = dmax(acc[i], __dsub_rn(__dmul_rn(a.x, f), w.x));
                  acc[GL + i] = dmax(acc[GL + i], __dsub_rn(__dmul_rn(a.y, f), w.y));
                }
            }
            // running addresses (W sits kMaxTile^2 doubles after A): the loop
            // body is the 4 loads and the 8 candidates, no index arithmetic
            const double* ap = A + sl * kMaxTile + my_tl;
            const double* fp = fr + sl * fsw;
#pragma unroll(GL == 4 ? 2 : 1)
            for (; sl < ns; ++sl, ap += kMaxTile, fp += fsw) {
              const double2 a = *reinterpret_cast<const double2*>(ap);
              const double2 w = *reinterpret_cast<const double2*>(ap + kMaxTile * kMaxTile);
#pragma unroll
              for (int q = 0; q < GL / 2; ++q) {
                const double2 f = *reinterpret_cast<const double2*>(fp + q * fo);
                acc[2 * q] = dmax(acc[2 * q], __dsub_rn(__dmul_rn(a.x, f.x), w.x));
                acc[2 * q + 1] = dmax(acc[2 * q + 1], __dsub_rn(__dmul_rn(a.x, f.y), w.x));
                acc[GL + 2 * q] = dmax(acc[GL + 2 * q], __dsub_rn(__dmul_rn(a.y, f.x), w.y));
                acc[GL + 2 * q + 1] = dmax(acc[GL + 2 * q + 1], __dsub_rn(__dmul_rn(a.y, f.y), w.y));
              }
            }
          }
          __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < 2 * GL; ++i)
          if (my_tp < kMaxTile / 2) accS[tid * kAccStride + i] = acc[i];
        // ---- inner part: s inside the tile, one t at a time, a level per
        // thread; only the warps holding levels take part (named barrier).
        span_terms(tb, cb, cum, kk, rows, k, t0, nt, t0, nt, A, W);
        for (int tl = tid; tl < nt; tl += kDpThreads)  // column 0: level l0 - 1
          ft[tl * ftw] = F[(size_t)(t0 + tl) * RW + ((l0 - 3) & cm)];
        __syncthreads();
        // The tile's rows in sub-tiles of kSubTile: a sub-tile's own split
        // points run sequentially (a step per row, chains of < kSubTile
        // candidates), then its rows' candidates for every later row of the
        // tile -- independent -- are folded into the hand-over by all threads.
        // (Row by row over the whole tile, chains of up to 31 candidates left
        // 6 of 8 warps waiting at the tile's barrier.)
        for (int sb0 = 0; sb0 < nt; sb0 += kSubTile) {
          const int sb1 = min(sb0 + kSubTile, nt);
          if (tid < inner_threads) {
            const int ll = tid, l = l0 + ll;
            for (int tl = sb0; tl < sb1; ++tl) {
              const int tt = t0 + tl;
              if (ll < nl && tt >= l && !(l == l_max && tt != k)) {
                // owner of cell (tl, ll): thread (tl/2)*ng + ll/GL, slot (tl&1)*GL + ll%GL
                double m = accS[((tl >> 1) * ng + ll / GL) * kAccStride + (tl & 1) * GL + ll % GL];
                const double* Ap = A + tl;
                const double* Wp = W + tl;
                for (int s = max(t0 + sb0, l - 1); s < tt; ++s) {
                  const int sl = s - t0;
                  m = dmax(m, __dsub_rn(__dmul_rn(Ap[sl * kMaxTile], ft[sl * ftw + ll]),
                                        Wp[sl * kMaxTile]));
                }
                ft[tl * ftw + ll + 1] = m;
                F[(size_t)tt * RW + ((l - 2) & cm)] = m;
                if (kRing && tt == k) fk[l - 2] = m;
              }
              named_sync(1, inner_threads);
            }
          }
          if (sb1 >= nt) break;
          __syncthreads();
          // rows [sb1, nt) x levels: candidates s in [t0 + sb0, t0 + sb1);
          // cell (tl, ll) = (sb1, 0) + thread index, walked without a division
          for (int tl = sb1 + st_sl, ll = st_j; tl < nt;) {
            const int l = l0 + ll, tt = t0 + tl;
            if (tt >= l && !(l == l_max && tt != k)) {
              double* slot = accS + ((tl >> 1) * ng + ll / GL) * kAccStride + (tl & 1) * GL + ll % GL;
              double m = *slot;
              for (int sl = max(sb0, l - 1 - t0); sl < sb1; ++sl)
                m = dmax(m, __dsub_rn(__dmul_rn(A[sl * kMaxTile + tl], ft[sl * ftw + ll]), W[sl * kMaxTile + tl]));
              *slot = m;
            }
            tl += st_dsl;
            ll += st_dj;
            if (ll >= nl) {
              ll -= nl;
              ++tl;
            }
          }
          __syncthreads();
        }
        __syncthreads();
      }
    }
    // ---- I_l (mutual_info.cpp:68-70) and the cells
    int X, Yv;
    sub_vars(ps, pl, orient, X, Yv);
    const double hq = vs.hq[(size_t)Yv * vs.ny + yp.yi];
    write_cells(
        tb, ocells, pl, orient, y, x_max, rows,
        [&](int l) {
          const int le = l <= l_max ? l : l_max;
          return dmax(0.0, __dadd_rn(hq, kRing ? fk[le - 2] : F[(size_t)k * RW + (le - 2)]));
        },
        dbg, has_dbg != 0);
  }
}

// ---------------------------------------------------------------------------
// Warp path: one warp per small subproblem (k <= kSmallK), t-outer with the
// whole F table, the span column and the clump bounds in this warp's slice of
// shared memory (the cumulative counts are read in place, L1) -- no
// block-level synchronisation, so 16+ independent subproblems interleave per
// SM.  The y's are launched in classes of F width (x_max - 1 <= 3, 7, 15,
// 31, more), each sized for its own widest F: one launch sized for y = 2 left
// c3's many narrow items (y >= 19, x_max = 3) at one CTA per SM.
#ifndef KDPW_SPAN_T
#define KDPW_SPAN_T 2  // measured: 2 best (c0 -5.6%, c2 -3.1%); 4 and 8 cost occupancy
#endif
constexpr int kWarpSpanT = KDPW_SPAN_T;  // span columns gathered together
struct WarpLayout {
  size_t F, A, W, cb, per_warp;
};

__host__ __device__ inline WarpLayout warp_layout(int y, int x_max) {
  (void)y;
  WarpLayout L;
  size_t o = 0;
  L.F = o;
  o += al16(sizeof(double) * (kSmallK + 1) * (size_t)(x_max - 1));
  L.A = o;
  o += al16(sizeof(double) * kWarpSpanT * (kSmallK + 1));
  L.W = o;
  o += al16(sizeof(double) * kWarpSpanT * (kSmallK + 1));
  L.cb = o;
  o += al16(sizeof(int) * (kSmallK + 1));
  L.per_warp = o;
  return L;
}
__host__ __device__ inline int warp_class(int x_max) {
  const int w = x_max - 1;
  return w <= 3 ? 0 : w <= 7 ? 1 : w <= 15 ? 2 : w <= 31 ? 3 : 4;
}

constexpr int kWarpThreads = 256;

// Persistent warps pulling the small subproblems of the y's gi0 .. gi0 +
// gcount - 1 in ascending y; each warp owns per_warp bytes of shared memory
// (the maximum warp_layout over the launch's y's).
// kMinBlocks: 4 (57 -> 64 registers, 4 CTAs per SM) for large batches, 1 (the
// compiler's choice, more registers per warp) for small ones, whose few long
// items want ILP more than occupancy (c0 -5%; c2 +0.8% if used there).
template <int kMinBlocks>
__global__ void __launch_bounds__(kWarpThreads, kMinBlocks) k_dp_warp(VarSet vs, Tables tb, PairSpace ps,
                                                          long long base, GenGroup grp, int gi0,
                                                          int gcount, int per_warp,
                                                          double* __restrict__ ocells,
                                                          SubDebug dbg, int has_dbg,
                                                          int orient_only) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* wb = smem + (size_t)wib * per_warp;
  const int norient = orient_only >= 0 ? 1 : 2;
  int gi = gi0;
  for (;;) {
    long long got = -1;
    if (lane == 0) {
      for (; gi < gi0 + gcount; ++gi) {
        const unsigned long long i = atomicAdd(grp.cnt + 3 * grp.ny + gi, 1ull);
        if (i < grp.cnt[gi]) {
          got = grp.ys[gi].small_list[i];
          break;
        }
      }
    }
    gi = __shfl_sync(0xffffffffu, gi, 0);
    const long long sub = __shfl_sync(0xffffffffu, got, 0);
    if (sub < 0) break;
    const GenY& GY = grp.ys[gi];
    const YParams yp = GY.yp;
    const GenScratch gs = scratch_of(GY, grp.nsub);
    const int y = yp.y, x_max = yp.x_max, LW = x_max - 1, kc = gs.kc;
    const WarpLayout L = warp_layout(y, x_max);
    MB_CHECK(L.per_warp <= (size_t)per_warp);
    double* F = reinterpret_cast<double*>(wb + L.F);
    double* A = reinterpret_cast<double*>(wb + L.A);  // kWarpSpanT columns of kSmallK + 1
    double* W = reinterpret_cast<double*>(wb + L.W);
    double* const A0 = A;
    double* const W0 = W;
    int* cb = reinterpret_cast<int*>(wb + L.cb);
    const int* __restrict__ cum = gs.cum + (size_t)sub * gs.cum_stride;  // in place (L1)
    const int4 d = reinterpret_cast<const int4*>(gs.desc)[sub];
    const int k = d.x, rows = d.y, l_max = d.w, kk = k + 1;
    MB_CHECK(k <= kSmallK && rows <= y && l_max <= x_max && sub < grp.nsub);
    {
      const int* gcb = gs.cb + (size_t)sub * (kc + 1);
      const double* gf2 = gs.f2 + (size_t)sub * (kc + 1);
      for (int j = lane; j <= k; j += 32) cb[j] = gcb[j];
      for (int t = 2 + lane; t <= k; t += 32) F[t * LW] = gf2[t];
    }
    __syncwarp();
    // span columns in blocks of kWarpSpanT t's: their entries (independent
    // of the DP) are gathered together -- one column at a time left each t's
    // L2 latency exposed, with few lanes busy at small t
    // with l_max = 3 only F(k, 3) is needed (rows t < k would feed level 3
    // of a later t, and there is none): only column k's span terms
    for (int tb0 = l_max >= 4 ? 3 : k; tb0 <= k; tb0 += kWarpSpanT) {
      const int tb1 = min(tb0 + kWarpSpanT - 1, k);
      // entries (s, t), t in [tb0, tb1], s in [2, t): column j = t - tb0
      // starts at entry off_j = sum_{i<j} (tb0 + i - 2)
      const int nent = (tb1 - tb0 + 1) * (tb0 - 2) + (tb1 - tb0) * (tb1 - tb0 + 1) / 2;
      for (int e = lane; e < nent; e += 32) {
        int j = 0, off = 0;
        while (j + 1 <= tb1 - tb0 && e >= off + (tb0 + j - 2)) {
          off += tb0 + j - 2;
          ++j;
        }
        const int t = tb0 + j, s = 2 + (e - off);
        const int ct = cb[t];
        const double dct = (double)ct, rct = __drcp_rn(dct);
        const int cs = cb[s];
        const unsigned plm = tri(ct - cs);  // 32-bit row base
        const double* __restrict__ pl = tb.pl;
        double acch = 0.0;
        int r = 0;
        if (rows == 2 && tb.h2) {  // the two-row sum as one H2 gather
          acch = h2_at(tb.h2, (unsigned)(ct - cs), (unsigned)cum[t] - (unsigned)cum[s]);
          r = rows;
        }
#if MB_HAVE_LOGDATA
        if (r < rows && tb.span_log) {  // computed p*log(p) (plog.cuh), row order
          const unsigned m = (unsigned)(ct - cs);
          const double rm = __drcp_rn((double)m);
          for (; r < rows; ++r)
            acch = __dadd_rn(acch, plog_dev((unsigned)cum[r * kk + t] - (unsigned)cum[r * kk + s], m, rm));
        }
#endif
        for (; r + 2 <= rows; r += 2) {  // two gathers in flight, added in row order
          const double v0 = __ldg(pl + (plm + ((unsigned)cum[r * kk + t] - (unsigned)cum[r * kk + s])));
          const double v1 = __ldg(pl + (plm + ((unsigned)cum[(r + 1) * kk + t] - (unsigned)cum[(r + 1) * kk + s])));
          acch = __dadd_rn(__dadd_rn(acch, v0), v1);
        }
        if (r < rows)
          acch = __dadd_rn(acch, __ldg(pl + (plm + ((unsigned)cum[r * kk + t] - (unsigned)cum[r * kk + s]))));
        double a, q;
        if (tb.div) {
          const double* dr = tb.div + tri(ct);
          a = __ldg(dr + cs);
          q = __ldg(dr + (ct - cs));
        } else {
          const double dcs = (double)cs;
          a = int_quot(dcs, dct, rct);
          q = int_quot(__dsub_rn(dct, dcs), dct, rct);
        }
        A[j * (kSmallK + 1) + s] = a;
        W[j * (kSmallK + 1) + s] = __dmul_rn(q, -acch);
      }
      __syncwarp();
    for (int t = tb0; t <= tb1; ++t) {
      const double* A = A0 + (t - tb0) * (kSmallK + 1);
      const double* W = W0 + (t - tb0) * (kSmallK + 1);
      // levels 3 .. l_hi of row t: P lanes per level (P = 32 / levels,
      // rounded down to a power of two) split the split points s by phase and
      // max-reduce by shuffles -- large y have few levels, and one lane per
      // level left most of the warp idle
      const int l_hi = t == k ? min(t, l_max) : min(t, l_max - 1);
      const int nlev = l_hi - 2;
      if (nlev > 0) {
        int lp = 0;  // log2 P
        while (lp < 5 && (nlev << (lp + 1)) <= 32) ++lp;
        const int P = 1 << lp;
        for (int base = 0; base < (nlev << lp); base += 32) {
          const int idx = base + lane, lev = idx >> lp, ph = idx & (P - 1);
          const int l = 3 + lev;
          double m = kLowest;
          if (lev < nlev) {
            const double* fc = F + (l - 3);
            for (int s = l - 1 + ph; s < t; s += P)
              m = dmax(m, __dsub_rn(__dmul_rn(A[s], fc[s * LW]), W[s]));
          }
          for (int o = P >> 1; o > 0; o >>= 1) m = dmax(m, __shfl_xor_sync(0xffffffffu, m, o));
          if (lev < nlev && ph == 0) F[t * LW + (l - 2)] = m;
        }
      }
      __syncwarp();
    }
    }
    // I_l (mutual_info.cpp:68-70) and the cells (char_matrix.cpp:57-64)
    const long long pl = base + sub / norient;
    const int orient = orient_only >= 0 ? orient_only : (int)(sub % 2);
    int X, Yv;
    sub_vars(ps, pl, orient, X, Yv);
    const double hq = vs.hq[(size_t)Yv * vs.ny + yp.yi];
    double* oc = ocells + (size_t)pl * 2 * tb.ncell + (size_t)orient * tb.ncell;
    const double logy = tb.logi[rows];
    for (int l = 2 + lane; l <= x_max; l += 32) {
      const int le = l <= l_max ? l : l_max;
      const double v = dmax(0.0, __dadd_rn(hq, F[k * LW + (le - 2)]));
      if (has_dbg) dbg.values[l - 2] = v;
      const int cell = orient ? tb.cell_off[l] + (y - 2) : tb.cell_off[y] + (l - 2);
      oc[cell] = norm_cell(v, tb.logi[l], logy);
    }
    __syncwarp();
  }
}

#if MB_HAVE_LOGDATA
// Every table entry pl[tri(m) + w] against plog_dev(w, m): counts differing bits.
__global__ void k_check_plog(const double* __restrict__ pl, int n, unsigned long long* bad) {
  const unsigned long long total = (unsigned long long)(n + 1) * (n + 2) / 2;
  unsigned long long nb = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    unsigned long long m = (unsigned long long)((sqrt(8.0 * (double)i + 1.0) - 1.0) / 2.0);
    while (m * (m + 1) / 2 > i) --m;
    while ((m + 1) * (m + 2) / 2 <= i) ++m;
    const unsigned w = (unsigned)(i - m * (m + 1) / 2);
    if (m == 0) continue;
    const double v = plog_dev(w, (unsigned)m, __drcp_rn((double)m));
    nb += __double_as_longlong(v) != __double_as_longlong(pl[i]);
  }
  if (nb) atomicAdd(bad, nb);
}
#endif

// Exact quotient table div[tri(m) + w] = w / m (IEEE, as the reference's
// c[s] / c[t]), so the span terms need no DDIV.
__global__ void k_build_div(double* div, int n) {
  const unsigned long long total = (unsigned long long)(n + 1) * (n + 2) / 2;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    // invert i = m(m+1)/2 + w
    unsigned long long m = (unsigned long long)((sqrt(8.0 * (double)i + 1.0) - 1.0) / 2.0);
    while (m * (m + 1) / 2 > i) --m;
    while ((m + 1) * (m + 2) / 2 <= i) ++m;
    const unsigned long long w = i - m * (m + 1) / 2;
    div[i] = m ? __ddiv_rn((double)w, (double)m) : 0.0;
  }
}

// H2(m, w) = pl(m, w) + pl(m, m - w) for w <= m/2: one thread per entry.
__global__ void k_build_h2(const double* __restrict__ pl, double* __restrict__ h2, int n) {
  const unsigned long long total = h2_off((unsigned)n + 1u);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    // invert i = h2_off(m) + w: h2_off is increasing, ~ m^2 / 4
    unsigned m = (unsigned)(2.0 * sqrt((double)i));
    while (m > 0 && h2_off(m) > i) --m;
    while (h2_off(m + 1u) <= i) ++m;
    const unsigned w = (unsigned)(i - h2_off(m));
    const double* row = pl + tri(m);
    h2[i] = __dadd_rn(row[w], row[m - w]);
  }
}

}  // namespace

size_t h2_table_doubles(int n) { return h2_off((unsigned)n + 1u); }

void launch_build_h2(const double* pl, double* h2, int n, cudaStream_t s) {
  const size_t total = h2_table_doubles(n);
  const unsigned blocks = (unsigned)std::min<size_t>(8192, (total + 255) / 256);
  k_build_h2<<<blocks, 256, 0, s>>>(pl, h2, n);
}

// ---------------------------------------------------------------------------
int gen_kc(int n, const YParams& yp) { return std::min(n, yp.k_hat); }

// cb / cum are read in place (L1 / L2) instead of staged in k_dp's shared
// memory when staging them would cost more than 48 KB -- c B large, e.g. c4
// (7.5k clumps at y = 2, ~60 KB of cumulative counts at every y): the smaller
// footprint lets 3 CTAs share an SM instead of 1 (c4 +14%).
bool gen_tables_global(int n, const YParams& yp) {
  static const bool force = std::getenv("MINE_B200_DP_GLOBAL") != nullptr;
  const size_t kc1 = (size_t)gen_kc(n, yp) + 1;
  const size_t staged = al16(sizeof(int) * kc1) + al16(sizeof(int) * (size_t)yp.y * kc1);
  return force || staged > 48 * 1024 ||
         dp_layout(yp.y, gen_kc(n, yp), yp.x_max, false, false).total > 200 * 1024;
}

bool gen_pts_global(int n, const YParams& yp) {
  static const bool force = std::getenv("MINE_B200_PF_GLOBAL") != nullptr;
  return force || gen_tables_global(n, yp) ||
         pf_layout(n, yp.y, gen_kc(n, yp), false).total > 200 * 1024;
}

size_t gen_pts_bytes(int n, const YParams& yp) {
  return gen_pts_global(n, yp) ? pf_layout(n, yp.y, gen_kc(n, yp), true).pts : 0;
}

size_t gen_scratch_per_sub(int n, const YParams& yp) {
  const size_t kc = (size_t)gen_kc(n, yp);
  return sizeof(int4) + sizeof(int) * (kc + 1) + sizeof(int) * (size_t)yp.y * (kc + 1) +
         sizeof(double) * (kc + 1) + gen_pts_bytes(n, yp) + 2 * sizeof(long long);
}

size_t gen_pf_smem(int n, const YParams& yp) {
  return pf_layout(n, yp.y, gen_kc(n, yp), gen_pts_global(n, yp), gen_tables_global(n, yp)).total;
}

// The lean k_dp (64 registers) pays off only where its compact layout lets 4
// CTAs share an SM; alone on an SM the 80-register variant is faster (c4).
bool gen_dp_lean(int n, const YParams& yp) {
  if (gen_tables_global(n, yp) || yp.x_max > kLeanXMax) return false;
  return dp_layout(yp.y, gen_kc(n, yp), yp.x_max, false, true).total + 1024 <= 228 * 1024 / 4;
}

size_t gen_dp_smem(int n, const YParams& yp) {
  return dp_layout(yp.y, gen_kc(n, yp), yp.x_max, gen_tables_global(n, yp), gen_dp_lean(n, yp)).total;
}

size_t gen_fslot_bytes(int n, const YParams& yp) {
  return sizeof(double) * fslot_doubles(gen_kc(n, yp), yp.x_max - 1);
}

static int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

static size_t warp_per_warp(const YParams& yp) { return warp_layout(yp.y, yp.x_max).per_warp; }
// The warp path takes y's whose items' tables are small: the cumulative
// counts are read in place, but their y (kSmallK + 1) ints per item must stay
// L1-friendly (c4's y ~ 300 items are faster on k_dp).
static bool warp_ok(const YParams& yp) {
  return yp.x_max >= 3 && warp_per_warp(yp) + sizeof(int) * (size_t)yp.y * (kSmallK + 1) <= 24 * 1024;
}

// up to this many samples the F(t,2) level runs on 128 threads too (c2,
// n = 500: +8%; 64 threads measured slower)
static int pf_small_n() {
  static const int v = [] {
    const char* e = std::getenv("MINE_B200_PF128_N");
    return e ? std::atoi(e) : 700;
  }();
  return v;
}

// k_part_f2 / k_dp template variant of a row target; a launch covers a run of
// consecutive y's with the same variant.
enum { kPfGlobalTables = 0, kPfGlobalPts, kPf256, kPf128 };
static int pf_variant(int n, const YParams& yp) {
  if (gen_tables_global(n, yp)) return kPfGlobalTables;
  if (gen_pts_bytes(n, yp)) return kPfGlobalPts;
  return yp.x_max >= 3 && n > pf_small_n() ? kPf256 : kPf128;
}
enum { kDpNone = -1, kDpGlobalTables = 0, kDpRing, kDpWide, kDpLean, kDpLeanInPlace };
// MINE_B200_DP_INPLACE=1: the lean k_dp reads cb / cum in place from the
// scratch slot (k_part_f2 always writes them there) instead of staging them,
// for a smaller shared footprint (more L1)
static bool dp_inplace() {
  static const bool on = [] {
    const char* e = std::getenv("MINE_B200_DP_INPLACE");
    return e && e[0] == '1';
  }();
  return on;
}
static int dp_variant(int n, const YParams& yp) {
  if (yp.x_max < 3) return kDpNone;
  if (gen_tables_global(n, yp)) return kDpGlobalTables;
  if (yp.x_max - 1 > kFRing) return kDpRing;
  if (!gen_dp_lean(n, yp)) return kDpWide;
  return dp_inplace() ? kDpLeanInPlace : kDpLean;
}
static size_t dp_variant_smem(int v, int n, const YParams& yp) {
  if (v == kDpLeanInPlace) return dp_layout(yp.y, gen_kc(n, yp), yp.x_max, true, true).total;
  return gen_dp_smem(n, yp);
}

// The k_dp launches of a group: runs of consecutive y's with one variant.
struct DpRun {
  int gi0, count, variant, grid;
  size_t smem, fslot_doubles;
};
static std::vector<DpRun> dp_runs(int n, const YParams* yps, int ny, long long nsub) {
  std::vector<DpRun> runs;
  const int sms = sm_count();
  for (int gi = 0; gi < ny;) {
    const int v = dp_variant(n, yps[gi]);
    int gj = gi + 1;
    while (gj < ny && dp_variant(n, yps[gj]) == v) ++gj;
    if (v != kDpNone) {
      DpRun r{gi, gj - gi, v, 0, 0, 0};
      for (int g = gi; g < gj; ++g) {
        r.smem = std::max(r.smem, dp_variant_smem(v, n, yps[g]));
        r.fslot_doubles = std::max(r.fslot_doubles, gen_fslot_bytes(n, yps[g]) / sizeof(double));
      }
      // up to 4 CTAs per SM, as shared memory allows (the wide variants are
      // register-bound at 3 resident; their extra CTAs start as others finish)
      const int per = (int)std::max<size_t>(1, std::min<size_t>(KDP_CTAS_PER_SM, (228 * 1024) / (r.smem + 1024)));
      // the F slots of one run stay within 4 GB (very large c B)
      const long long cap = std::max<long long>(1, (4LL << 30) / (long long)(8 * r.fslot_doubles));
      r.grid = (int)std::min<long long>(std::min<long long>((long long)sms * per, cap),
                                        nsub * (gj - gi));
      runs.push_back(r);
    }
    gi = gj;
  }
  return runs;
}

size_t gen_group_fslot_bytes(int n, const YParams* yps, int ny, long long nsub) {
  size_t b = 0;
  for (const DpRun& r : dp_runs(n, yps, ny, nsub)) b += al16(8 * r.fslot_doubles * (size_t)r.grid);
  return b;
}

// Row-map dedup, second half: subproblems k_part_f2 marked as copies
// (l_max = -1, desc.z = the canonical y's group index) take that y's cells
// (l, y') for l = 2 .. x_max(y) once every kernel of the group has written
// them.  One thread per (y, subproblem).
__global__ void k_copy_dups(VarSet vs, Tables tb, PairSpace ps, long long base, GenGroup grp,
                            double* __restrict__ ocells, int orient_only) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= grp.nsub * grp.ny) return;
  const int gi = (int)(i / grp.nsub);
  const long long sub = i % grp.nsub;
  const int4 d = reinterpret_cast<const int4*>(grp.ys[gi].desc)[sub];
  if (d.w != -1) return;
  const int norient = orient_only >= 0 ? 1 : 2;
  const long long pl = base + sub / norient;
  const int orient = orient_only >= 0 ? orient_only : (int)(sub % 2);
  const int y = grp.ys[gi].yp.y, yc = grp.ys[d.z].yp.y, x_max = grp.ys[gi].yp.x_max;
  MB_CHECK(d.z < gi && yc < y && grp.ys[d.z].yp.x_max >= x_max);
  double* oc = ocells + (size_t)pl * 2 * tb.ncell + (size_t)orient * tb.ncell;
  for (int l = 2; l <= x_max; ++l) {
    const int to = orient ? tb.cell_off[l] + (y - 2) : tb.cell_off[y] + (l - 2);
    const int from = orient ? tb.cell_off[l] + (yc - 2) : tb.cell_off[yc] + (l - 2);
    oc[to] = oc[from];
  }
}

// Which y's of a group take k_part_warp: the suffix wp0 .. ny-1 of y's whose
// clump budget min(n, k_hat) is at most 160000 / n (MINE_B200_WARP_PART_KC
// overrides; 0 turns the warp kernel off) -- with more clumps the F(t,2)
// level, not the partition, dominates and the CTA kernel's 4-8 warps per
// subproblem win (measured: c2, n = 500, fastest with every y here, 13.1 ->
// 10.8 ms; c0, n = 1000, with k_hat <= 64..160) -- and n <= kWarpPartMaxN
// with the point arrays on chip, no debug export.  Returns the per-warp
// shared memory (0: none).
static size_t warp_part_bytes(int n, const YParams* yps, int ny, bool dbg, long long nsub, int& wp0) {
  static const int kc_env = [] {
    const char* e = std::getenv("MINE_B200_WARP_PART_KC");
    return e ? std::atoi(e) : -1;
  }();
  // small batches (fewer than 8 subproblems per SM and y) want the CTA
  // kernel's warps per subproblem: a single pair through the reference API
  // is latency-bound (n = 400: 747 -> ~620 us per pair)
  const int kc_max = kc_env >= 0 ? kc_env
                     : nsub < 8LL * sm_count() ? 0
                                               : std::max(64, 160000 / std::max(n, 1));
  wp0 = ny;
  if (kc_max <= 0 || dbg || n > kWarpPartMaxN) return 0;
  while (wp0 > 0 && gen_kc(n, yps[wp0 - 1]) <= kc_max && !gen_tables_global(n, yps[wp0 - 1]) &&
         !gen_pts_global(n, yps[wp0 - 1]))
    --wp0;
  size_t cum = 0;
  for (int gi = wp0; gi < ny; ++gi) cum = std::max(cum, (size_t)yps[gi].y * (gen_kc(n, yps[gi]) + 1));
  const size_t b = wp_layout(n, cum).per_warp;
  if (wp0 == ny || b * kWpWarps > 200 * 1024) {
    wp0 = ny;
    return 0;
  }
  return b;
}

static int launch_copy_dups(const VarSet& vs, const Tables& tb, const PairSpace& ps, long long base,
                            const GenGroup& g, int ny, long long nsub, double* ocells, int orient_only,
                            cudaStream_t s) {
  const long long total = nsub * ny;
  k_copy_dups<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(vs, tb, ps, base, g, ocells, orient_only);
  return 1;
}

int gen_run_group(const VarSet& vs, const Tables& tb, const PairSpace& ps, long long base,
                  long long npairs, const YParams* yps, int ny, void* scratch, GenY* d_ys,
                  unsigned long long* d_cnt, double* fslots, double* ocells, const SubDebug* dbg,
                  int orient_only, unsigned long long* counters, cudaStream_t s0,
                  const cudaStream_t* sides, cudaEvent_t* ev) {
  if (npairs <= 0 || ny <= 0) return 0;
  const int n = vs.n;
  const long long nsub = npairs * (orient_only >= 0 ? 1 : 2);
  // ---- per-y scratch regions, carved from one buffer
  std::vector<GenY> hy(ny);
  char* p = static_cast<char*>(scratch);
  auto carve = [&](size_t bytes) {
    char* q = p;
    p += al16(bytes);
    return q;
  };
  // the descriptors of all y's first, contiguous: one memset clears them for
  // the row-map dedup (k_part_f2 reads a smaller y's raw k there)
  for (int gi = 0; gi < ny; ++gi) hy[gi].desc = reinterpret_cast<int*>(carve(sizeof(int4) * nsub));
  if (vs.qsame) cudaMemsetAsync(hy[0].desc, 0, (size_t)(p - static_cast<char*>(scratch)), s0);
  for (int gi = 0; gi < ny; ++gi) {
    GenY& Y = hy[gi];
    int* const desc = Y.desc;
    std::memset(&Y, 0, sizeof(Y));
    Y.desc = desc;
    Y.yp = yps[gi];
    Y.kc = gen_kc(n, Y.yp);
    Y.small_ok = warp_ok(Y.yp);
    Y.tables_global = gen_tables_global(n, Y.yp);
    Y.cum_stride = (unsigned long long)Y.yp.y * (Y.kc + 1);
    Y.cb = reinterpret_cast<int*>(carve(sizeof(int) * (size_t)(Y.kc + 1) * nsub));
    Y.cum = reinterpret_cast<int*>(carve(sizeof(int) * Y.cum_stride * nsub));
    Y.f2 = reinterpret_cast<double*>(carve(sizeof(double) * (size_t)(Y.kc + 1) * nsub));
    const size_t ptsb = gen_pts_bytes(n, Y.yp);
    Y.pts = ptsb ? reinterpret_cast<unsigned char*>(carve(ptsb * nsub)) : nullptr;
    Y.small_list = reinterpret_cast<long long*>(carve(sizeof(long long) * nsub));
    Y.big_list = reinterpret_cast<long long*>(carve(sizeof(long long) * nsub));
  }
  cudaMemcpyAsync(d_ys, hy.data(), sizeof(GenY) * ny, cudaMemcpyHostToDevice, s0);
  cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * (4 * ny + 4), s0);
  GenGroup g;
  g.ys = d_ys;
  g.ny = ny;
  g.nsub = nsub;
  g.cnt = d_cnt;
  SubDebug d{};
  if (dbg) d = *dbg;
  const int dg = dbg ? 1 : 0;
  int launches = 0;
  // ---- partitions + F(t,2): the warp kernel over every (y, subproblem) of
  // the group when the per-point arrays fit a warp's slice of shared memory,
  // else one k_part_f2 launch per run of one variant; y-major either way
  int wp0 = ny;  // the y's from wp0 on take the warp kernel
  const size_t wpw = warp_part_bytes(n, yps, ny, dbg != nullptr, nsub, wp0);
  for (int gi = 0; gi < wp0;) {
    const int v = pf_variant(n, yps[gi]);
    int gj = gi + 1;
    while (gj < wp0 && pf_variant(n, yps[gj]) == v) ++gj;
    size_t sm = 0;
    for (int q = gi; q < gj; ++q) sm = std::max(sm, gen_pf_smem(n, yps[q]));
    const unsigned blocks = (unsigned)(nsub * (gj - gi));
#define PF_LAUNCH(T, PG, CG) \
  k_part_f2<T, PG, CG><<<blocks, T, sm, s0>>>(vs, tb, ps, base, g, gi, ocells, d, dg, orient_only, counters)
    switch (v) {
      case kPfGlobalTables: PF_LAUNCH(256, true, true); break;
      case kPfGlobalPts: PF_LAUNCH(256, true, false); break;
      case kPf256: PF_LAUNCH(256, false, false); break;
      default: PF_LAUNCH(128, false, false); break;
    }
#undef PF_LAUNCH
    ++launches;
    gi = gj;
  }
  if (wp0 < ny) {  // after the CTA launches: their y's are smaller (row-map dedup order)
    const long long warps = nsub * (ny - wp0);
    const int per = (int)std::max<size_t>(1, std::min<size_t>(4, (228 * 1024) / (kWpWarps * wpw + 1024)));
    const long long grid = std::min<long long>((warps + kWpWarps - 1) / kWpWarps, (long long)sm_count() * per);
    k_part_warp<<<(unsigned)grid, kWpWarps * 32, kWpWarps * wpw, s0>>>(
        vs, tb, ps, base, g, wp0, ny - wp0, (int)wpw, ocells, orient_only, counters);
    ++launches;
  }
  // ---- levels >= 3: the k_dp runs and the warp path, each on its own lane
  const std::vector<DpRun> runs = dp_runs(n, yps, ny, nsub);
  int wlo = ny, whi = -1;
  for (int gi = 0; gi < ny; ++gi)
    if (warp_ok(yps[gi])) {
      wlo = std::min(wlo, gi);
      whi = std::max(whi, gi);
    }
  if (runs.empty() && whi < wlo) {
    if (vs.qsame) launches += launch_copy_dups(vs, tb, ps, base, g, ny, nsub, ocells, orient_only, s0);
    return launches;
  }
  // the warp path on the side lane (its items are disjoint from k_dp's), the
  // k_dp runs in ascending y on the main lane
  const bool forked = whi >= wlo && sides && sides[0];
  if (forked) cudaEventRecord(ev[0], s0);
  bool used[kGenSides] = {};
  auto launch_dp = [&] {
  char* fp = reinterpret_cast<char*>(fslots);
    for (const DpRun& r : runs) {
      double* fs = reinterpret_cast<double*>(fp);
      fp += al16(8 * r.fslot_doubles * (size_t)r.grid);
  #define DP_LAUNCH(GT, RG, LN)                                                                 \
    k_dp<GT, RG, LN><<<r.grid, kDpThreads, r.smem, s0>>>(vs, tb, ps, base, g, r.gi0, r.count, fs, \
                                                          r.fslot_doubles, ocells, d, dg, orient_only)
      switch (r.variant) {
        case kDpGlobalTables: DP_LAUNCH(true, true, false); break;
        case kDpRing: DP_LAUNCH(false, true, false); break;
        case kDpWide: DP_LAUNCH(false, false, false); break;
        case kDpLeanInPlace: DP_LAUNCH(true, false, true); break;
        default: DP_LAUNCH(false, false, true); break;
      }
  #undef DP_LAUNCH
      ++launches;
    }
  };
  auto launch_warp = [&] {
  // the warp path after the k_dp runs are enqueued: the persistent k_dp CTAs
    // (the long y = 2 items) are dispatched first, the warp CTAs fill the rest
    // one k_dp_warp launch per F-width class (consecutive y's), in ascending y
    // Five classes in sequence on one side stream for large batches (c2 -4%,
    // c3 -2.4% against concurrent), on concurrent side streams for small
    // ones (c0, 512 subproblems per y: -6%; a class with few long items
    // would otherwise hold up the next).  MINE_B200_DPW_MODE (A/B): 0 five
    // classes concurrent, 1 five in sequence, 2 / 3 two classes (F width
    // <= 7, wider) concurrent / in sequence, 4 one launch.
    static const int mode_env = [] {
      const char* e = std::getenv("MINE_B200_DPW_MODE");
      return e ? std::atoi(e) : -1;
    }();
    // (a handful of subproblems, e.g. one pair through the reference API:
    // one launch, the class split only costs launch latency)
    const int mode = mode_env >= 0 ? mode_env : nsub > 2048 ? 1 : nsub >= 64 ? 0 : 4;
    auto wclass = [&](int x_max) {
      if (mode == 4) return 0;
      const int c = warp_class(x_max);
      return mode >= 2 ? (c <= 1 ? 0 : 1) : c;
    };
    const bool seq = mode == 1 || mode == 3;
    for (int gi = wlo; gi <= whi;) {
      const int cls = wclass(yps[gi].x_max);
      int gj = gi;
      size_t per_warp = 0;
      while (gj <= whi && warp_ok(yps[gj]) && wclass(yps[gj].x_max) == cls)
        per_warp = std::max(per_warp, warp_per_warp(yps[gj++]));
      if (gj == gi) {  // not on the warp path
        ++gi;
        continue;
      }
      const int warps = kWarpThreads / 32;
      const size_t sm = per_warp * warps;
      const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (220 * 1024) / (sm + 1024)));
      const int grid = (int)std::max<long long>(
          1, std::min<long long>((nsub * (gj - gi) + warps - 1) / warps, (long long)sm_count() * per_sm));
      // each class on its own side stream: the classes run concurrently
      cudaStream_t sw = s0;
      if (forked) {
        const int si = seq ? 0 : cls % kGenSides;
        sw = sides[si];
        if (!used[si]) cudaStreamWaitEvent(sw, ev[0], 0);
        used[si] = true;
      }
      if (seq)
        k_dp_warp<4><<<grid, kWarpThreads, sm, sw>>>(vs, tb, ps, base, g, gi, gj - gi, (int)per_warp, ocells,
                                                     d, dg, orient_only);
      else
        k_dp_warp<1><<<grid, kWarpThreads, sm, sw>>>(vs, tb, ps, base, g, gi, gj - gi, (int)per_warp, ocells,
                                                     d, dg, orient_only);
      ++launches;
      gi = gj;
    }
  };
  // MINE_B200_DPW_FIRST=1: the warp path enqueued first (A/B)
  static const bool warp_first = [] {
    const char* e = std::getenv("MINE_B200_DPW_FIRST");
    return e && e[0] == '1';
  }();
  if (warp_first) {
    launch_warp();
    launch_dp();
  } else {
    launch_dp();
    launch_warp();
  }
  for (int si = 0; si < kGenSides; ++si)
    if (used[si]) {
      cudaEventRecord(ev[1 + si], sides[si]);
      cudaStreamWaitEvent(s0, ev[1 + si], 0);
    }
  if (vs.qsame) launches += launch_copy_dups(vs, tb, ps, base, g, ny, nsub, ocells, orient_only, s0);
  return launches;
}

size_t div_table_doubles(int n) { return (size_t)(n + 1) * (n + 2) / 2; }

long long check_plog_table(const double* pl, int n, unsigned long long* scratch, cudaStream_t s) {
#if MB_HAVE_LOGDATA
  const size_t total = (size_t)(n + 1) * (n + 2) / 2;
  cudaMemsetAsync(scratch, 0, sizeof(unsigned long long), s);
  const unsigned blocks = (unsigned)std::min<size_t>(4096, (total + 255) / 256);
  k_check_plog<<<blocks, 256, 0, s>>>(pl, n, scratch);
  unsigned long long bad = 0;
  if (cudaMemcpyAsync(&bad, scratch, sizeof(bad), cudaMemcpyDeviceToHost, s) != cudaSuccess) return -1;
  if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
  return (long long)bad;
#else
  (void)pl, (void)n, (void)scratch, (void)s;
  return -1;
#endif
}

void launch_build_div(double* div, int n, cudaStream_t s) {
  const size_t total = div_table_doubles(n);
  const unsigned blocks = (unsigned)std::min<size_t>(4096, (total + 255) / 256);
  k_build_div<<<blocks, 256, 0, s>>>(div, n);
}

cudaError_t init_general_attributes(int device) {
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) return e;
  const void* fns[] = {reinterpret_cast<const void*>(k_part_f2<256, false, false>),
                       reinterpret_cast<const void*>(k_part_f2<128, false, false>),
                       reinterpret_cast<const void*>(k_part_f2<256, true, false>),
                       reinterpret_cast<const void*>(k_part_f2<256, true, true>),
                       reinterpret_cast<const void*>(k_dp<false, false, false>),
                       reinterpret_cast<const void*>(k_dp<false, false, true>),
                       reinterpret_cast<const void*>(k_dp<false, true, false>),
                       reinterpret_cast<const void*>(k_dp<true, true, false>),
                       reinterpret_cast<const void*>(k_dp<true, false, true>),
                       reinterpret_cast<const void*>(k_dp_warp<1>),
                       reinterpret_cast<const void*>(k_dp_warp<4>),
                       reinterpret_cast<const void*>(k_part_warp)};
  for (const void* f : fns) {
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
  }
  // Preferred shared-memory carveout of the wide / ring / global-table k_dp
  // (large c B, e.g. c4): 58% (132 KB) leaves the rest of the SM's 256 KB as
  // L1, where the span terms' p*log(p) rows and the in-place cb / cum hit
  // (c4 +11% over the default; MINE_B200_DP_CARVEOUT overrides, and also
  // applies it to the lean variant, which is fastest at the default).
  {
    const char* cv = std::getenv("MINE_B200_DP_CARVEOUT");
    const int pct = cv ? std::atoi(cv) : 58;
    const void* dps[] = {reinterpret_cast<const void*>(k_dp<false, false, false>),
                         reinterpret_cast<const void*>(k_dp<false, true, false>),
                         reinterpret_cast<const void*>(k_dp<true, true, false>),
                         cv ? reinterpret_cast<const void*>(k_dp<false, false, true>) : nullptr,
                         cv ? reinterpret_cast<const void*>(k_dp<true, false, true>) : nullptr};
    for (const void* f : dps) {
      if (!f) continue;
      e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace mb200
