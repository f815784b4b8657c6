"""Python binding of the C ABI (include/mine_b200.h) of libmine_b200.so.

Mirrors the reference's interface for the hot path (proj/include/mine/*.hpp):
``Parameters``, ``validate_parameters``, ``grid_bound``, ``compute_score`` ->
``CharacteristicMatrix``, ``compute_statistics``, plus the batch calls
``pairwise`` / ``cross`` / ``pairs`` that replace ``run_analysis``.  Every
number comes from the GPU; if the library or a Blackwell GPU is missing the
call raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MINE_B200_LIB", os.path.join(_PKG, "libmine_b200.so"))

MIC_APPROX = 0
MIC_E = 1
STATS = ("mic", "mas", "mev", "mcn", "mic_e", "tic")
# statistics.cpp:39-51, computed only when requested
EXTRA_STATS = ("pearson_r", "nonlinearity")
ALL_STATS = STATS + EXTRA_STATS

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


class MineError(ValueError):
    """The condition the reference throws std::invalid_argument for."""


class MineParameter(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("c", ctypes.c_double), ("est", ctypes.c_int)]


class MineStatsOut(ctypes.Structure):
    _fields_ = [(k, _dp) for k in STATS] + [("cells", _dp)] + [(k, _dp) for k in EXTRA_STATS]


NCOUNTERS = 10
COUNTERS = ("fp64_ops", "lookups", "dp_candidates", "span_entries", "subproblems", "gathers",
            "rank_gathers", "point_visits", "f2_candidates", "span_lookups")


class MineOpts(ctypes.Structure):
    _fields_ = [("device_io", ctypes.c_int), ("async_", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("tier", ctypes.c_int), ("first", ctypes.c_longlong), ("count", ctypes.c_longlong),
                ("counters", ctypes.POINTER(ctypes.c_ulonglong)), ("ev_begin", ctypes.c_void_p),
                ("ev_end", ctypes.c_void_p), ("reuse_vars", ctypes.c_int),
                ("ndevices", ctypes.c_int), ("devices", ctypes.POINTER(ctypes.c_int)),
                ("shard_chunk", ctypes.c_longlong)]


class MineDataset(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int), ("n", ctypes.c_int), ("values", _dp),
                ("names", ctypes.POINTER(ctypes.c_char_p))]


class MineTask(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("master", ctypes.c_int), ("first", ctypes.c_int),
                ("second", ctypes.c_int), ("alpha", ctypes.c_double), ("c", ctypes.c_double),
                ("has_min_variance", ctypes.c_int), ("min_variance", ctypes.c_double),
                ("workers", ctypes.c_int)]


MODES = {"all_pairs": 0, "master_vs_all": 1, "single_pair": 2}


class MineProblem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("x", _dp), ("y", _dp)]


class MineMatrix(ctypes.Structure):
    """mine_matrix: n variables x m samples, variable-major."""
    _fields_ = [("data", ctypes.POINTER(ctypes.c_double)), ("n", ctypes.c_int), ("m", ctypes.c_int)]


class MinePstats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_longlong), ("mic", ctypes.POINTER(ctypes.c_double)),
                ("tic", ctypes.POINTER(ctypes.c_double))]


class MineCstats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_longlong), ("m", ctypes.c_longlong),
                ("mic", ctypes.POINTER(ctypes.c_double)), ("tic", ctypes.POINTER(ctypes.c_double))]


class MineScore(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("m", _ip), ("M", ctypes.POINTER(_dp)),
                ("M_e", ctypes.POINTER(_dp)), ("B", ctypes.c_int), ("est", ctypes.c_int)]


_LIB = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libmine_b200.so; raises if it is absent (never falls back)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with __graft_entry__.build() "
                           "(the engine has no CPU fallback)")
    L = ctypes.CDLL(path)
    vp = ctypes.c_void_p
    L.mine_b200_last_error.restype = ctypes.c_char_p
    L.mine_b200_create.restype = vp
    L.mine_b200_create.argtypes = [ctypes.c_int]
    L.mine_b200_destroy.argtypes = [vp]
    L.mine_b200_destroy.restype = None
    L.mine_b200_grid_bound.argtypes = [ctypes.c_longlong, ctypes.c_double]
    L.mine_b200_cell_count.argtypes = [ctypes.c_int]
    L.mine_b200_last_launches.argtypes = [vp]
    L.mine_b200_last_launches.restype = ctypes.c_longlong
    L.mine_b200_sync.argtypes = [vp]
    P = ctypes.POINTER
    L.mine_b200_pairwise.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, P(MineParameter),
                                     P(MineOpts), P(MineStatsOut)]
    L.mine_b200_cross.argtypes = [vp, vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int,
                                  P(MineParameter), P(MineOpts), P(MineStatsOut)]
    L.mine_b200_pairs.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_longlong,
                                  P(MineParameter), P(MineOpts), P(MineStatsOut)]
    L.mine_b200_debug_subproblem.argtypes = [vp, ctypes.c_int, _dp, _dp, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, _ip, _ip, _ip, _ip, _ip, _dp, _dp]
    L.mine_check_parameter.argtypes = [P(MineParameter)]
    L.mine_check_parameter.restype = ctypes.c_char_p
    L.mine_compute_score.argtypes = [P(MineProblem), P(MineParameter)]
    L.mine_compute_score.restype = P(MineScore)
    L.mine_free_score.argtypes = [P(P(MineScore))]
    L.mine_free_score.restype = None
    L.mine_compute_pstats.argtypes = [P(MineMatrix), P(MineParameter)]
    L.mine_compute_pstats.restype = P(MinePstats)
    L.mine_compute_cstats.argtypes = [P(MineMatrix), P(MineMatrix), P(MineParameter)]
    L.mine_compute_cstats.restype = P(MineCstats)
    L.mine_free_pstats.argtypes = [P(P(MinePstats))]
    L.mine_free_pstats.restype = None
    L.mine_free_cstats.argtypes = [P(P(MineCstats))]
    L.mine_free_cstats.restype = None
    for f in ("mine_mic", "mine_mas", "mine_mev", "mine_mcn_general", "mine_mic_e"):
        getattr(L, f).argtypes = [P(MineScore)]
        getattr(L, f).restype = ctypes.c_double
    L.mine_mcn.argtypes = [P(MineScore), ctypes.c_double]
    L.mine_mcn.restype = ctypes.c_double
    L.mine_tic.argtypes = [P(MineScore), ctypes.c_int]
    L.mine_tic.restype = ctypes.c_double
    L.mine_b200_read_dataset.argtypes = [ctypes.c_char_p, P(P(MineDataset))]
    L.mine_b200_free_dataset.argtypes = [P(MineDataset)]
    L.mine_b200_free_dataset.restype = None
    L.mine_b200_variances.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, _dp]
    L.mine_b200_filter_low_variance.argtypes = [vp, P(MineDataset), ctypes.c_double,
                                                P(P(MineDataset))]
    L.mine_b200_run_analysis.argtypes = [vp, P(MineDataset), P(MineTask), ctypes.c_char_p]
    L.mine_b200_run_analysis.restype = ctypes.c_longlong
    _LIB = L
    return L


def _dataset_to_py(ds_p) -> tuple[list[str], np.ndarray]:
    ds = ds_p.contents
    values = np.ctypeslib.as_array(ds.values, (ds.p, ds.n)).copy()
    names = [ds.names[j].decode() for j in range(ds.p)]
    return names, values


class _NativeDataset:
    """A mine_b200_dataset built from Python names / values (kept alive here)."""

    def __init__(self, names, values):
        self.values = _f64(values)
        if self.values.ndim != 2 or len(names) != self.values.shape[0]:
            raise ValueError("dataset: one name per variable row expected")
        self._names = (ctypes.c_char_p * len(names))(*[str(s).encode() for s in names])
        self.ds = MineDataset(self.values.shape[0], self.values.shape[1],
                              self.values.ctypes.data_as(_dp), self._names)


def read_dataset(path: str) -> tuple[list[str], np.ndarray]:
    """mine::read_dataset (io.cpp:48-120), host-only: (names, p x n values).
    Raises MineError with the reference's message on a malformed file."""
    L = load_library()
    out = ctypes.POINTER(MineDataset)()
    if L.mine_b200_read_dataset(str(path).encode(), ctypes.byref(out)) != 0:
        raise MineError(L.mine_b200_last_error().decode())
    try:
        return _dataset_to_py(out)
    finally:
        L.mine_b200_free_dataset(out)


def exported_symbols() -> list[str]:
    """Entry points declared in include/mine_b200.h (checked by the CPU tests)."""
    hdr = os.path.join(os.path.dirname(_PKG), "include", "mine_b200.h")
    import re
    names = []
    for m in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b(mine_\w+)\s*\(", open(hdr).read(), re.M):
        names.append(m.group(1))
    return sorted(set(names))


# ---------------------------------------------------------------------------
@dataclass
class Parameters:
    """mine::Parameters (char_matrix.hpp:11-14) plus the est extension."""
    alpha: float = 0.6
    c: float = 15.0
    est: int = MIC_APPROX

    def _c(self) -> MineParameter:
        return MineParameter(float(self.alpha), float(self.c), int(self.est))


def validate_parameters(params: Parameters) -> None:
    """char_matrix.cpp:11-15 -- raises MineError."""
    if not (params.alpha > 0.0) or params.alpha > 1.0:
        raise MineError("parameters: alpha must be in (0, 1]")
    if not (params.c > 0.0):
        raise MineError("parameters: c must be > 0")
    if params.est not in (MIC_APPROX, MIC_E):
        raise MineError("parameters: est must be MIC_APPROX or MIC_E")


def grid_bound(n: int, alpha: float) -> int:
    """char_matrix.cpp:17-20 (pure arithmetic, host side)."""
    return max(int(math.floor(math.pow(float(n), alpha))), 4)


def cell_shapes(bound: int) -> list[tuple[int, int]]:
    """(x, y) in for_each order, char_matrix.hpp:43-47."""
    return [(x, y) for y in range(2, bound // 2 + 1) for x in range(2, bound // y + 1)]


class CharacteristicMatrix:
    """mine::CharacteristicMatrix (char_matrix.hpp:25-49), built from the GPU's
    per-orientation cells.  entry(x, y) = max of the two orientations
    (update_max, char_matrix.cpp:28-35)."""

    def __init__(self, bound: int, o1: np.ndarray, o2: np.ndarray):
        self._bound = bound
        self.shapes = cell_shapes(bound)
        self.o1 = np.asarray(o1, dtype=np.float64)
        self.o2 = np.asarray(o2, dtype=np.float64)
        self.cells = np.where(self.o2 > self.o1, self.o2, self.o1)
        self._index = {s: i for i, s in enumerate(self.shapes)}

    def bound(self) -> int:
        return self._bound

    def max_row_target(self) -> int:
        return self._bound // 2

    def max_col_target(self, y: int) -> int:
        return self._bound // y

    def contains(self, x: int, y: int) -> bool:
        return x >= 2 and y >= 2 and x * y <= self._bound

    def entry(self, x: int, y: int) -> float:
        return float(self.cells[self._index[(x, y)]])

    def for_each(self):
        for (x, y), v in zip(self.shapes, self.cells):
            yield x, y, float(v)

    def equicharacteristic(self) -> np.ndarray:
        """Extension: E(x,y) = O1 if x<y, O2 if x>y, max if x==y."""
        return np.array([a if x < y else (b if x > y else m) for (x, y), a, b, m in
                         zip(self.shapes, self.o1, self.o2, self.cells)])


# ---------------------------------------------------------------------------
def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


class Engine:
    """One engine context (device buffers, cached tables, streams) on one GPU."""

    def __init__(self, device: int = 0):
        self.L = load_library()
        self.ctx = self.L.mine_b200_create(device)
        if not self.ctx:
            raise RuntimeError("mine_b200_create failed: " + self.L.mine_b200_last_error().decode())
        self.device = device
        self.count_work = False  # batch calls fill last_work (instrumented pass)
        self._cnt = None

    def close(self):
        if getattr(self, "ctx", None):
            self.L.mine_b200_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != 0:
            raise MineError(self.L.mine_b200_last_error().decode())

    def sync(self) -> None:
        """Waits for the last call; raises if an async device-io call's
        inputs were not finite (mine_b200_sync)."""
        self._check(self.L.mine_b200_sync(self.ctx))

    @property
    def last_launches(self) -> int:
        return int(self.L.mine_b200_last_launches(self.ctx))

    # -- output plumbing ----------------------------------------------------
    @staticmethod
    def _outputs(count: int, stats, cells: bool, bound: int | None):
        unknown = set(stats) - set(ALL_STATS)
        if unknown:
            raise ValueError(f"unknown statistics {sorted(unknown)}")
        res = {k: np.empty(count) for k in stats}
        so = MineStatsOut()
        for k in ALL_STATS:
            setattr(so, k, res[k].ctypes.data_as(_dp) if k in res else None)
        if cells:
            nc = len(cell_shapes(bound))
            res["cells"] = np.empty((count, 2, nc))
            so.cells = res["cells"].ctypes.data_as(_dp)
        return res, so

    @staticmethod
    def _count(total: int, first: int, count: int | None) -> int:
        """Items of [first, first + count) to score; an explicit 0 is an
        empty range (never passed to the C ABI, where count <= 0 means all)."""
        if not 0 <= first <= total:
            raise MineError("expand_pairs: first index out of range")
        count = total - first if count is None else int(count)
        if count < 0 or first + count > total:
            raise MineError("expand_pairs: pair range out of range")
        return count

    def _opts(self, first=0, count=0, tier=0, reuse_vars=False, devices=None,
              shard_chunk=0) -> MineOpts:
        o = MineOpts()
        o.first, o.count, o.tier = int(first), int(count), int(tier)
        o.reuse_vars = int(bool(reuse_vars))
        if devices is not None and len(devices) > 0:
            self._devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
            o.ndevices, o.devices, o.shard_chunk = len(devices), self._devs, int(shard_chunk)
        if self.count_work:
            self._cnt = (ctypes.c_ulonglong * NCOUNTERS)()
            o.counters = self._cnt
        return o

    @property
    def last_work(self) -> dict | None:
        """Realised-work totals of the last batch call made with
        `count_work = True` (an instrumented, synchronising pass)."""
        return dict(zip(COUNTERS, list(self._cnt))) if self._cnt is not None else None

    # -- batch calls ----------------------------------------------------------
    def pairwise(self, vars_, params: Parameters = Parameters(), first: int = 0, count: int | None = None,
                 stats=STATS, cells: bool = False, tier: int = 0, reuse_vars: bool = False,
                 devices=None, shard_chunk: int = 0):
        """All pairs i<j in PairSequence order (analysis.cpp:66-81).
        reuse_vars: `vars_` is the same array as in the previous call (e.g. the
        next window of one job): skip the per-variable stages.
        devices: a list of CUDA devices (repeats allowed) to spread the call
        over (mine_b200_opts.ndevices / devices / shard_chunk)."""
        v = _f64(vars_)
        p, n = v.shape
        total = p * (p - 1) // 2
        count = self._count(total, first, count)
        res, so = self._outputs(count, stats, cells, grid_bound(n, params.alpha))
        if count == 0:  # the C ABI reads count <= 0 as "all from first"
            return res
        self._check(self.L.mine_b200_pairwise(self.ctx, _ptr(v), p, n, ctypes.byref(params._c()),
                                              ctypes.byref(self._opts(first, count, tier, reuse_vars,
                                                                      devices, shard_chunk)),
                                              ctypes.byref(so)))
        return res

    def cross(self, X, Y, params: Parameters = Parameters(), stats=STATS, cells: bool = False,
              tier: int = 0, first: int = 0, count: int | None = None, reuse_vars: bool = False,
              devices=None, shard_chunk: int = 0):
        X, Y = _f64(X), _f64(Y)
        if X.shape[1] != Y.shape[1]:
            raise MineError("compute_score: input lengths differ")
        total = X.shape[0] * Y.shape[0]
        count = self._count(total, first, count)
        res, so = self._outputs(count, stats, cells, grid_bound(X.shape[1], params.alpha))
        if count == 0:
            return res
        self._check(self.L.mine_b200_cross(self.ctx, _ptr(X), X.shape[0], _ptr(Y), Y.shape[0],
                                           X.shape[1], ctypes.byref(params._c()),
                                           ctypes.byref(self._opts(first, count, tier, reuse_vars,
                                                                   devices, shard_chunk)),
                                           ctypes.byref(so)))
        return res

    def pairs(self, vars_, xi, yi, params: Parameters = Parameters(), stats=STATS,
              cells: bool = False, tier: int = 0, reuse_vars: bool = False, devices=None,
              shard_chunk: int = 0):
        v = _f64(vars_)
        xi = np.ascontiguousarray(xi, dtype=np.int32)
        yi = np.ascontiguousarray(yi, dtype=np.int32)
        if xi.shape != yi.shape:
            raise MineError("expand_pairs: index arrays differ in length")
        res, so = self._outputs(xi.size, stats, cells, grid_bound(v.shape[1], params.alpha))
        if xi.size == 0:
            return res
        self._check(self.L.mine_b200_pairs(self.ctx, _ptr(v), v.shape[0], v.shape[1], _ptr(xi),
                                           _ptr(yi), xi.size, ctypes.byref(params._c()),
                                           ctypes.byref(self._opts(0, xi.size, tier, reuse_vars,
                                                                   devices, shard_chunk)),
                                           ctypes.byref(so)))
        return res

    def master_vs_all(self, vars_, master: int, params: Parameters = Parameters(), stats=STATS,
                      tier: int = 0, reuse_vars: bool = False):
        """AnalysisMode::master_vs_all (analysis.cpp:25-30, PairSequence::at
        :82-85): the pairs (master, j) for every j != master in index order,
        each oriented lower index first (score_pair, :117-129).  `master` is
        0-based here.  With reuse_vars=True over the same `vars_` array, the
        per-variable stages run once for a whole sweep of masters (SURVEY 8f
        rank 1)."""
        v = _f64(vars_)
        p = v.shape[0]
        if not 0 <= master < p:
            raise MineError("expand_pairs: master index out of range")
        others = np.array([j for j in range(p) if j != master], dtype=np.int32)
        xi = np.minimum(others, master).astype(np.int32)
        yi = np.maximum(others, master).astype(np.int32)
        res, so = self._outputs(xi.size, stats, False, grid_bound(v.shape[1], params.alpha))
        self._check(self.L.mine_b200_pairs(self.ctx, _ptr(v), p, v.shape[1], _ptr(xi), _ptr(yi),
                                           xi.size, ctypes.byref(params._c()),
                                           ctypes.byref(self._opts(0, xi.size, tier, reuse_vars)),
                                           ctypes.byref(so)))
        return res

    # -- analysis front end (io.cpp / analysis.cpp) ----------------------------
    def variances(self, vars_) -> np.ndarray:
        """Per-variable sample variance on the GPU (analysis.cpp:98-100)."""
        v = _f64(vars_)
        out = np.empty(v.shape[0])
        self._check(self.L.mine_b200_variances(self.ctx, _ptr(v), v.shape[0], v.shape[1],
                                               out.ctypes.data_as(_dp)))
        return out

    def filter_low_variance(self, names, values, threshold: float):
        """filter_low_variance (analysis.cpp:92-113): (names, values) kept."""
        src = _NativeDataset(names, values)
        out = ctypes.POINTER(MineDataset)()
        self._check(self.L.mine_b200_filter_low_variance(self.ctx, ctypes.byref(src.ds),
                                                         float(threshold), ctypes.byref(out)))
        try:
            return _dataset_to_py(out)
        finally:
            self.L.mine_b200_free_dataset(out)

    def run_analysis(self, names, values, out_path: str, mode: str = "all_pairs",
                     master: int = 0, first: int = 0, second: int = 0,
                     params: Parameters = Parameters(), min_variance: float | None = None,
                     workers: int = 0) -> int:
        """run_analysis + write_results (analysis.cpp:133-191, io.cpp:122-154):
        writes the results file the reference's CLI writes (1-based indices
        as AnalysisTask).  Returns the record count."""
        src = _NativeDataset(names, values)
        t = MineTask(MODES[mode], int(master), int(first), int(second), float(params.alpha),
                     float(params.c), int(min_variance is not None),
                     float(min_variance if min_variance is not None else 0.0),
                     int(workers or os.cpu_count() or 1))
        rc = self.L.mine_b200_run_analysis(self.ctx, ctypes.byref(src.ds), ctypes.byref(t),
                                           str(out_path).encode())
        if rc < 0:
            raise MineError(self.L.mine_b200_last_error().decode())
        return int(rc)

    def pairwise_device(self, vars_ptr: int, p: int, n: int, params: Parameters, out_ptrs: dict,
                        stream: int = 0, first: int = 0, count: int = 0, tier: int = 0,
                        async_: bool = True, counters: bool = False, ev_begin: int = 0,
                        ev_end: int = 0):
        """Device-resident variant (torch tensors' data_ptr()s): inputs and
        outputs in HBM, enqueued on `stream`.  counters=True returns the
        realised-work totals (synchronises)."""
        so = MineStatsOut()
        for k in ALL_STATS:
            setattr(so, k, ctypes.cast(ctypes.c_void_p(out_ptrs[k]), _dp) if out_ptrs.get(k) else None)
        o = MineOpts()
        o.first, o.count, o.tier = int(first), int(count), int(tier)
        o.device_io, o.async_, o.stream = 1, int(async_), ctypes.c_void_p(stream)
        cnt = (ctypes.c_ulonglong * NCOUNTERS)()
        if counters:
            o.counters = cnt
        o.ev_begin, o.ev_end = ctypes.c_void_p(ev_begin or None), ctypes.c_void_p(ev_end or None)
        self._check(self.L.mine_b200_pairwise(self.ctx, ctypes.c_void_p(vars_ptr), p, n,
                                              ctypes.byref(params._c()), ctypes.byref(o),
                                              ctypes.byref(so)))
        return dict(zip(COUNTERS, list(cnt))) if counters else None

    def device_call(self, kind: str, params: Parameters, out_ptrs: dict, *, vars_ptr: int = 0,
                    p: int = 0, n: int = 0, y_ptr: int = 0, py: int = 0, xi_ptr: int = 0,
                    yi_ptr: int = 0, npairs: int = 0, stream: int = 0, first: int = 0,
                    count: int = 0, counters: bool = False, ev_begin: int = 0, ev_end: int = 0,
                    reuse_vars: bool = False):
        """Any batch call with device-resident inputs / outputs (data_ptr()s):
        kind = "pairwise" (vars p x n), "cross" (X = vars p x n, Y = y_ptr
        py x n) or "pairs" (vars p x n, device index arrays xi / yi of
        npairs).  Synchronous; counters=True returns the realised work."""
        so = MineStatsOut()
        for k in ALL_STATS:
            setattr(so, k, ctypes.cast(ctypes.c_void_p(out_ptrs[k]), _dp) if out_ptrs.get(k) else None)
        o = MineOpts()
        o.first, o.count, o.tier = int(first), int(count), 0
        o.device_io, o.async_, o.stream = 1, 0, ctypes.c_void_p(stream or None)
        o.reuse_vars = int(bool(reuse_vars))
        cnt = (ctypes.c_ulonglong * NCOUNTERS)()
        if counters:
            o.counters = cnt
        o.ev_begin, o.ev_end = ctypes.c_void_p(ev_begin or None), ctypes.c_void_p(ev_end or None)
        par = ctypes.byref(params._c())
        vp = ctypes.c_void_p
        if kind == "pairwise":
            rc = self.L.mine_b200_pairwise(self.ctx, vp(vars_ptr), p, n, par, ctypes.byref(o),
                                           ctypes.byref(so))
        elif kind == "cross":
            rc = self.L.mine_b200_cross(self.ctx, vp(vars_ptr), p, vp(y_ptr), py, n, par,
                                        ctypes.byref(o), ctypes.byref(so))
        elif kind == "pairs":
            rc = self.L.mine_b200_pairs(self.ctx, vp(vars_ptr), p, n, vp(xi_ptr), vp(yi_ptr), npairs,
                                        par, ctypes.byref(o), ctypes.byref(so))
        else:
            raise ValueError(kind)
        self._check(rc)
        return dict(zip(COUNTERS, list(cnt))) if counters else None

    def pairwise_host(self, vars_np: np.ndarray, params: Parameters, outs: dict, first: int = 0,
                      count: int = 0):
        """The reference-facing call with HOST buffers (e2e leg): H2D of the
        variables, scoring, D2H of the requested statistics into `outs`
        (preallocated, ideally pinned, numpy arrays)."""
        so = MineStatsOut()
        for k in ALL_STATS:
            setattr(so, k, outs[k].ctypes.data_as(_dp) if k in outs else None)
        p, n = vars_np.shape
        self._check(self.L.mine_b200_pairwise(self.ctx, _ptr(vars_np), p, n, ctypes.byref(params._c()),
                                              ctypes.byref(self._opts(first, count)), ctypes.byref(so)))

    def debug_subproblem(self, col_var, row_var, y_target: int, x_max: int, k_hat: int):
        """GPU general-tier partition + DP of one (orientation, y) subproblem
        (the stage sequence of score_orientation, char_matrix.cpp:44-56)."""
        col_var, row_var = _f64(col_var), _f64(row_var)
        n = col_var.size
        rc, raw, k = (np.zeros(1, np.int32) for _ in range(3))
        qx = np.zeros(n, np.int32)
        bounds = np.zeros(n + 1, np.int32)
        hq = np.zeros(1)
        vals = np.zeros(max(x_max - 1, 1))
        self._check(self.L.mine_b200_debug_subproblem(
            self.ctx, n, col_var.ctypes.data_as(_dp), row_var.ctypes.data_as(_dp), y_target, x_max,
            k_hat, rc.ctypes.data_as(_ip), qx.ctypes.data_as(_ip), raw.ctypes.data_as(_ip),
            k.ctypes.data_as(_ip), bounds.ctypes.data_as(_ip), hq.ctypes.data_as(_dp),
            vals.ctypes.data_as(_dp)))
        return dict(row_count=int(rc[0]), q_x=qx, clump_count=int(raw[0]), k=int(k[0]),
                    bounds=bounds[: int(k[0]) + 1].copy(), h_q=float(hq[0]), values=vals[: x_max - 1])

    # -- single pair, the reference's signatures -----------------------------
    def compute_score(self, xs, ys, params: Parameters = Parameters(), tier: int = 0) -> CharacteristicMatrix:
        """mine::compute_score (char_matrix.cpp:70-81)."""
        xs, ys = _f64(xs), _f64(ys)
        if xs.shape != ys.shape:
            raise MineError("compute_score: input lengths differ")
        validate_parameters(params)
        if xs.size < 2:
            raise MineError("compute_score: need at least 2 samples")
        b = grid_bound(xs.size, params.alpha)
        res = self.pairs(np.stack([xs, ys]), [0], [1], params, stats=("mic",), cells=True, tier=tier)
        return CharacteristicMatrix(b, res["cells"][0, 0], res["cells"][0, 1])

    def compute_statistics(self, xs, ys, params: Parameters = Parameters(), tier: int = 0) -> dict:
        """mine::compute_statistics (statistics.cpp:53-63): MIC, MAS, MEV, MCN,
        pearson_r, nonlinearity, plus MIC_e and TIC."""
        xs, ys = _f64(xs), _f64(ys)
        if xs.shape != ys.shape:
            raise MineError("compute_score: input lengths differ")
        res = self.pairs(np.stack([xs, ys]), [0], [1], params, stats=ALL_STATS, tier=tier)
        return {k: float(v[0]) for k, v in res.items()}


_DEFAULT: Engine | None = None


def default_engine() -> Engine:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Engine(int(os.environ.get("MINE_B200_DEVICE", "0")))
    return _DEFAULT


def compute_score(xs, ys, params: Parameters = Parameters()) -> CharacteristicMatrix:
    return default_engine().compute_score(xs, ys, params)


def compute_statistics(xs, ys, params: Parameters = Parameters()) -> dict:
    return default_engine().compute_statistics(xs, ys, params)
