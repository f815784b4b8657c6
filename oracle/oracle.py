"""ctypes bindings for the TEST-ONLY oracles (never imported by the product).

* ``Oracle``    -- our plain-C restatement (oracle/mine_oracle.c), always built.
* ``Reference`` -- the reference's own C++ engine compiled unmodified against
  the Eigen shim (oracle/_ref/libmine_ref.so); exists only where it was built
  (this container, or a GPU box the prebuilt .so travelled to).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
ORACLE_SO = os.path.join(REF_DIR, "libmine_oracle.so")
REF_SO = os.path.join(REF_DIR, "libmine_ref.so")
REFERENCE_SRC = "/root/reference/proj"

MIC, MAS, MEV, MCN, MICE, TIC = range(6)
NSTAT = 6

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


def build(reference: bool = True, reference_tests: bool = False) -> None:
    """Build the C restatement, and the reference .so (plus, on request, the
    reference's own test binaries against the GPU adapter) when its sources
    exist."""
    subprocess.run(["make", "-s", "-C", HERE, os.path.join("_ref", "libmine_oracle.so")], check=True)
    if reference and os.path.isdir(REFERENCE_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
        if reference_tests:
            subprocess.run(["make", "-s", "-C", HERE, "ref-tests"], check=True)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _i(a: np.ndarray):
    return a.ctypes.data_as(_ip)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def grid_bound(n: int, alpha: float) -> int:
    """char_matrix.cpp:17-20 (pure arithmetic; mirrored here for the tests)."""
    import math
    return max(int(math.floor(math.pow(float(n), alpha))), 4)


def cell_shapes(bound: int):
    """(x, y) in for_each order (char_matrix.hpp:43-47)."""
    return [(x, y) for y in range(2, bound // 2 + 1) for x in range(2, bound // y + 1)]


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(reference=False)
        L = ctypes.CDLL(path)
        L.mo_grid_bound.argtypes = [ctypes.c_long, ctypes.c_double]
        L.mo_cell_count.argtypes = [ctypes.c_int]
        L.mo_compute_score.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_double, ctypes.c_double,
                                       _dp, _dp, _dp]
        L.mo_reduce.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_int, _dp]
        L.mo_reduce.restype = None
        L.mo_statistics.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_int, _dp]
        L.mo_subproblem.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    _ip, _ip, _ip, _ip, _ip, _dp, _dp]
        L.mo_optimize_x_axis.argtypes = [_ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.mo_pairwise.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_long, ctypes.c_long, _dp]
        L.mo_cross.argtypes = [_dp, ctypes.c_int, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                               ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp]
        L.mo_pairs.argtypes = [_dp, ctypes.c_int, _ip, _ip, ctypes.c_long, ctypes.c_double,
                               ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp]
        L.mo_pearson.argtypes = [ctypes.c_int, _dp, _dp, _dp]
        L.mo_pair_at.argtypes = [ctypes.c_long, ctypes.c_long, _ip, _ip]
        L.mo_pair_at.restype = None
        L.mo_last_error.restype = ctypes.c_char_p
        self.L = L

    def _check(self, rc):
        if rc < 0:
            raise ValueError(self.L.mo_last_error().decode())
        return rc

    def grid_bound(self, n, alpha):
        return self.L.mo_grid_bound(n, alpha)

    def score(self, x, y, alpha=0.6, c=15.0):
        """Returns (bound, o1, o2, m) -- per-orientation and merged cells."""
        x, y = _f64(x), _f64(y)
        if x.shape != y.shape:
            raise ValueError("compute_score: input lengths differ")
        n = x.size
        b = grid_bound(n, alpha) if n >= 2 else 4
        cells = self.L.mo_cell_count(b)
        o1, o2, m = (np.zeros(cells) for _ in range(3))
        self._check(self.L.mo_compute_score(n, _d(x), _d(y), alpha, c, _d(o1), _d(o2), _d(m)))
        return b, o1, o2, m

    def statistics(self, x, y, alpha=0.6, c=15.0, est=0):
        x, y = _f64(x), _f64(y)
        if x.shape != y.shape:
            raise ValueError("compute_score: input lengths differ")
        out = np.zeros(NSTAT)
        self._check(self.L.mo_statistics(x.size, _d(x), _d(y), alpha, c, est, _d(out)))
        return out

    def pearson(self, x, y):
        """statistics.cpp:39-49 (NaN for a zero-variance input)."""
        x, y = _f64(x), _f64(y)
        if x.shape != y.shape:
            raise ValueError("pearson: input lengths differ")
        r = np.zeros(1)
        self._check(self.L.mo_pearson(x.size, _d(x), _d(y), _d(r)))
        return float(r[0])

    def reduce(self, bound, o1, o2, est=0):
        out = np.zeros(NSTAT)
        self.L.mo_reduce(bound, _d(_f64(o1)), _d(_f64(o2)), est, _d(out))
        return out

    def subproblem(self, col_var, row_var, y_target, x_max, k_hat):
        col_var, row_var = _f64(col_var), _f64(row_var)
        n = col_var.size
        rc, raw, k = (np.zeros(1, np.int32) for _ in range(3))
        qx = np.zeros(n, np.int32)
        bounds = np.zeros(n + 1, np.int32)
        hq = np.zeros(1)
        vals = np.zeros(max(x_max - 1, 1))
        self._check(self.L.mo_subproblem(n, _d(col_var), _d(row_var), y_target, x_max, k_hat,
                                         _i(rc), _i(qx), _i(raw), _i(k), _i(bounds), _d(hq), _d(vals)))
        return dict(row_count=int(rc[0]), q_x=qx, clump_count=int(raw[0]), k=int(k[0]),
                    bounds=bounds[: int(k[0]) + 1].copy(), h_q=float(hq[0]), values=vals[: x_max - 1])

    def optimize_x_axis(self, counts, x):
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        rows, k = counts.shape
        vals = np.zeros(max(x - 1, 1))
        hq = np.zeros(1)
        self._check(self.L.mo_optimize_x_axis(_i(counts), rows, k, x, _d(vals), _d(hq)))
        return vals[: x - 1], float(hq[0])

    def pairwise(self, vars_, alpha=0.6, c=15.0, est=0, threads=0, first=0, count=None):
        vars_ = _f64(vars_)
        p, n = vars_.shape
        total = p * (p - 1) // 2
        count = total - first if count is None else count
        out = np.zeros((count, NSTAT))
        threads = threads or os.cpu_count() or 1
        self._check(self.L.mo_pairwise(_d(vars_), p, n, alpha, c, est, threads, first, count, _d(out)))
        return out

    def cross(self, X, Y, alpha=0.6, c=15.0, est=0, threads=0):
        X, Y = _f64(X), _f64(Y)
        out = np.zeros((X.shape[0] * Y.shape[0], NSTAT))
        threads = threads or os.cpu_count() or 1
        self._check(self.L.mo_cross(_d(X), X.shape[0], _d(Y), Y.shape[0], X.shape[1], alpha, c, est,
                                    threads, _d(out)))
        return out

    def pairs(self, vars_, xi, yi, alpha=0.6, c=15.0, est=0, threads=0):
        vars_ = _f64(vars_)
        xi = np.ascontiguousarray(xi, dtype=np.int32)
        yi = np.ascontiguousarray(yi, dtype=np.int32)
        out = np.zeros((xi.size, NSTAT))
        threads = threads or os.cpu_count() or 1
        self._check(self.L.mo_pairs(_d(vars_), vars_.shape[1], _i(xi), _i(yi), xi.size, alpha, c, est,
                                    threads, _d(out)))
        return out

    def pair_at(self, p, w):
        i = np.zeros(1, np.int32)
        j = np.zeros(1, np.int32)
        self.L.mo_pair_at(p, w, _i(i), _i(j))
        return int(i[0]), int(j[0])


class Reference:
    """The reference engine itself (unmodified sources + Eigen shim)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs {REFERENCE_SRC} at build time)")
        L = ctypes.CDLL(path)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_grid_bound.argtypes = [ctypes.c_long, ctypes.c_double]
        L.ref_compute_score.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_double, ctypes.c_double, _ip, _dp]
        L.ref_compute_statistics.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_double, ctypes.c_double, _dp]
        L.ref_reference_statistics.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_double, ctypes.c_double, _dp]
        L.ref_run_analysis.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_uint,
                                       _dp, ctypes.POINTER(ctypes.c_long)]
        L.ref_subproblem.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     _ip, _ip, _ip, _ip, _ip, _dp, _dp]
        L.ref_equipartition.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_int, _ip, _ip]
        L.ref_clumps.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_int, ctypes.c_int, _ip, _ip]
        L.ref_optimize_x_axis.argtypes = [_ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.ref_brute_force.argtypes = [_ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp,
                                      ctypes.POINTER(ctypes.c_longlong)]
        L.ref_entropy.argtypes = [_dp, ctypes.c_int, _dp]
        L.ref_analysis_file.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_uint, ctypes.POINTER(ctypes.c_long)]
        L.ref_read_dataset.argtypes = [ctypes.c_char_p, _ip, _ip, _dp, ctypes.c_long, ctypes.c_char_p,
                                       ctypes.c_long]
        L.ref_filter_low_variance.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, _ip, _ip]
        self.L = L

    def _check(self, rc):
        if rc < 0:
            raise ValueError(self.L.ref_last_error().decode())
        return rc

    def score(self, x, y, alpha=0.6, c=15.0):
        x, y = _f64(x), _f64(y)
        if x.shape != y.shape:
            raise ValueError("compute_score: input lengths differ")
        n = x.size
        b = grid_bound(n, alpha)
        cells = np.zeros(max(len(cell_shapes(b)), 1))
        bound = np.zeros(1, np.int32)
        self._check(self.L.ref_compute_score(n, _d(x), _d(y), alpha, c, _i(bound), _d(cells)))
        return int(bound[0]), cells[: len(cell_shapes(b))]

    def statistics(self, x, y, alpha=0.6, c=15.0):
        """mic, mas, mev, mcn, pearson_r, nonlinearity."""
        x, y = _f64(x), _f64(y)
        if x.shape != y.shape:
            raise ValueError("compute_score: input lengths differ")
        out = np.zeros(6)
        self._check(self.L.ref_compute_statistics(x.size, _d(x), _d(y), alpha, c, _d(out)))
        return out

    def cache_free_statistics(self, x, y, alpha=0.6, c=15.0):
        x, y = _f64(x), _f64(y)
        out = np.zeros(6)
        self._check(self.L.ref_reference_statistics(x.size, _d(x), _d(y), alpha, c, _d(out)))
        return out

    def run_analysis(self, vars_, alpha=0.6, c=15.0, workers=1, mode=0, a=0, b=0):
        vars_ = _f64(vars_)
        p, n = vars_.shape
        cap = p * (p - 1) // 2 if mode == 0 else (p - 1 if mode == 1 else 1)
        out = np.zeros((max(cap, 1), 6))
        rec = ctypes.c_long(0)
        self._check(self.L.ref_run_analysis(_d(vars_), p, n, mode, a, b, alpha, c, workers, _d(out),
                                            ctypes.byref(rec)))
        return out[: rec.value]

    def subproblem(self, col_var, row_var, y_target, x_max, k_hat):
        col_var, row_var = _f64(col_var), _f64(row_var)
        n = col_var.size
        rc, raw, k = (np.zeros(1, np.int32) for _ in range(3))
        qx = np.zeros(n, np.int32)
        bounds = np.zeros(n + 1, np.int32)
        hq = np.zeros(1)
        vals = np.zeros(max(x_max - 1, 1))
        self._check(self.L.ref_subproblem(n, _d(col_var), _d(row_var), y_target, x_max, k_hat,
                                          _i(rc), _i(qx), _i(raw), _i(k), _i(bounds), _d(hq), _d(vals)))
        return dict(row_count=int(rc[0]), q_x=qx, clump_count=int(raw[0]), k=int(k[0]),
                    bounds=bounds[: int(k[0]) + 1].copy(), h_q=float(hq[0]), values=vals[: x_max - 1])

    def equipartition(self, x, y, y_target):
        x, y = _f64(x), _f64(y)
        rows = np.zeros(x.size, np.int32)
        rc = np.zeros(1, np.int32)
        self._check(self.L.ref_equipartition(x.size, _d(x), _d(y), y_target, _i(rows), _i(rc)))
        return rows, int(rc[0])

    def clumps(self, x, y, y_target, k_hat=0):
        x, y = _f64(x), _f64(y)
        cols = np.zeros(x.size, np.int32)
        k = np.zeros(1, np.int32)
        self._check(self.L.ref_clumps(x.size, _d(x), _d(y), y_target, k_hat, _i(cols), _i(k)))
        return cols, int(k[0])

    def optimize_x_axis(self, counts, x):
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        rows, k = counts.shape
        vals = np.zeros(max(x - 1, 1))
        hq = np.zeros(1)
        self._check(self.L.ref_optimize_x_axis(_i(counts), rows, k, x, _d(vals), _d(hq)))
        return vals[: x - 1], float(hq[0])

    def brute_force(self, counts, x):
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        rows, k = counts.shape
        vals = np.zeros(max(x - 1, 1))
        e = ctypes.c_longlong(0)
        self._check(self.L.ref_brute_force(_i(counts), rows, k, x, _d(vals), ctypes.byref(e)))
        return vals[: x - 1], e.value

    def entropy(self, w):
        w = _f64(w)
        out = np.zeros(1)
        self._check(self.L.ref_entropy(_d(w), w.size, _d(out)))
        return float(out[0])


def _ref_methods():
    """File-level front end of the reference (io.cpp / analysis.cpp)."""

    def analysis_file(self, in_path, out_path, mode=0, a=0, b=0, alpha=0.6, c=15.0,
                      min_variance=None, workers=4):
        """read_dataset -> run_analysis -> ResultWriter, as run_cli does."""
        rec = ctypes.c_long(0)
        self._check(self.L.ref_analysis_file(str(in_path).encode(), str(out_path).encode(), mode, a, b,
                                             alpha, c, -1.0 if min_variance is None else min_variance,
                                             workers, ctypes.byref(rec)))
        return rec.value

    def read_dataset(self, path):
        p, n = np.zeros(1, np.int32), np.zeros(1, np.int32)
        self._check(self.L.ref_read_dataset(str(path).encode(), _i(p), _i(n), None, 0, None, 0))
        vals = np.zeros(int(p[0]) * int(n[0]))
        buf = ctypes.create_string_buffer(1 << 22)
        self._check(self.L.ref_read_dataset(str(path).encode(), _i(p), _i(n), _d(vals), vals.size,
                                            buf, len(buf)))
        names = buf.value.decode().split("\n")[:-1]
        return names, vals.reshape(int(p[0]), int(n[0]))

    def filter_low_variance(self, values, threshold):
        v = _f64(values)
        keep = np.zeros(v.shape[0], np.int32)
        nk = np.zeros(1, np.int32)
        self._check(self.L.ref_filter_low_variance(_d(v), v.shape[0], v.shape[1], threshold,
                                                   _i(keep), _i(nk)))
        return keep[: int(nk[0])]

    Reference.analysis_file = analysis_file
    Reference.read_dataset = read_dataset
    Reference.filter_low_variance = filter_low_variance


_ref_methods()
