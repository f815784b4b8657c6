"""CPU: pin the oracle (oracle/mine_oracle.c, our restatement) against the
reference's own golden vectors / known-answer tests and against the reference
engine itself (oracle/_ref, compiled from /root/reference/proj/src).

Test names cite the reference test each one follows."""
import math
import os

import numpy as np
import pytest

from conftest import bits, random_pair

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# Fig. 2 worked example (test_helpers.hpp:26-40).
FIG2_X = np.array([1, 1, 1, 1, 2, 2, 3, 4, 5, 6, 7, 8, 9, 9], float)
FIG2_Y = np.array([1, 2, 3, 4, 3, 4, 5, 6, 6, 6, 5, 3, 2, 1], float)
FIG2_Q = [1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 3, 2, 1, 1]
FIG2_P = [1, 1, 1, 1, 2, 2, 3, 3, 3, 3, 3, 4, 5, 5]


def _per_point(assign_sorted, x, y, key):
    """Carry ordinals from a sorted order back to point order (the stable
    (a,b) sort of partition.cpp:13-38)."""
    order = sorted(range(len(x)), key=(lambda i: (x[i], y[i])) if key == 0 else (lambda i: (y[i], x[i])))
    out = [0] * len(x)
    for pos, i in enumerate(order):
        out[i] = assign_sorted[pos]
    return out


# --- KATs from the reference's tests -----------------------------------------
def test_grid_bound_kats(oracle):
    """test_char_matrix.cpp:14-19."""
    assert oracle.grid_bound(1001, 0.6) == 63
    assert oracle.grid_bound(4, 0.6) == 4
    assert oracle.grid_bound(100, 1.0) == 100
    assert oracle.grid_bound(2, 0.3) == 4


def test_fig2_rows_and_clumps(oracle):
    """test_partition.cpp:61-69 (Q), :128-139 (P); acceptance.cpp:322-344."""
    d = oracle.subproblem(FIG2_X, FIG2_Y, 3, 2, 100)
    assert d["row_count"] == 3 and d["clump_count"] == 5 and d["k"] == 5
    # row labels in x-sorted order back to point order
    qx = _per_point(list(d["q_x"]), FIG2_X, FIG2_Y, 0)
    assert qx == FIG2_Q
    # clump ordinal of each x-sorted position from the boundaries
    clump = np.searchsorted(d["bounds"][1:], np.arange(14), side="right") + 1
    assert _per_point(list(clump), FIG2_X, FIG2_Y, 0) == FIG2_P


def test_fig2_superclumps_k3(oracle):
    """test_partition.cpp:193-206: budget 3 -> (1,1,1,1,2,2,2,2,2,2,2,3,3,3)."""
    d = oracle.subproblem(FIG2_X, FIG2_Y, 3, 2, 3)
    assert d["k"] == 3 and list(d["bounds"]) == [0, 4, 11, 14]


def test_fig2_cell_counts(oracle):
    """test_mutual_info.cpp:50-68 -- via the DP input: the cumulative counts
    at the boundaries reproduce the per-clump row histogram."""
    d = oracle.subproblem(FIG2_X, FIG2_Y, 3, 2, 100)
    qx = np.array(d["q_x"])
    b = d["bounds"]
    counts = np.array([[np.sum(qx[b[j]:b[j + 1]] == r) for j in range(5)] for r in (1, 2, 3)])
    assert counts.tolist() == [[2, 0, 0, 0, 2], [2, 2, 0, 1, 0], [0, 0, 5, 0, 0]]


def test_entropy_kats(reference):
    """test_mutual_info.cpp:12-29."""
    assert abs(reference.entropy([1, 1]) - math.log(2)) <= 1e-12 * math.log(2)
    assert reference.entropy([5]) == 0.0
    want = -(0.25 * math.log(0.25) + 0.75 * math.log(0.75))
    assert abs(reference.entropy([1, 3]) - want) <= 1e-14 * want
    assert abs(reference.entropy([2, 0, 2]) - math.log(2)) <= 1e-12


def test_dp_kats(oracle):
    """test_mutual_info.cpp:113-138."""
    v, hq = oracle.optimize_x_axis(np.array([[2, 0], [0, 2]]), 2)
    assert abs(v[0] - math.log(2)) <= 1e-14 and abs(hq - math.log(2)) <= 1e-14
    v, _ = oracle.optimize_x_axis(np.array([[4], [3], [5]]), 6)
    assert (v == 0.0).all() and v.size == 5
    v, _ = oracle.optimize_x_axis(np.array([[3, 0, 1], [0, 2, 2]]), 6)
    assert v[2] == v[1] and v[3] == v[1] and v[4] == v[1]


def test_dp_equals_brute_force(oracle, reference):
    """test_oracle.cpp:62-72 / acceptance.cpp:189-228: the DP restatement
    agrees with the reference's exhaustive enumeration to 1e-12."""
    rng = np.random.default_rng(92)
    worst = 0.0
    for _ in range(300):
        rows, k = int(rng.integers(1, 5)), int(rng.integers(1, 9))
        counts = np.zeros((rows, k), np.int32)
        for j in range(k):
            for _ in range(1 + int(rng.integers(0, max(1, (40 - k) // k) + 1))):
                counts[int(rng.integers(0, rows)), j] += 1
        x = int(rng.integers(2, 7))
        dp, _ = oracle.optimize_x_axis(counts, x)
        bf, _ = reference.brute_force(counts, x)
        worst = max(worst, float(np.max(np.abs(dp - bf))))
    assert worst <= 1e-12


def test_identity_and_constant(oracle):
    """test_statistics.cpp:41-60; test_char_matrix.cpp:54-76."""
    x = np.arange(100.0)
    s = oracle.statistics(x, x)
    assert s[0] == 1.0 and s[1] == 0.0 and s[2] == 1.0 and s[3] == 2.0
    s = oracle.statistics(np.arange(40.0), np.full(40, 2.0))
    assert s[0] == 0.0 and s[3] == 2.0
    b, o1, o2, m = oracle.score(np.arange(50.0), np.full(50, 3.25))
    assert (m == 0.0).all()


def test_sine_golden(oracle):
    """acceptance.cpp:62-92."""
    n = 1001
    x = np.arange(n) / (n - 1)
    y = np.sin(10 * np.pi * x) + x
    s = oracle.statistics(x, y)
    assert abs(s[0] - 0.999999) <= 1e-3 and abs(s[2] - 0.999999) <= 1e-3
    assert abs(s[3] - 4.584963) <= 1e-3 and abs(s[1] - 0.728144) <= 0.02


def test_transposition_and_swap_invariance(oracle):
    """test_char_matrix.cpp:89-97, test_statistics.cpp:114-132."""
    rng = np.random.default_rng(12)
    for it in range(20):
        x, y = random_pair(rng, 40 + it, it % 4)
        b, _, _, m = oracle.score(x, y)
        _, _, _, t = oracle.score(y, x)
        shapes = [(xx, yy) for yy in range(2, b // 2 + 1) for xx in range(2, b // yy + 1)]
        idx = {s: i for i, s in enumerate(shapes)}
        for (xx, yy), i in idx.items():
            assert m[i] == t[idx[(yy, xx)]]
        sa, sb = oracle.statistics(x, y), oracle.statistics(y, x)
        assert (sa[:5] == sb[:5]).all()


def test_c_saturation(oracle):
    """test_char_matrix.cpp:111-121: a saturated clump budget no longer
    changes any entry."""
    rng = np.random.default_rng(14)
    for it in range(10):
        x, y = random_pair(rng, 60, it % 4)
        _, _, _, a = oracle.score(x, y, 0.6, 60.0)
        _, _, _, b = oracle.score(x, y, 0.6, 3 * 60 + 7.5)
        assert (bits(a) == bits(b)).all()


def test_validation(oracle):
    """test_char_matrix.cpp:123-137."""
    with pytest.raises(ValueError):
        oracle.statistics([1, 2, 3, 4], [1, 2, 3])
    with pytest.raises(ValueError):
        oracle.statistics([1.0], [2.0])
    with pytest.raises(ValueError):
        oracle.statistics([1, 2, 3, 4], [1, 2, np.nan, 4])
    with pytest.raises(ValueError):
        oracle.statistics([1, 2, 3, 4], [1, 2, 3, 4], 0.6, -1.0)


# --- the restatement against the reference engine itself --------------------
@pytest.mark.parametrize("style", range(4))
def test_oracle_matches_reference_bit_exact(oracle, reference, style):
    rng = np.random.default_rng(100 + style)
    for it in range(40):
        n = int(rng.integers(2, 220))
        alpha = [0.6, 0.5, 0.75, 0.4][it % 4]
        c = [15.0, 1.0, 2.5, 0.6][(it // 4) % 4]
        x, y = random_pair(rng, n, style)
        b, o1, o2, m = oracle.score(x, y, alpha, c)
        b2, mr = reference.score(x, y, alpha, c)
        assert b == b2
        assert (bits(m) == bits(mr)).all(), (it, n, alpha, c)
        assert (bits(oracle.statistics(x, y, alpha, c)[:4]) ==
                bits(reference.statistics(x, y, alpha, c)[:4])).all()


def test_oracle_subproblems_match_reference(oracle, reference):
    rng = np.random.default_rng(77)
    for it in range(80):
        n = int(rng.integers(2, 300))
        x, y = random_pair(rng, n, it % 4)
        args = (x, y, int(rng.integers(2, 15)), int(rng.integers(2, 10)), int(rng.integers(1, 50)))
        a, b = oracle.subproblem(*args), reference.subproblem(*args)
        for k in ("row_count", "clump_count", "k", "h_q"):
            assert a[k] == b[k]
        assert (a["q_x"] == b["q_x"]).all() and (a["bounds"] == b["bounds"]).all()
        assert (bits(a["values"]) == bits(b["values"])).all()


def test_cache_free_reference_matches_engine(reference):
    """test_oracle.cpp:74-88 run on the compiled reference: its recount path
    equals its engine bit for bit (sanity of the oracle build itself)."""
    rng = np.random.default_rng(93)
    for it in range(20):
        x, y = random_pair(rng, int(rng.integers(10, 200)), it % 4)
        a = reference.statistics(x, y)
        b = reference.cache_free_statistics(x, y)
        assert (bits(a[:4]) == bits(b[:4])).all()


def test_run_analysis_order_and_workers(oracle, reference):
    """test_analysis.cpp:132-163: pairwise batch == direct per-pair scoring,
    and worker count never changes the records."""
    rng = np.random.default_rng(53)
    V = rng.uniform(-2, 2, (20, 30))
    V[3] = rng.integers(0, 7, 30)
    base = reference.run_analysis(V, workers=1)
    for w in (2, 4, 8):
        assert (bits(reference.run_analysis(V, workers=w)) == bits(base)).all()
    ours = oracle.pairwise(V, threads=3)
    assert (bits(ours[:, :4]) == bits(base[:, :4])).all()


# --- committed golden fixtures (generated from the reference) ---------------
def _load(name):
    return np.load(os.path.join(GOLDEN, name))


def test_golden_pairs(oracle):
    g = _load("ref_pairs.npz")
    for i in range(len(g["n"])):
        x = g["x"][g["off"][i]:g["off"][i + 1]]
        y = g["y"][g["off"][i]:g["off"][i + 1]]
        b, o1, o2, m = oracle.score(x, y, float(g["alpha"][i]), float(g["c"][i]))
        assert b == g["bound"][i]
        assert (bits(m) == bits(g["cells"][g["coff"][i]:g["coff"][i + 1]])).all(), i
        s = oracle.statistics(x, y, float(g["alpha"][i]), float(g["c"][i]))
        assert (bits(s[:4]) == bits(g["stats"][i])).all(), i


def test_golden_subproblems(oracle):
    g = _load("ref_subproblems.npz")
    for i, (n, yt, xm, kh, rc, raw, k) in enumerate(g["meta"]):
        x = g["x"][g["off"][i]:g["off"][i + 1]]
        y = g["y"][g["off"][i]:g["off"][i + 1]]
        d = oracle.subproblem(x, y, int(yt), int(xm), int(kh))
        assert (d["row_count"], d["clump_count"], d["k"]) == (rc, raw, k)
        assert d["h_q"] == g["h_q"][i]
        assert (d["bounds"] == g["bounds"][g["boff"][i]:g["boff"][i + 1]]).all()
        assert (bits(d["values"]) == bits(g["values"][g["voff"][i]:g["voff"][i + 1]])).all()


def test_golden_configs(oracle):
    g = _load("ref_configs.npz")
    assert (bits(oracle.pairwise(g["c1_vars"])[:, :4]) == bits(g["c1_stats"])).all()
    V = g["c0_vars"]
    got = oracle.pairs(V, np.arange(0, len(V), 2), np.arange(1, len(V), 2))
    assert (bits(got[:, :4]) == bits(g["c0_stats"])).all()
    assert (bits(oracle.pairwise(g["c2_vars"], est=1)[:, :4]) == bits(g["c2_stats"])).all()
    assert (bits(oracle.pairwise(g["c3_vars"])[:, :4]) == bits(g["c3_stats"])).all()
    got = oracle.cross(g["c4r_X"], g["c4r_Y"], 0.75, 15.0, 1)
    assert (bits(got[:, :4]) == bits(g["c4r_stats"])).all()


def _same(a, b):
    """Bit-equal, treating any two NaNs as equal (NaN payloads are not part
    of the reference's contract: pearson returns quiet_NaN, statistics.cpp:46)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    nan = np.isnan(a) & np.isnan(b)
    return bool(((bits(a) == bits(b)) | nan).all())


def test_golden_pearson(oracle):
    """statistics.cpp:39-51 against the reference's own compute_statistics
    (pearson_r, nonlinearity columns of the golden fixture)."""
    g = _load("ref_pairs.npz")
    s6 = g["stats6"]
    for i in range(len(g["n"])):
        x = g["x"][g["off"][i]:g["off"][i + 1]]
        y = g["y"][g["off"][i]:g["off"][i + 1]]
        r = oracle.pearson(x, y)
        assert _same(r, s6[i, 4]), i
        assert _same(s6[i, 0] - r * r, s6[i, 5]), i
    assert np.isnan(s6[:, 4]).any() and not np.isnan(s6[:, 4]).all()
