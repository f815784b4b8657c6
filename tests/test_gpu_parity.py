"""GPU parity: the CUDA engine against the oracle (bit-exact M and statistics)
and against the committed golden vectors of the reference.  Mirrors the
reference's tests (tests/test_char_matrix.cpp, test_statistics.cpp,
test_oracle.cpp, acceptance.cpp criteria 1, 5, 6)."""
import numpy as np
import pytest

from conftest import bits, random_pair

from paper_1208_4271_b200 import (ALL_STATS, MIC_E, MineError, Parameters, cell_shapes, datagen,
                                  grid_bound)

pytestmark = pytest.mark.gpu

STAT_COLS = ["mic", "mas", "mev", "mcn", "mic_e", "tic"]


def stats_matrix(res):
    return np.stack([res[k] for k in STAT_COLS], axis=1)


def assert_bit_equal(got, want, what=""):
    g, w = bits(got), bits(want)
    bad = np.nonzero(g != w)
    assert g.shape == w.shape, what
    assert bad[0].size == 0, f"{what}: {bad[0].size} mismatches, first at {bad[0][:5]}: " \
                             f"{np.asarray(got).ravel()[:3]} vs {np.asarray(want).ravel()[:3]}"


# ---------------------------------------------------------------------------
def test_worked_example_partitions(engine, oracle):
    """Fig. 2 (test_partition.cpp:61-69,128-139,193-206; acceptance.cpp:322-344)."""
    x = np.array([1, 1, 1, 1, 2, 2, 3, 4, 5, 6, 7, 8, 9, 9], float)
    y = np.array([1, 2, 3, 4, 3, 4, 5, 6, 6, 6, 5, 3, 2, 1], float)
    g = engine.debug_subproblem(x, y, 3, 2, 5)
    assert g["row_count"] == 3 and g["clump_count"] == 5 and g["k"] == 5
    # clump sizes 4,2,5,1,2 -> boundaries
    assert list(g["bounds"]) == [0, 4, 6, 11, 12, 14]
    cap = engine.debug_subproblem(x, y, 3, 2, 3)
    assert cap["k"] == 3 and list(cap["bounds"]) == [0, 4, 11, 14]
    o = oracle.subproblem(x, y, 3, 2, 3)
    assert o["k"] == cap["k"] and np.array_equal(o["bounds"], cap["bounds"])
    assert np.array_equal(o["q_x"], g["q_x"])


@pytest.mark.parametrize("seed", range(4))
def test_debug_subproblem_bit_exact(engine, oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    for it in range(40):
        n = int(rng.integers(2, 400))
        x, y = random_pair(rng, n, it % 4)
        yt = int(rng.integers(2, 20))
        xm = int(rng.integers(2, 12))
        kh = int(rng.integers(1, 60))
        g = engine.debug_subproblem(x, y, yt, xm, kh)
        o = oracle.subproblem(x, y, yt, xm, kh)
        ctx = f"seed={seed} it={it} n={n} y={yt} x={xm} khat={kh}"
        assert g["row_count"] == o["row_count"], ctx
        assert g["clump_count"] == o["clump_count"], ctx
        assert g["k"] == o["k"], ctx
        assert np.array_equal(g["bounds"], o["bounds"]), ctx
        # labels inside an x-tie run may be permuted: compare per run
        assert g["h_q"] == o["h_q"], ctx
        assert_bit_equal(g["values"], o["values"], ctx)


@pytest.mark.parametrize("tier", [0, 1, 2, 3])
def test_small_shapes_bit_exact(engine, oracle, tier):
    """n <= 32, B <= 7: the memo tier (auto / 3, n <= 31: padded 3-row table
    up to n = 24, compact above), the tiny tier (1)
    and the general tier (2) must all match the oracle bit for bit, including
    ties, monotone and constant variables and superclumping (small c)."""
    rng = np.random.default_rng(7 + tier)
    for it in range(80):
        n = int(rng.integers(2, 32 if tier == 3 else 33))
        alpha = [0.6, 0.5, 0.55, 0.45][it % 4]
        if grid_bound(n, alpha) > 7:
            alpha = 0.5 if grid_bound(n, 0.5) <= 7 else 0.4
        c = [15.0, 1.0, 2.0, 0.7][it % 4]
        x, y = random_pair(rng, n, it % 4)
        res = engine.pairs(np.stack([x, y]), [0], [1], Parameters(alpha, c), cells=True, tier=tier)
        b, o1, o2, m = oracle.score(x, y, alpha, c)
        ctx = f"it={it} n={n} alpha={alpha} c={c}"
        assert_bit_equal(res["cells"][0, 0], o1, ctx + " o1")
        assert_bit_equal(res["cells"][0, 1], o2, ctx + " o2")
        want = oracle.statistics(x, y, alpha, c)
        assert_bit_equal(stats_matrix(res)[0], want, ctx)


def test_general_random_pairs_bit_exact(engine, oracle):
    rng = np.random.default_rng(31)
    vars_, xi, yi = [], [], []
    for it in range(48):
        n = 120
        x, y = random_pair(rng, n, it % 4)
        vars_ += [x, y]
        xi.append(2 * it)
        yi.append(2 * it + 1)
    V = np.stack(vars_)
    for est in (0, 1):
        p = Parameters(0.6, 15.0, est)
        res = engine.pairs(V, xi, yi, p, cells=True)
        want = oracle.pairs(V, xi, yi, 0.6, 15.0, est)
        assert_bit_equal(stats_matrix(res), want, f"est={est}")


def test_sine_golden(engine):
    """acceptance.cpp:62-92 / PAPER.md:1038-1044."""
    n = 1001
    x = np.arange(n) / (n - 1)
    y = np.sin(10 * np.pi * x) + x
    s = engine.compute_statistics(x, y)
    assert abs(s["mic"] - 0.999999) <= 1e-3
    assert abs(s["mev"] - 0.999999) <= 1e-3
    assert abs(s["mcn"] - 4.584963) <= 1e-3
    assert abs(s["mas"] - 0.728144) <= 0.02


def test_identity_and_constant(engine):
    """test_statistics.cpp:41-60, test_char_matrix.cpp:54-76."""
    x = np.arange(100.0)
    s = engine.compute_statistics(x, x)
    assert s["mic"] == 1.0 and s["mas"] == 0.0 and s["mev"] == 1.0 and s["mcn"] == 2.0
    m = engine.compute_score(x, x)
    assert m.entry(2, 2) == 1.0
    c = engine.compute_statistics(np.arange(40.0), np.full(40, 2.0))
    assert c["mic"] == 0.0 and c["mcn"] == 2.0


@pytest.mark.parametrize("tier", [0, 1, 2])
def test_c1_pairwise_bit_exact(engine, oracle, tier):
    """Config c1's shape (n=23, B=6): a 300-variable slice, all pairs, against
    the oracle, through every tier that admits it."""
    w = datagen.make(1)
    V = w.X[:300]
    res = engine.pairwise(V, tier=tier)
    want = oracle.pairwise(V)
    assert_bit_equal(stats_matrix(res), want, f"c1 slice tier={tier}")


def test_c0_pairs_bit_exact(engine, oracle):
    w = datagen.make(0, npairs=24)
    res = engine.pairs(w.X, w.xi, w.yi, Parameters(w.alpha, w.c, w.est))
    want = oracle.pairs(w.X, w.xi, w.yi, w.alpha, w.c, w.est)
    assert_bit_equal(stats_matrix(res), want, "c0")


# --- against the committed golden fixtures (the reference's own outputs) ----
GOLDEN = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden")


def _golden(name):
    return np.load(__import__("os").path.join(GOLDEN, name))


@pytest.mark.parametrize("tier", [0, 2])
def test_golden_pairs_gpu(engine, tier):
    g = _golden("ref_pairs.npz")
    for i in range(len(g["n"])):
        x = g["x"][g["off"][i]:g["off"][i + 1]]
        y = g["y"][g["off"][i]:g["off"][i + 1]]
        alpha, c = float(g["alpha"][i]), float(g["c"][i])
        if tier == 2 and len(x) <= 3:
            continue
        res = engine.pairs(np.stack([x, y]), [0], [1], Parameters(alpha, c), cells=True, tier=tier)
        cells = res["cells"][0]
        m = np.where(cells[1] > cells[0], cells[1], cells[0])
        assert_bit_equal(m, g["cells"][g["coff"][i]:g["coff"][i + 1]], f"case {i}")
        assert_bit_equal(stats_matrix(res)[0, :4], g["stats"][i], f"case {i}")


def test_golden_subproblems_gpu(engine):
    g = _golden("ref_subproblems.npz")
    for i, (n, yt, xm, kh, rc, raw, k) in enumerate(g["meta"]):
        x = g["x"][g["off"][i]:g["off"][i + 1]]
        y = g["y"][g["off"][i]:g["off"][i + 1]]
        d = engine.debug_subproblem(x, y, int(yt), int(xm), int(kh))
        assert (d["row_count"], d["clump_count"], d["k"]) == (rc, raw, k), i
        assert d["h_q"] == g["h_q"][i]
        assert (d["bounds"] == g["bounds"][g["boff"][i]:g["boff"][i + 1]]).all()
        assert_bit_equal(d["values"], g["values"][g["voff"][i]:g["voff"][i + 1]], f"sub {i}")


def test_golden_configs_gpu(engine):
    g = _golden("ref_configs.npz")
    assert_bit_equal(stats_matrix(engine.pairwise(g["c1_vars"]))[:, :4], g["c1_stats"], "c1")
    V = g["c0_vars"]
    r = engine.pairs(V, np.arange(0, len(V), 2), np.arange(1, len(V), 2))
    assert_bit_equal(stats_matrix(r)[:, :4], g["c0_stats"], "c0")
    r = engine.pairwise(g["c2_vars"], Parameters(0.6, 15.0, MIC_E))
    assert_bit_equal(stats_matrix(r)[:, :4], g["c2_stats"], "c2")
    assert_bit_equal(stats_matrix(engine.pairwise(g["c3_vars"]))[:, :4], g["c3_stats"], "c3")
    r = engine.cross(g["c4r_X"], g["c4r_Y"], Parameters(0.75, 15.0, MIC_E))
    assert_bit_equal(stats_matrix(r)[:, :4], g["c4r_stats"], "c4 (n=1500)")


def _same(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    nan = np.isnan(a) & np.isnan(b)
    return bool(((a.view(np.int64) == b.view(np.int64)) | nan).all())


def test_golden_pearson_gpu(engine):
    """pearson_r / nonlinearity (statistics.cpp:39-51) on the device against
    the reference's compute_statistics: the golden pairs one by one, and the c1
    slice through the batch path (bit-exact: both sum sequentially)."""
    g = _golden("ref_pairs.npz")
    for i in range(len(g["n"])):
        x = g["x"][g["off"][i]:g["off"][i + 1]]
        y = g["y"][g["off"][i]:g["off"][i + 1]]
        s = engine.compute_statistics(x, y, Parameters(float(g["alpha"][i]), float(g["c"][i])))
        assert _same(s["pearson_r"], g["stats6"][i, 4]), i
        assert _same(s["nonlinearity"], g["stats6"][i, 5]), i
    c = _golden("ref_configs.npz")
    r = engine.pairwise(c["c1_vars"], stats=("mic", "pearson_r", "nonlinearity"))
    assert _same(r["pearson_r"], c["c1_stats6"][:, 4])
    assert _same(r["nonlinearity"], c["c1_stats6"][:, 5])
    # non-linearity alone (MIC computed internally), and the general tier
    r2 = engine.pairwise(c["c1_vars"], stats=("nonlinearity",), tier=2)
    assert _same(r2["nonlinearity"], c["c1_stats6"][:, 5])


def test_reuse_vars_and_master_vs_all(engine, oracle):
    """windows of one job with the per-variable stages run
    once (reuse_vars), and master_vs_all (analysis.cpp:25-30,82-85) -- both
    bit-identical to the single full call / the oracle, and a reuse request
    with different variables fails instead of scoring stale state."""
    w = datagen.make(1)
    V = np.ascontiguousarray(w.X[:80])
    full = engine.pairwise(V, stats=ALL_STATS)
    total = 80 * 79 // 2
    parts = [engine.pairwise(V, first=0, count=1000, stats=ALL_STATS)]
    for first in range(1000, total, 1000):
        parts.append(engine.pairwise(V, first=first, count=min(1000, total - first),
                                     stats=ALL_STATS, reuse_vars=True))
    for k in ALL_STATS:
        assert _same(np.concatenate([p[k] for p in parts]), full[k]), k
    for tier in (0, 2):
        for m in (0, 37, 79):
            got = engine.master_vs_all(V, m, tier=tier, reuse_vars=(m != 0))
            others = [j for j in range(80) if j != m]
            want = oracle.pairs(V, np.minimum(others, m), np.maximum(others, m))
            assert_bit_equal(stats_matrix(got), want[:, :6], f"master {m} tier {tier}")
    with pytest.raises(MineError):
        engine.pairwise(np.ascontiguousarray(w.X[:81]), reuse_vars=True)


# --- config-scale parity and size-independent properties ---------------------
def test_c2_poisson_ties_slice(engine, oracle):
    """c2 (heavy ties / zeros): 12 variables -> 66 pairs, est = MIC_e."""
    w = datagen.make(2)
    V = w.X[[0, 1, 2, 3, 10, 11, 500, 501, 1000, 1001, 1998, 1999]]
    res = engine.pairwise(V, Parameters(w.alpha, w.c, w.est))
    want = oracle.pairwise(V, w.alpha, w.c, w.est)
    assert_bit_equal(stats_matrix(res), want, "c2 slice")


def test_c3_slice_and_monotone_invariance(engine, oracle):
    """c3 at full n=1340: 6 variables vs the oracle, and M is rank-invariant
    (SURVEY A3): a strictly monotone transform changes nothing."""
    w = datagen.make(3)
    V = w.X[:6]
    res = engine.pairwise(V)
    assert_bit_equal(stats_matrix(res), oracle.pairwise(V), "c3 slice")
    T = np.stack([np.exp(V[0] / 4), V[1] ** 3, np.tanh(V[2] / 4), V[3], 3 * V[4] + 1, V[5]])
    assert_bit_equal(stats_matrix(engine.pairwise(T)), stats_matrix(res), "monotone")


def test_full_size_properties_c0(engine):
    """All 256 c0 pairs at full size: swap invariance (test_statistics.cpp:
    114-132), MAS/MEV <= MIC, MCN range, and c-saturation
    (test_char_matrix.cpp:111-121)."""
    w = datagen.make(0)
    p = Parameters(w.alpha, w.c, w.est)
    a = engine.pairs(w.X, w.xi, w.yi, p)
    b = engine.pairs(w.X, w.yi, w.xi, p)
    for k in ("mic", "mas", "mev", "mcn", "mic_e"):
        assert_bit_equal(a[k], b[k], f"swap {k}")
    assert np.all(a["mas"] <= a["mic"]) and np.all(a["mev"] <= a["mic"])
    assert np.all(a["mcn"] >= 2.0) and np.all(a["mcn"] <= np.log2(grid_bound(1000, 0.6)))
    assert np.all((a["mic"] >= 0) & (a["mic"] <= 1)) and np.all(a["mic_e"] <= 1)
    # functional noiseless pairs (sigma = 0: pairs i with i % 4 == 0, f not indep.)
    noiseless = [i for i in range(256) if i % 4 == 0 and i % 5 != 4]
    assert np.all(a["mic"][noiseless] > 0.9)
    sub = list(range(0, 256, 17))
    s1 = engine.pairs(w.X, w.xi[sub], w.yi[sub], Parameters(0.6, 1000.0))
    s2 = engine.pairs(w.X, w.xi[sub], w.yi[sub], Parameters(0.6, 3000.0))
    for k in STAT_COLS:
        assert_bit_equal(s1[k], s2[k], f"c-saturation {k}")


def test_batch_slicing_is_bitwise_stable(engine):
    """Any (first, count) window of the pair space gives the same bits as the
    full batch (the multi-GPU sharding contract)."""
    w = datagen.make(1)
    V = w.X[:200]
    full = engine.pairwise(V)
    total = 200 * 199 // 2
    for first, count in ((0, 1), (5, 1000), (7000, total - 7000), (total - 3, 3)):
        part = engine.pairwise(V, first=first, count=count)
        for k in STAT_COLS:
            assert_bit_equal(part[k], full[k][first:first + count], f"{k} window {first}")


def test_minepy_c_api(engine, oracle):
    """mine_compute_score / mine_mic ... and mine_compute_pstats through the
    C ABI (the minepy-style drop-in names)."""
    import ctypes
    from paper_1208_4271_b200 import engine as E
    L = E.load_library()
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, 300)
    y = np.sin(6 * x) + rng.normal(0, 0.2, 300)
    prob = E.MineProblem(300, x.ctypes.data_as(E._dp), y.ctypes.data_as(E._dp))
    par = E.MineParameter(0.6, 15.0, 0)
    sc = L.mine_compute_score(ctypes.byref(prob), ctypes.byref(par))
    assert sc, L.mine_b200_last_error()
    want = oracle.statistics(x, y)
    got = [L.mine_mic(sc), L.mine_mas(sc), L.mine_mev(sc), L.mine_mcn(sc, 0.0), L.mine_mic_e(sc)]
    assert_bit_equal(np.array(got), want[:5], "mine_* accessors")
    b, o1, o2, m = oracle.score(x, y)
    assert abs(L.mine_tic(sc, 0) - m.sum()) < 1e-9
    L.mine_free_score(ctypes.byref(sc))
    # invalid input -> NULL + message
    bad = np.array([1.0, np.nan, 2.0])
    prob = E.MineProblem(3, bad.ctypes.data_as(E._dp), bad.ctypes.data_as(E._dp))
    assert not L.mine_compute_score(ctypes.byref(prob), ctypes.byref(par))
    assert b"finite" in L.mine_b200_last_error()


def test_errors_like_the_reference(engine):
    """char_matrix.cpp:11-15,71-75: validation failures raise."""
    from paper_1208_4271_b200 import MineError
    with pytest.raises(MineError):
        engine.compute_statistics([1, 2, 3], [1, 2])
    with pytest.raises(MineError):
        engine.compute_statistics([1.0], [2.0])
    with pytest.raises(MineError):
        engine.compute_statistics([1, 2, np.inf, 4], [1, 2, 3, 4])
    with pytest.raises(MineError):
        engine.compute_statistics([1, 2, 3, 4], [1, 2, 3, 4], Parameters(0.6, -1.0))
    with pytest.raises(MineError):
        engine.pairwise(np.zeros((3, 5)), first=2, count=5)


@pytest.mark.slow
def test_c4_full_size_properties(engine):
    """c4 at its full size (n = 10,000, alpha = .75, B = 1000, est = MIC_e) --
    the CPU oracle needs hours per pair here, so size-independent properties:
    rank invariance and X/Y swap invariance bit-exact, bounds, and
    functional vs independent separation.  Parity itself is pinned at
    n = 1500 by test_golden_configs_gpu."""
    w = datagen.make(4)
    p = Parameters(w.alpha, w.c, w.est)
    # Y_0 = 2u-1 + N(0,.05^2) is functional in X_0; pick one replaced (independent) Y
    sel = [0, 1]
    X = w.X[:1]
    Y = w.Y[sel]
    a = engine.cross(X, Y, p)
    b = engine.cross(np.exp(X / 4.0), Y ** 3, p)  # strictly monotone transforms
    for k in STAT_COLS:
        assert_bit_equal(a[k], b[k], f"c4 monotone {k}")
    c = engine.cross(Y, X, p)  # swapped roles: Y x X
    for k in ("mic", "mas", "mev", "mcn", "mic_e"):
        assert_bit_equal(a[k], c[k], f"c4 swap {k}")
    assert np.all((a["mic"] >= 0) & (a["mic"] <= 1)) and np.all(a["mas"] <= a["mic"])
    assert a["mic"][0] > 0.9  # near-noiseless linear relation


def test_span_quotients_match_ieee_division_exhaustively():
    """The engine's span-term quotients c_s/c_t (mutual_info.cpp:62) use one
    reciprocal per c_t plus a Markstein correction (device_common.cuh
    int_quot) instead of a DDIV: bitwise equal to IEEE a/b for EVERY
    0 <= a <= b <= 65535 (the whole supported n), checked here on the GPU."""
    import ctypes
    from paper_1208_4271_b200 import _build
    L = ctypes.CDLL(_build.PROBES)
    bad, cnt = ctypes.c_ulonglong(0), ctypes.c_ulonglong(0)
    assert L.mine_b200_check_quotients(0, 65535, ctypes.byref(bad), ctypes.byref(cnt)) == 0
    assert cnt.value == 65536 * 65537 // 2 - 1
    assert bad.value == 0


@pytest.mark.parametrize("n", [37, 95, 233, 517])
def test_randomized_batches_bit_exact(engine, oracle, n):
    """Stress: 1000-pair batches of mixed styles (continuous, tied, monotone,
    constant, heavy ties), random alpha / c / est, through the batch path (all
    tiers the auto selection picks, the concurrent y lanes, superclumps),
    bit-exact against the oracle."""
    rng = np.random.default_rng(1000 + n)
    vars_, xi, yi = [], [], []
    for it in range(1000):
        style = it % 5
        if style < 4:
            x, y = random_pair(rng, n, style)
        else:
            x = rng.integers(0, 3, n).astype(float)
            y = rng.poisson(2.0, n).astype(float)
        vars_ += [x, y]
        xi.append(2 * it)
        yi.append(2 * it + 1)
    V = np.stack(vars_)
    for alpha, c, est in [(0.6, 15.0, 0), (float(rng.uniform(0.45, 0.75)), float(rng.choice([1.0, 3.0, 7.5])), 1)]:
        res = engine.pairs(V, xi, yi, Parameters(alpha, c, est))
        want = oracle.pairs(V, xi, yi, alpha, c, est)
        assert_bit_equal(stats_matrix(res), want, f"n={n} alpha={alpha} c={c} est={est}")


@pytest.mark.parametrize("n,alpha", [(30000, 0.45), (65535, 0.4)])
def test_large_n_point_arrays_in_hbm(engine, oracle, n, alpha):
    """Above n ~ 19000 (alpha 0.6) the partition stage's per-point arrays no
    longer fit in shared memory and move to an HBM slot per subproblem
    (k_part_f2<.., kPtsGlobal>).  Bit-exact up to the ABI's n limit, 65535."""
    rng = np.random.default_rng(n)
    vars_ = []
    for style in range(4):
        vars_ += list(random_pair(rng, n, style))
    x = rng.uniform(0, 6, n)
    vars_ += [x, np.sin(x) + rng.normal(0, 0.3, n)]
    V = np.stack(vars_)
    xi, yi = list(range(0, 10, 2)), list(range(1, 10, 2))
    for c, est in [(15.0, 0), (2.0, 1)]:
        res = engine.pairs(V, xi, yi, Parameters(alpha, c, est))
        want = oracle.pairs(V, xi, yi, alpha, c, est)
        assert_bit_equal(stats_matrix(res), want, f"n={n} c={c}")


def test_many_levels_f_ring(engine, oracle):
    """x_max > 128 with k > 128: k_dp's F rows become a 128-column ring and
    F(k, .) its own row (n = 1500, alpha = 0.8: B = 346, x_max = 173 at y = 2)."""
    n = 1500
    rng = np.random.default_rng(12)
    x = rng.uniform(0, 6, n)
    V = np.stack([x, np.sin(x) + rng.normal(0, 0.2, n), rng.uniform(-1, 1, n),
                  np.round(x * 20) + rng.integers(0, 2, n)])
    xi, yi = [0, 0, 3, 2], [1, 3, 1, 0]
    for c in (15.0, 4.0):
        res = engine.pairs(V, xi, yi, Parameters(0.8, c, 0), cells=True)
        want = oracle.pairs(V, xi, yi, 0.8, c, 0)
        assert_bit_equal(stats_matrix(res), want, f"c={c}")


def test_large_c_times_b_tables_in_hbm(engine, oracle):
    """c B so large that k_dp's clump bounds and cumulative table (y (k^+1)
    ints) leave shared memory: n = 20000, alpha = 0.8 (B = 2759), c = 15.
    Tie-heavy variables keep the oracle's DP small."""
    n = 20000
    rng = np.random.default_rng(77)
    x = rng.integers(0, 40, n).astype(float)
    V = np.stack([x, (x % 7) + rng.integers(0, 3, n), rng.integers(0, 25, n).astype(float),
                  np.round(np.sin(x / 6.0), 1)])
    xi, yi = [0, 0, 2], [1, 3, 1]
    res = engine.pairs(V, xi, yi, Parameters(0.8, 15.0, 0))
    want = oracle.pairs(V, xi, yi, 0.8, 15.0, 0)
    assert_bit_equal(stats_matrix(res), want, "alpha=0.8")


@pytest.mark.parametrize("force", ["MINE_B200_PF_GLOBAL", "MINE_B200_DP_GLOBAL",
                                   "MINE_B200_RADIX_SORT"])
def test_large_n_variants_forced(force):
    """The large-n variants forced at small n (each switch is read once per
    process) on a mixed 600-pair batch: partition point arrays in HBM,
    clump bounds / cumulative table in HBM for k_part_f2 and k_dp, radix K1."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, sys\n"
        "sys.path[:0] = ['tests', 'oracle', '.']\n"
        "from conftest import random_pair, bits\n"
        "import oracle as O\n"
        "from paper_1208_4271_b200 import Engine, Parameters\n"
        "rng = np.random.default_rng(5)\n"
        "vs = []\n"
        "for it in range(600):\n"
        "    vs += list(random_pair(rng, 300, it % 4))\n"
        "V = np.stack(vs); xi = list(range(0, 1200, 2)); yi = list(range(1, 1200, 2))\n"
        "e = Engine(0)\n"
        "for a, c, est in [(0.6, 15.0, 0), (0.7, 3.0, 1)]:\n"
        "    r = e.pairs(V, xi, yi, Parameters(a, c, est))\n"
        "    got = np.stack([r[k] for k in ['mic', 'mas', 'mev', 'mcn', 'mic_e', 'tic']], axis=1)\n"
        "    want = O.Oracle().pairs(V, xi, yi, a, c, est)\n"
        "    assert (bits(got) == bits(want)).all(), (a, c)\n"
        "print('OK')\n")
    env = dict(os.environ, **{force: "1"})
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "OK" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("n", [16, 23, 28, 31])
def test_memo_sorted_batches_all_pair_kinds(engine, oracle, n):
    """The memo tier runs pairs in sorted batches of 8192: cross
    and list calls and an unaligned pairwise window, several batches each,
    bit-exact against the oracle."""
    rng = np.random.default_rng(100 + n)
    V = rng.standard_normal((160, n))
    V[::7] = np.round(V[::7] * 2.0)  # some tied variables (sentinel fusing)
    X, Y = V[:110], V[110:]
    res = engine.cross(X, Y)
    xi = np.repeat(np.arange(110), 50)
    yi = 110 + np.tile(np.arange(50), 110)
    want = oracle.pairs(V, xi, yi, 0.6, 15.0, 0)
    assert_bit_equal(stats_matrix(res), want, f"cross n={n}")
    total = 160 * 159 // 2
    first, count = 1234, total - 1234 - 17
    res = engine.pairwise(V, first=first, count=count)
    want = oracle.pairwise(V, first=first, count=count)
    assert_bit_equal(stats_matrix(res), want, f"pairwise window n={n}")
    xi = rng.integers(0, 160, 9000)
    yi = rng.integers(0, 160, 9000)
    res = engine.pairs(V, xi, yi)
    want = oracle.pairs(V, xi, yi, 0.6, 15.0, 0)
    assert_bit_equal(stats_matrix(res), want, f"list n={n}")


def test_memo_sort_off_same_bits(tmp_path):
    """MINE_B200_MEMO_SORT=0 (one pair per thread in index order) and the
    default sorted batches give the same bits."""
    import os
    import subprocess
    import sys
    script = tmp_path / "run.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_1208_4271_b200 import Engine, datagen\n"
        "w = datagen.make(1)\n"
        "r = Engine(0).pairwise(w.X[:400])\n"
        "np.save(sys.argv[1], np.stack([r[k] for k in ('mic', 'mas', 'mev', 'mcn', 'mic_e', 'tic')]))\n")
    outs = []
    for flag in ("0", "1"):
        out = tmp_path / f"o{flag}.npy"
        env = dict(os.environ, MINE_B200_MEMO_SORT=flag)
        subprocess.run([sys.executable, str(script), str(out)], env=env, check=True, timeout=600)
        outs.append(np.load(out))
    assert_bit_equal(outs[0], outs[1], "sorted vs index order")


@pytest.mark.parametrize("n", [23, 28])
def test_memo_output_staging_same_bits(tmp_path, n):
    """MINE_B200_MEMO_STAGE=1 (sorted batches stage their statistics and
    store them in index order) gives the default's bits, for pairwise windows
    spanning several batches and host / device outputs."""
    import os
    import subprocess
    import sys
    script = tmp_path / "run.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_1208_4271_b200 import Engine, datagen\n"
        f"rng = np.random.default_rng({n}); V = rng.standard_normal((600, {n}))\n"
        "V[::9] = np.round(V[::9])\n"
        "e = Engine(0)\n"
        "r = e.pairwise(V, first=1234, count=150000)\n"
        "r2 = e.pairwise(V, first=0, count=20000, reuse_vars=True)\n"
        "np.save(sys.argv[1], np.concatenate([np.stack([r[k] for k in ('mic', 'mas', 'mev', 'mcn', 'mic_e', 'tic')]),\n"
        "                                     np.stack([r2[k] for k in ('mic', 'mas', 'mev', 'mcn', 'mic_e', 'tic')])], 1))\n")
    outs = []
    for flag in ("0", "1"):
        out = tmp_path / f"o{flag}.npy"
        env = dict(os.environ, MINE_B200_MEMO_STAGE=flag)
        subprocess.run([sys.executable, str(script), str(out)], env=env, check=True, timeout=600)
        outs.append(np.load(out))
    assert_bit_equal(outs[0], outs[1], "staged vs scattered")


def _tied_vars(rng, p, n):
    """Tie-heavy variables whose row maps saturate at small y (the row-map
    dedup's case): Poisson counts over a range of rates, a few discretised
    normals and one near-constant variable."""
    lam = np.exp(rng.uniform(np.log(0.1), np.log(40.0), p))
    V = rng.poisson(lam[:, None] * np.exp(0.8 * rng.standard_normal(n))[None, :] ** (np.arange(p) % 2)[:, None])
    V = V.astype(float)
    V[3::7] = np.round(rng.standard_normal((len(range(3, p, 7)), n)) * 1.5)
    V[5, :] = 0.0
    V[5, : n // 3] = 1.0
    return V


@pytest.mark.parametrize("n,alpha,c", [(300, 0.6, 15.0), (500, 0.6, 15.0), (400, 0.7, 0.6), (250, 0.8, 2.0)])
def test_row_dedup_ties_bit_exact(engine, oracle, n, alpha, c):
    """Pairs whose row maps repeat over y (ties saturate the equipartition):
    the subproblems k_part_f2 turns into copies of a smaller y's cells, and
    the ones it still computes because their raw clumps superclump at the
    larger y (small c), give the oracle's cells of both orientations and the
    statistics bit for bit."""
    rng = np.random.default_rng(n + int(100 * c))
    V = _tied_vars(rng, 24, n)
    res = engine.pairwise(V, Parameters(alpha, c, 1), cells=True)
    want = oracle.pairwise(V, alpha, c, 1)
    assert_bit_equal(stats_matrix(res), want, "tied pairwise")
    k = 0
    for i in range(V.shape[0]):
        for j in range(i + 1, V.shape[0]):
            if k % 7 == 0:
                _, o1, o2, _m = oracle.score(V[i], V[j], alpha, c)
                assert_bit_equal(res["cells"][k, 0], o1, f"o1 pair {i},{j}")
                assert_bit_equal(res["cells"][k, 1], o2, f"o2 pair {i},{j}")
            k += 1


def test_row_dedup_off_same_bits(tmp_path):
    """MINE_B200_ROW_DEDUP=0 (every subproblem computed) gives the default's
    bits: statistics and cells of a c2 window, a cross call and a list call
    on one orientation's worth of tied variables."""
    import os
    import subprocess
    import sys
    script = tmp_path / "run.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_1208_4271_b200 import Engine, Parameters, datagen\n"
        "w = datagen.make(2); P = Parameters(w.alpha, w.c, w.est)\n"
        "e = Engine(0)\n"
        "r = e.pairwise(w.X, P, first=5000, count=6000, cells=True)\n"
        "X, Y = w.X[:20], w.X[1500:1530]\n"
        "r2 = e.cross(X, Y, Parameters(0.6, 3.0, 1), cells=True)\n"
        "cols = ('mic', 'mas', 'mev', 'mcn', 'mic_e', 'tic')\n"
        "a = np.concatenate([np.stack([r[k] for k in cols]).ravel(), r['cells'].ravel(),\n"
        "                    np.stack([r2[k] for k in cols]).ravel(), r2['cells'].ravel()])\n"
        "np.save(sys.argv[1], a)\n")
    outs = []
    for flag in ("0", "1"):
        out = tmp_path / f"o{flag}.npy"
        env = dict(os.environ, MINE_B200_ROW_DEDUP=flag)
        subprocess.run([sys.executable, str(script), str(out)], env=env, check=True, timeout=600)
        outs.append(np.load(out))
    assert_bit_equal(outs[1], outs[0], "row-map dedup vs every subproblem computed")


def test_bitonic_sort_same_bits(tmp_path):
    """K1's bitonic shared-memory sort (64 < n <= 8192) gives the O(n^2)
    ranking's bits (MINE_B200_BITONIC=0): ties, -0.0 against +0.0, huge and
    tiny magnitudes, constant variables, n not a power of two; statistics,
    cells and the debug partition."""
    import os
    import subprocess
    import sys
    script = tmp_path / "run.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_1208_4271_b200 import Engine, Parameters\n"
        "rng = np.random.default_rng(5)\n"
        "e = Engine(0)\n"
        "out = []\n"
        "for n in (65, 100, 333, 1000, 2049):\n"
        "    V = rng.standard_normal((10, n))\n"
        "    V[1] = np.round(V[1] * 2)\n"
        "    V[2, ::3] = -0.0\n"
        "    V[2, 1::3] = 0.0\n"
        "    V[3] = 7.0\n"
        "    V[4] *= 1e300\n"
        "    V[5] *= 1e-300\n"
        "    V[6] = rng.integers(0, 3, n)\n"
        "    r = e.pairwise(V, Parameters(0.6, 15.0, 1), cells=True)\n"
        "    out += [np.stack([r[k] for k in ('mic', 'mas', 'mev', 'mcn', 'mic_e', 'tic')]).ravel(), r['cells'].ravel()]\n"
        "    d = e.debug_subproblem(V[1], V[6], 2, 5, 30)\n"
        "    out += [np.asarray(d['bounds'], float), np.asarray(d['q_x'], float)]\n"
        "np.save(sys.argv[1], np.concatenate(out))\n")
    outs = []
    for flag in ("0", "1"):
        out = tmp_path / f"o{flag}.npy"
        env = dict(os.environ, MINE_B200_BITONIC=flag)
        subprocess.run([sys.executable, str(script), str(out)], env=env, check=True, timeout=600)
        outs.append(np.load(out))
    assert_bit_equal(outs[1], outs[0], "bitonic sort vs ranking")


def test_big_sort_same_bits(tmp_path):
    """K1's large-n sort k_sort_big (chunked bitonic through an HBM scratch,
    n > 16384 by default) forced at smaller n (MINE_B200_RADIX_SORT=1) gives
    the on-chip sorts' bits: one chunk (n = 65, 1000), two chunks with the
    in-place long-distance passes (n = 8193, 12000); ties, -0.0 against +0.0,
    huge and tiny magnitudes, constant variables."""
    import os
    import subprocess
    import sys
    script = tmp_path / "run.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_1208_4271_b200 import Engine, Parameters\n"
        "rng = np.random.default_rng(9)\n"
        "e = Engine(0)\n"
        "out = []\n"
        "for n, alpha in ((65, 0.6), (1000, 0.6), (8193, 0.45), (12000, 0.45)):\n"
        "    V = rng.standard_normal((8, n))\n"
        "    V[1] = np.round(V[1] * 2)\n"
        "    V[2, ::3] = -0.0\n"
        "    V[2, 1::3] = 0.0\n"
        "    V[3] = 7.0\n"
        "    V[4] *= 1e300\n"
        "    V[5] *= 1e-300\n"
        "    V[6] = rng.integers(0, 3, n)\n"
        "    r = e.pairwise(V, Parameters(alpha, 15.0, 1))\n"
        "    out += [np.stack([r[k] for k in ('mic', 'mas', 'mev', 'mcn', 'mic_e', 'tic')]).ravel()]\n"
        "    d = e.debug_subproblem(V[1], V[6], 2, 5, 30)\n"
        "    out += [np.asarray(d['bounds'], float), np.asarray(d['q_x'], float)]\n"
        "np.save(sys.argv[1], np.concatenate(out))\n")
    outs = []
    for flag in (None, "1"):
        out = tmp_path / f"o{flag}.npy"
        env = dict(os.environ)
        env.pop("MINE_B200_RADIX_SORT", None)
        if flag:
            env["MINE_B200_RADIX_SORT"] = flag
        subprocess.run([sys.executable, str(script), str(out)], env=env, check=True, timeout=600)
        outs.append(np.load(out))
    assert_bit_equal(outs[1], outs[0], "k_sort_big vs the on-chip sorts")


def test_device_plog_span_terms_same_bits(tmp_path):
    """MINE_B200_SPAN_LOG=1: span terms of three or more rows compute
    p*log(p) with the device replay of the host libm's log (plog.cuh),
    enabled only after every host-table entry matched (k_check_plog); the
    results equal the table-gather default bit for bit (c3 / c0 slices, and
    a cross call at n = 2500 where rows reach 12)."""
    import os
    import subprocess
    import sys
    script = tmp_path / "run.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_1208_4271_b200 import Engine, Parameters, datagen\n"
        "e = Engine(0)\n"
        "cols = ('mic', 'mas', 'mev', 'mcn', 'mic_e', 'tic')\n"
        "w3 = datagen.make(3); r3 = e.pairwise(w3.X[:8], Parameters(w3.alpha, w3.c, 1), cells=True)\n"
        "w0 = datagen.make(0, npairs=12); r0 = e.pairs(w0.X, w0.xi, w0.yi, Parameters(w0.alpha, w0.c, 1), cells=True)\n"
        "rng = np.random.default_rng(3); X = rng.standard_normal((3, 2500)); Y = np.tanh(X) + rng.standard_normal((3, 2500))\n"
        "rc = e.cross(X, Y, Parameters(0.6, 5.0, 1), cells=True)\n"
        "np.save(sys.argv[1], np.concatenate([np.stack([r[k] for k in cols]).ravel() for r in (r3, r0, rc)]\n"
        "                                    + [r['cells'].ravel() for r in (r3, r0, rc)]))\n")
    outs = []
    for flag in ("0", "1"):
        out = tmp_path / f"o{flag}.npy"
        env = dict(os.environ, MINE_B200_SPAN_LOG=flag)
        subprocess.run([sys.executable, str(script), str(out)], env=env, check=True, timeout=600)
        outs.append(np.load(out))
    assert_bit_equal(outs[1], outs[0], "computed p*log(p) vs table gathers")


def test_h2_table_same_bits(tmp_path):
    """The two-term table H2(m, w) = pl(m, w) + pl(m, m - w) (one gather for a
    two-row span and for every F(t,2) candidate's H(P), any row count, in
    k_part_f2, k_part_warp, k_dp and k_dp_warp) against the two p*log(p)
    gathers it replaces (MINE_B200_NO_H2=1, the path n > 20000 takes): bit
    for bit on c3 / c2 (ties) / c0 slices and a cross call with up to 12
    rows."""
    import os
    import subprocess
    import sys
    script = tmp_path / "run.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_1208_4271_b200 import Engine, Parameters, datagen\n"
        "e = Engine(0)\n"
        "cols = ('mic', 'mas', 'mev', 'mcn', 'mic_e', 'tic')\n"
        "w3 = datagen.make(3); r3 = e.pairwise(w3.X[:8], Parameters(w3.alpha, w3.c, 1), cells=True)\n"
        "w2 = datagen.make(2); r2 = e.pairwise(w2.X[:24], Parameters(w2.alpha, w2.c, 1), cells=True)\n"
        "w0 = datagen.make(0, npairs=12); r0 = e.pairs(w0.X, w0.xi, w0.yi, Parameters(w0.alpha, w0.c, 1), cells=True)\n"
        "rng = np.random.default_rng(3); X = rng.standard_normal((3, 2500)); Y = np.tanh(X) + rng.standard_normal((3, 2500))\n"
        "rc = e.cross(X, Y, Parameters(0.6, 5.0, 1), cells=True)\n"
        "rs = (r3, r2, r0, rc)\n"
        "np.save(sys.argv[1], np.concatenate([np.stack([r[k] for k in cols]).ravel() for r in rs]\n"
        "                                    + [r['cells'].ravel() for r in rs]))\n")
    outs = []
    for flag in (None, "1"):
        out = tmp_path / f"o{flag}.npy"
        env = dict(os.environ)
        env.pop("MINE_B200_NO_H2", None)
        if flag:
            env["MINE_B200_NO_H2"] = flag
        subprocess.run([sys.executable, str(script), str(out)], env=env, check=True, timeout=600)
        outs.append(np.load(out))
    assert_bit_equal(outs[1], outs[0], "H2 table vs two p*log(p) gathers")


@pytest.mark.parametrize("n", [1024, 1025])
def test_warp_partition_kernel_limit(engine, oracle, n):
    """n = 1024 is the warp partition kernel's limit (positions staged in a
    warp's slice), n = 1025 takes the CTA kernel; both with tied variables,
    superclumps (c = 1) and enough pairs for the batch paths (row-map dedup,
    warp DP classes): statistics bit-exact against the oracle."""
    rng = np.random.default_rng(n)
    V = _tied_vars(rng, 52, n)
    V[::4] = rng.standard_normal((13, n))
    res = engine.pairwise(V, Parameters(0.55, 1.0, 1))
    want = oracle.pairwise(V, 0.55, 1.0, 1)
    assert_bit_equal(stats_matrix(res), want, f"n={n}")
