"""GPU parity: the CUDA engine against the oracle (bit-exact M and statistics)
and against the committed golden vectors of the reference.  Mirrors the
reference's tests (tests/test_char_matrix.cpp, test_statistics.cpp,
test_oracle.cpp, acceptance.cpp criteria 1, 5, 6)."""
import numpy as np
import pytest

from conftest import bits, random_pair

from paper_1208_4271_b200 import MIC_E, Parameters, cell_shapes, datagen, grid_bound

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
    """n <= 32, B <= 7: the memo tier (auto / 3, n <= 24), the tiny tier (1)
    and the general tier (2) must all match the oracle bit for bit, including
    ties, monotone and constant variables and superclumping (small c)."""
    rng = np.random.default_rng(7 + tier)
    for it in range(80):
        n = int(rng.integers(2, 25 if tier == 3 else 33))
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
