"""Full-size parity in the driver-run GPU suite: the GPU
engine against the reference's own engine -- oracle/_ref/libmine_ref.so, the
reference's sources compiled unmodified, `run_analysis` on all host threads --
on the whole headline config c1 (all 9,594,390 pairs), all of c0, and windows
of c2 (the first 317 variables: 50,086 pairs, heavy ties, row-map dedup and
the warp partition kernel) and c3 (the first 46 variables: 1,035 pairs).  MIC,
MAS, MEV, MCN, Pearson r and non-linearity, bit for bit.  ~40 s of CPU time.
tools/full_parity.py runs the whole of c2 as well (profiles/r02)."""
import os

import numpy as np
import pytest

from paper_1208_4271_b200 import Parameters, datagen

pytestmark = pytest.mark.gpu

COLS = ("mic", "mas", "mev", "mcn", "pearson_r", "nonlinearity")


@pytest.fixture(scope="module")
def reference():
    import oracle as O
    if not os.path.exists(O.REF_SO):
        pytest.skip("oracle/_ref/libmine_ref.so (the compiled reference) is not present")
    return O.Reference()


def _check(got, want, what):
    g = np.stack([got[k] for k in COLS], axis=1)
    gb, wb = g.view(np.int64), np.ascontiguousarray(want).view(np.int64)
    assert g.shape == want.shape, what
    bad = np.nonzero((gb != wb).any(axis=1))[0]
    assert bad.size == 0, f"{what}: {bad.size} pairs differ, first {bad[:5]}"


@pytest.mark.parametrize("cfg,p", [(1, None), (2, 317), (3, 46)])
def test_pairwise_config_vs_reference(engine, reference, cfg, p):
    w = datagen.make(cfg)
    X = w.X if p is None else w.X[:p]
    got = engine.pairwise(X, Parameters(w.alpha, w.c, 0), stats=COLS)
    want = reference.run_analysis(X, w.alpha, w.c, workers=os.cpu_count() or 1)
    _check(got, want, f"c{cfg} ({X.shape[0]} variables)")


def test_c0_all_pairs_vs_reference(engine, reference):
    w = datagen.make(0)
    got = engine.pairs(w.X, w.xi, w.yi, Parameters(w.alpha, w.c, 0), stats=COLS)
    want = np.stack([reference.statistics(w.X[i], w.X[j], w.alpha, w.c) for i, j in zip(w.xi, w.yi)])
    _check(got, want, "c0 (all 256 pairs)")
