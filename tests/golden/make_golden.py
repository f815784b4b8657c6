"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/
libmine_ref.so, compiled unmodified from /root/reference/proj/src).  Run in
the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The fixtures travel with the repo, so the GPU box (no /root/reference) can
check the engine against the reference's own outputs.  Inputs are seeded
numpy draws in the styles of the reference's tests/test_helpers.hpp:49-79
(continuous / tied / monotone / constant_y) plus slices of the BASELINE
configs; nothing here is copied from the reference's test files.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.dirname(HERE))

import oracle as O  # noqa: E402
from conftest import random_pair  # noqa: E402
from paper_1208_4271_b200 import datagen  # noqa: E402


def pairs_fixture(R):
    rng = np.random.default_rng(20261020)
    xs, ys, meta, cells, stats = [], [], [], [], []
    for it in range(160):
        n = int(rng.integers(2, 160)) if it % 5 else int(rng.integers(2, 40))
        alpha = [0.6, 0.5, 0.75, 0.45, 1.0][it % 5] if n < 120 else 0.6
        c = [15.0, 1.0, 2.5, 40.0, 0.8][(it // 5) % 5]
        x, y = random_pair(rng, n, it % 4)
        b, m = R.score(x, y, alpha, c)
        s = R.statistics(x, y, alpha, c)
        xs.append(x)
        ys.append(y)
        meta.append((n, alpha, c, b))
        cells.append(m)
        stats.append(s[:6])
    off = np.cumsum([0] + [len(x) for x in xs])
    coff = np.cumsum([0] + [len(m) for m in cells])
    np.savez_compressed(os.path.join(HERE, "ref_pairs.npz"),
                        x=np.concatenate(xs), y=np.concatenate(ys), off=off,
                        n=np.array([m[0] for m in meta]), alpha=np.array([m[1] for m in meta]),
                        c=np.array([m[2] for m in meta]), bound=np.array([m[3] for m in meta]),
                        cells=np.concatenate(cells), coff=coff, stats=np.array(stats)[:, :4],
                        stats6=np.array(stats))


def subproblem_fixture(R):
    rng = np.random.default_rng(404404)
    rows = []
    xs, ys = [], []
    q_all, b_all, v_all = [], [], []
    for it in range(60):
        n = int(rng.integers(2, 200))
        x, y = random_pair(rng, n, it % 4)
        yt, xm, kh = int(rng.integers(2, 12)), int(rng.integers(2, 9)), int(rng.integers(1, 40))
        d = R.subproblem(x, y, yt, xm, kh)
        xs.append(x)
        ys.append(y)
        rows.append((n, yt, xm, kh, d["row_count"], d["clump_count"], d["k"], d["h_q"]))
        b_all.append(d["bounds"])
        v_all.append(d["values"])
    np.savez_compressed(os.path.join(HERE, "ref_subproblems.npz"),
                        x=np.concatenate(xs), y=np.concatenate(ys),
                        off=np.cumsum([0] + [len(x) for x in xs]),
                        meta=np.array([r[:7] for r in rows], dtype=np.int64),
                        h_q=np.array([r[7] for r in rows]),
                        bounds=np.concatenate(b_all), boff=np.cumsum([0] + [len(b) for b in b_all]),
                        values=np.concatenate(v_all), voff=np.cumsum([0] + [len(v) for v in v_all]))


def configs_fixture(R):
    """Reference run_analysis / compute_statistics on slices of c0..c3 and a
    reduced-n c4 (the full c4 pair costs the CPU reference minutes)."""
    out = {}
    w1 = datagen.make(1)
    out["c1_vars"] = w1.X[:60]
    c1 = R.run_analysis(w1.X[:60], w1.alpha, w1.c, workers=8)
    out["c1_stats"] = c1[:, :4]
    out["c1_stats6"] = c1[:, :6]  # + pearson_r, nonlinearity (statistics.cpp:39-51)
    w0 = datagen.make(0, npairs=10)
    out["c0_vars"] = w0.X
    out["c0_stats"] = np.array([R.statistics(w0.X[2 * i], w0.X[2 * i + 1], 0.6, 15.0)[:4]
                                for i in range(10)])
    w2 = datagen.make(2)
    out["c2_vars"] = w2.X[:6]
    out["c2_stats"] = R.run_analysis(w2.X[:6], w2.alpha, w2.c, workers=8)[:, :4]
    w3 = datagen.make(3)
    out["c3_vars"] = w3.X[:4]
    out["c3_stats"] = R.run_analysis(w3.X[:4], w3.alpha, w3.c, workers=8)[:, :4]
    w4 = datagen.config4(px=2, py=2, n=1500)
    out["c4r_X"], out["c4r_Y"] = w4.X, w4.Y
    out["c4r_stats"] = np.array([R.statistics(w4.X[i], w4.Y[j], 0.75, 15.0)[:4]
                                 for i in range(2) for j in range(2)])
    np.savez_compressed(os.path.join(HERE, "ref_configs.npz"), **out)


if __name__ == "__main__":
    if not os.path.exists(O.REF_SO):
        O.build(reference=True)
    R = O.Reference()
    pairs_fixture(R)
    subproblem_fixture(R)
    configs_fixture(R)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")
