"""Full-size c4 fixtures from the REFERENCE itself (oracle/_ref/libmine_ref.so).

BASELINE configs[4]: 64 x 64 cross, n = 10,000, alpha = .75 (B = 1000), c = 15.
The CPU reference takes seconds (functional pairs) to minutes (noisy and
independent pairs, where k reaches thousands of clumps at y = 2) per pair, so
this runs once in the build container:

    python tests/golden/make_golden_c4.py [workers]

For each chosen (i, j) of the c4 cross it calls the reference's compute_score
once and its own reductions mic/mas/mev/mcn over that matrix
(char_matrix.cpp:70-81, statistics.cpp:10-37; oracle/ref_capi.cpp
ref_score_statistics) and stores the cells in for_each order.  The inputs are
not stored: datagen.config4() regenerates them bit-for-bit on the GPU box
(seeded PCG64); a checksum of the used rows guards against drift.

Pairs: every Y function (f0..f3) at both noise levels, the independent
(replaced) Y variables, and a few more X rows -- functional pairs have few
clumps, noisy ones reach k ~ n/2 at y = 2 and x_max = 500 (the 128-level F
ring of the GPU DP), independent ones hit k-hat.
"""
import ctypes
import hashlib
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
from paper_1208_4271_b200 import datagen  # noqa: E402

ALPHA, C = 0.75, 15.0
OUT = os.path.join(HERE, "ref_c4_full.npz")
NPAIRS = 32


def rows_digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:32]


def choose_pairs(w) -> list[tuple[int, int]]:
    u = w.X.mean(axis=0)
    resid = np.array([np.std(w.Y[j] - datagen._FUNCS[j % 4](u)) for j in range(w.Y.shape[0])])
    sigma = np.array([[0.05, 0.5][j % 2] for j in range(w.Y.shape[0])])
    indep = [j for j in range(w.Y.shape[0]) if abs(resid[j] - sigma[j]) > 0.05]  # replaced by U[0,1)
    js = list(range(8)) + [j for j in indep if j >= 8]
    pairs = [(j % w.X.shape[0], j) for j in js]
    extra = [(10, 8), (21, 11), (33, 14), (47, 19), (63, 63), (5, 30), (11, 9), (12, 10),
             (13, 12), (14, 13), (15, 15), (16, 16), (17, 17), (18, 18), (19, 20), (20, 21),
             (23, 23), (24, 24), (50, 25), (51, 26)]
    for p in extra:
        if len(pairs) >= NPAIRS:
            break
        if p not in pairs:
            pairs.append(p)
    return pairs[:NPAIRS], indep


def score_one(args):
    i, j = args
    w = datagen.config4()
    R = O.Reference()
    f = R.L.ref_score_statistics
    f.argtypes = [ctypes.c_int, O._dp, O._dp, ctypes.c_double, ctypes.c_double, O._ip, O._dp, O._dp]
    x = np.ascontiguousarray(w.X[i])
    y = np.ascontiguousarray(w.Y[j])
    n = x.size
    b = O.grid_bound(n, ALPHA)
    cells = np.zeros(len(O.cell_shapes(b)))
    out = np.zeros(4)
    bd = np.zeros(1, np.int32)
    t = time.time()
    R._check(f(n, O._d(x), O._d(y), ALPHA, C, O._i(bd), O._d(cells), O._d(out)))
    dt = time.time() - t
    print(f"pair ({i},{j}): {dt:.1f} s  mic={out[0]:.6f} mcn={out[3]:.4f}", flush=True)
    return i, j, cells, out, dt


def main():
    workers = int(sys.argv[1]) if len(sys.argv) > 1 else max(1, (os.cpu_count() or 2) - 1)
    if not os.path.exists(O.REF_SO):
        O.build(reference=True)
    w = datagen.config4()
    pairs, indep = choose_pairs(w)
    print("pairs:", pairs, "independent Y:", indep, flush=True)
    # longest first (independent / noisy), so the pool drains evenly
    order = sorted(pairs, key=lambda p: -(p[1] in indep) * 2 - (p[1] % 2))
    t0 = time.time()
    with Pool(workers) as pool:
        res = {(i, j): (cells, out, dt) for i, j, cells, out, dt in pool.imap_unordered(score_one, order)}
    cells = np.stack([res[p][0] for p in pairs])
    stats = np.stack([res[p][1] for p in pairs])
    secs = np.array([res[p][2] for p in pairs])
    xi = np.array([p[0] for p in pairs], np.int32)
    yi = np.array([p[1] for p in pairs], np.int32)
    np.savez_compressed(OUT, xi=xi, yi=yi, cells=cells, stats=stats, cpu_seconds=secs,
                        alpha=ALPHA, c=C, n=w.X.shape[1],
                        x_digest=rows_digest(w.X[xi]), y_digest=rows_digest(w.Y[yi]))
    print(f"wrote {OUT}: {len(pairs)} pairs, {time.time() - t0:.0f} s wall, "
          f"{secs.sum():.0f} s CPU", flush=True)


if __name__ == "__main__":
    main()
