#!/usr/bin/env python3
"""Small cases of every kernel family, run against the bounds-checked
library (device asserts on the general tier's scratch / slot / layout
indexing; compute-sanitizer is closed on this GPU pool):

    MINE_B200_LIB=paper_1208_4271_b200/libmine_b200_checked.so python tools/sanitize_cases.py

(tests/test_bounds_checked_gpu.py).  Where compute-sanitizer is available the
same script runs under it, one tool per process:

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py

memo tier (n = 23 sorted batches and n = 28 compact tables), tiny tier,
general tier (k_part_f2 both widths, k_dp lean / wide / ring / global-table
variants, k_dp_warp) with cells, the debug export, Pearson, the GPU record
formatter and the multi-device pool.  Each case is checked against the oracle
so a sanitizer-clean run is also a correct one."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]


def main():
    import oracle as O
    from conftest import random_pair
    from paper_1208_4271_b200 import Engine, Parameters, datagen
    orc = O.Oracle()
    eng = Engine(0)
    cols = ["mic", "mas", "mev", "mcn", "mic_e", "tic"]

    def check(res, want, what):
        got = np.stack([res[k] for k in cols], axis=1)
        assert np.array_equal(got.view(np.int64), want.view(np.int64)), what
        print("ok", what, flush=True)

    rng = np.random.default_rng(11)
    V = datagen.make(1).X[:70]
    check(eng.pairwise(V, tier=3), orc.pairwise(V, threads=4), "memo n=23")
    check(eng.pairwise(V, tier=1), orc.pairwise(V, threads=4), "tiny n=23")
    V28 = rng.standard_normal((40, 28))
    V28[::5] = np.round(V28[::5])
    check(eng.pairwise(V28), orc.pairwise(V28, threads=4), "memo n=28")
    w0 = datagen.make(0, npairs=6)
    p0 = Parameters(w0.alpha, w0.c, w0.est)
    check(eng.pairs(w0.X, w0.xi, w0.yi, p0, cells=True), orc.pairs(w0.X, w0.xi, w0.yi, w0.alpha, w0.c, w0.est),
          "general c0 (lean k_dp, warp path, both k_part_f2 widths)")
    w2 = datagen.make(2)
    V2 = w2.X[[0, 1, 2, 3, 10, 11, 500, 501, 1000, 1001, 1998, 1999, 7, 8, 9, 40, 41, 42]]
    p2 = Parameters(w2.alpha, w2.c, w2.est)
    check(eng.pairwise(V2, p2), orc.pairwise(V2, w2.alpha, w2.c, w2.est),
          "general c2 ties (row-map dedup, warp partition kernel, warp DP width classes)")
    xs, ys = [], []
    for it in range(8):
        x, y = random_pair(rng, 300, it % 4)
        xs += [x]
        ys += [y]
    VV = np.stack(xs + ys)
    xi, yi = np.arange(8), np.arange(8, 16)
    check(eng.pairs(VV, xi, yi, Parameters(0.85, 15.0, 1)), orc.pairs(VV, xi, yi, 0.85, 15.0, 1),
          "general alpha=.85 (wide / ring k_dp)")
    d = eng.debug_subproblem(xs[0], ys[0], 3, 5, 20)
    dd = orc.subproblem(xs[0], ys[0], 3, 5, 20)
    assert d["k"] == dd["k"] and np.array_equal(d["bounds"], dd["bounds"]), "debug export"
    print("ok debug export", flush=True)
    r = eng.pairs(VV, xi, yi, Parameters(0.6, 15.0, 0), stats=("mic", "pearson_r", "nonlinearity"))
    want = np.array([orc.pearson(VV[a], VV[b]) for a, b in zip(xi, yi)])
    assert np.array_equal(r["pearson_r"].view(np.int64), want.view(np.int64)), "pearson"
    print("ok pearson", flush=True)
    res = eng.pairwise(V, devices=[0, 0], shard_chunk=100)
    check(res, orc.pairwise(V, threads=4), "virtual shards")
    from paper_1208_4271_b200 import engine as E
    L = E.load_library()
    L.mine_b200_check_format.restype = __import__("ctypes").c_longlong
    L.mine_b200_check_format.argtypes = [__import__("ctypes").c_longlong, __import__("ctypes").c_ulonglong,
                                         __import__("ctypes").c_int]
    assert L.mine_b200_check_format(20000, 7, 0) == 0, "GPU formatter"
    print("ok formatter", flush=True)
    print("ALL OK", flush=True)


if __name__ == "__main__":
    main()
