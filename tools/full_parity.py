"""Full-size parity run (GPU box): the engine against the reference's own
engine (oracle/_ref/libmine_ref.so, run_analysis with all host threads) on
whole BASELINE configs -- c0 (all 256 pairs), c1 (all 9,594,390 pairs), c2
(all 1,999,000 pairs) -- and a c3 window.  Compares MIC, MAS, MEV, MCN,
Pearson r and non-linearity bit for bit; prints one JSON line per config.
Test infrastructure: imports oracle/ only as the checker.
usage: python tools/full_parity.py [c3_pairs]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_1208_4271_b200 import Engine, Parameters, datagen  # noqa: E402

COLS = ("mic", "mas", "mev", "mcn", "pearson_r", "nonlinearity")


def compare(got, ref):
    g = np.stack([got[k] for k in COLS], axis=1)
    gb, rb = g.view(np.int64), np.ascontiguousarray(ref).view(np.int64)
    bad = np.nonzero((gb != rb).any(axis=1))[0]
    return int(bad.size), [int(i) for i in bad[:5]]


def main():
    c3_pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
    eng, ref = Engine(0), O.Reference()
    cores = os.cpu_count() or 1
    for cfg in (0, 1, 2, 3):
        w = datagen.make(cfg)
        prm = Parameters(w.alpha, w.c, 0)
        t0 = time.perf_counter()
        if w.call == "pairs":
            got = eng.pairs(w.X, w.xi, w.yi, prm, stats=COLS)
            tg = time.perf_counter() - t0
            t0 = time.perf_counter()
            want = np.stack([ref.statistics(w.X[i], w.X[j], w.alpha, w.c) for i, j in zip(w.xi, w.yi)])
            npairs = len(w.xi)
        else:
            X = w.X
            count = None
            if cfg == 3:  # a window: the CPU engine needs ~10 ms per c3 pair
                p = int((1 + np.sqrt(1 + 8 * c3_pairs)) / 2) + 1
                X = w.X[:p]
                count = p * (p - 1) // 2
            got = eng.pairwise(X, prm, stats=COLS)
            tg = time.perf_counter() - t0
            t0 = time.perf_counter()
            want = ref.run_analysis(X, w.alpha, w.c, workers=cores)
            npairs = X.shape[0] * (X.shape[0] - 1) // 2
        tr = time.perf_counter() - t0
        nbad, first = compare(got, want)
        print(json.dumps({"config": cfg, "pairs": npairs, "n": int(w.X.shape[1]), "mismatching_pairs": nbad,
                          "first_mismatches": first, "stats": list(COLS), "gpu_s": round(tg, 3),
                          "reference_s": round(tr, 1), "reference_threads": cores}), flush=True)


if __name__ == "__main__":
    main()
