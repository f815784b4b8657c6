#!/usr/bin/env python3
"""Per-pair latency of the reference-API path (Engine.compute_statistics in a
loop, one pair per call = one mine::compute_score through the adapter):
python tools/per_pair_latency.py [n] [pairs]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_1208_4271_b200 import Engine, Parameters
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    pairs = int(sys.argv[2]) if len(sys.argv) > 2 else 300
    rng = np.random.default_rng(1)
    X = rng.standard_normal((pairs, n))
    Y = np.sin(3 * X) + 0.5 * rng.standard_normal((pairs, n))
    eng = Engine(0)
    p = Parameters(0.6, 15.0)
    for i in range(10):
        eng.compute_statistics(X[i], Y[i], p)
    t0 = time.perf_counter()
    for i in range(pairs):
        eng.compute_statistics(X[i], Y[i], p)
    dt = time.perf_counter() - t0
    print(json.dumps({"n": n, "pairs": pairs, "pairs_per_s": pairs / dt, "us_per_pair": dt / pairs * 1e6,
                      "launches_per_call": eng.last_launches}))


if __name__ == "__main__":
    main()
