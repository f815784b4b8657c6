"""Memo-tier throughput by sample count n (device-resident, random data,
p variables -> p(p-1)/2 pairs, MIC + TIC), CUDA-event timed.  Used for the
DESIGN.md memo table:  python tools/memo_n_sweep.py [p] [n ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1208_4271_b200 import Engine, Parameters  # noqa: E402


def main():
    p = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    ns = [int(a) for a in sys.argv[2:]] or [16, 20, 23, 24, 25, 26, 28, 30, 31]
    eng = Engine(0)
    stream = torch.cuda.Stream()  # a real stream: the engine enqueues on it
    torch.cuda.set_stream(stream)
    prm = Parameters(0.6, 15.0)
    npairs = p * (p - 1) // 2
    for n in ns:
        rng = np.random.default_rng(n)
        X = torch.tensor(rng.uniform(size=(p, n)), device="cuda", dtype=torch.float64)
        outs = {k: torch.empty(npairs, device="cuda", dtype=torch.float64) for k in ("mic", "tic")}
        ptrs = {k: v.data_ptr() for k, v in outs.items()}
        s = stream.cuda_stream
        for _ in range(3):
            eng.pairwise_device(X.data_ptr(), p, n, prm, ptrs, stream=s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(stream)
        for _ in range(reps):
            eng.pairwise_device(X.data_ptr(), p, n, prm, ptrs, stream=s)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"n": n, "p": p, "pairs": npairs, "ms": round(ms, 4),
                          "gpairs_per_s": round(npairs / ms / 1e6, 3)}))


if __name__ == "__main__":
    main()
