#!/usr/bin/env python3
"""Device-resident timing of one general-tier call (CUDA events around the
whole call on its stream), for a BASELINE config window.

    python tools/gen_timing.py CONFIG PAIRS [REPS]

Prints one JSON line: device seconds per call (median), pairs/s, launches,
and the realised work.  Used with ncu's launch list to split a call's time
by kernel (tools/gen_profile.sh)."""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1208_4271_b200 import Engine, Parameters, datagen
    cfg, pairs = int(sys.argv[1]), int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    w = datagen.make(cfg)
    eng = Engine(0)
    params = Parameters(w.alpha, w.c, w.est)
    dev = torch.device("cuda", 0)
    if w.call == "pairwise":
        V = w.X
        count = min(pairs, V.shape[0] * (V.shape[0] - 1) // 2)
        xi = yi = None
    elif w.call == "cross":
        V = np.ascontiguousarray(np.concatenate([w.X, w.Y]))
        count = min(pairs, w.X.shape[0] * w.Y.shape[0])
        xi = (np.arange(count) // w.Y.shape[0]).astype(np.int32)
        yi = (w.X.shape[0] + np.arange(count) % w.Y.shape[0]).astype(np.int32)
    else:
        V = w.X
        xi, yi = w.xi[:pairs].astype(np.int32), w.yi[:pairs].astype(np.int32)
        count = xi.size
    dV = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
    outs = {k: torch.empty(count, dtype=torch.float64, device=dev) for k in ("mic", "tic")}
    ptr = {k: t.data_ptr() for k, t in outs.items()}
    dxi = torch.from_numpy(xi).to(dev) if xi is not None else None
    dyi = torch.from_numpy(yi).to(dev) if yi is not None else None
    kind = "pairwise" if xi is None else "pairs"
    s = torch.cuda.current_stream(dev)

    def call(counters=False):
        return eng.device_call(kind, params, ptr, vars_ptr=dV.data_ptr(), p=V.shape[0], n=V.shape[1],
                               xi_ptr=dxi.data_ptr() if dxi is not None else 0,
                               yi_ptr=dyi.data_ptr() if dyi is not None else 0, npairs=count,
                               count=count if kind == "pairwise" else 0, stream=s.cuda_stream,
                               counters=counters)

    call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        call()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    work = call(counters=True)
    dt = statistics.median(ts)
    print(json.dumps({"config": cfg, "pairs": count, "device_s": dt, "pairs_per_s": count / dt,
                      "all_s": ts, "launches": eng.last_launches,
                      "work": {k: int(v) for k, v in work.items()}}), flush=True)


if __name__ == "__main__":
    main()
