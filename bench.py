#!/usr/bin/env python3
"""Headline benchmark: variable pairs/s (MIC+TIC) of the all-pairs MINE score
on config c1 (BASELINE.json configs[1]: 4381 variables x 23 samples, alpha=0.6,
c=15), on N B200s of one node.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full pass of the hot path (per-variable sort + equipartition,
then every pair's clumps / superclumps / exact OptimizeXAxis DP / reductions)
over the whole pair batch.  `value` is device-resident throughput (inputs in
HBM, CUDA events on the launching stream, L2 flushed before every step, max
over ranks); `e2e` is the same metric through the C ABI with pinned HOST
buffers (H2D of the variables and D2H of MIC+TIC inside the timed region).
Multi-GPU (torchrun): weak scaling -- the dataset grows to p = round(4381
sqrt(N)) variables so every GPU keeps ~9.59M pairs, sharded by contiguous
condensed-index range; no collective touches the data path.
`--impl reference` times the reference's own CPU engine (oracle/_ref, built
from /root/reference/proj/src) with all host threads on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "variable pairs/sec (MIC+TIC) at 1/2/4/8 B200 and % of limiting-pipe roofline"
UNIT = "pairs/s"
BASE_P = 4381


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def workload(n_gpus: int):
    from paper_1208_4271_b200 import datagen
    p = BASE_P if n_gpus == 1 else int(round(BASE_P * math.sqrt(n_gpus)))
    return datagen.config1(p=p), p


def config_dict(w, p, n_gpus, total):
    return {
        "workload": f"c1: all pairs of p={p} variables x n={w.n} samples (BASELINE configs[1]"
                    f"{'' if n_gpus == 1 else ', weak-scaled p=round(4381*sqrt(N))'}), "
                    f"alpha={w.alpha}, c={w.c}, est=MIC_approx",
        "p": p, "n": w.n, "pairs_per_step": total,
        "stats_written": ["mic", "tic"],
        "l2": "flushed (256 MiB write) before every timed step",
        "inputs": "HBM-resident (value); pinned host (e2e)",
        "parallelism": f"pairs sharded by condensed-index range over {n_gpus} GPU(s), no collective",
    }


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) during the timed region."""

    def __init__(self, device: int, period: float = 0.05):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self.device = period, device
        self._stop = threading.Event()
        self._th = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            log("clock sampler unavailable:", e)
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def hbm_line(bytes_per_launch: int, kern_s: float) -> dict:
    peak, src = None, None
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        peak, src = 7700.0, "B200 nominal (MEASURED_PEAKS.json absent)"
    ach = bytes_per_launch / kern_s / 1e9
    return {"achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "bytes_per_launch": int(bytes_per_launch), "peak_source": src}


def probe_peaks(device: int):
    import ctypes
    from paper_1208_4271_b200 import _build
    L = ctypes.CDLL(_build.PROBES)
    D = ctypes.POINTER(ctypes.c_double)
    L.mine_b200_probe.argtypes = [ctypes.c_int, D, D, D]
    a, b, c = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_double(0)
    if L.mine_b200_probe(device, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)) != 0:
        return None, None, None
    return a.value, b.value, c.value


def cpu_reference(w, p, budget_s: float, cores: int):
    """The reference's own run_analysis (oracle/_ref, the unmodified reference
    sources) on all pairs of the first p' variables, p' sized to ~budget_s."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    try:
        R = O.Reference()
        kind = "reference"
        run = lambda V: R.run_analysis(V, w.alpha, w.c, workers=cores)  # noqa: E731
    except FileNotFoundError:
        Or = O.Oracle()
        kind = "port"
        run = lambda V: Or.pairwise(V, w.alpha, w.c, threads=cores)  # noqa: E731
    cal = min(p, 120)
    t0 = time.perf_counter()
    run(w.X[:cal])
    rate = cal * (cal - 1) / 2 / max(time.perf_counter() - t0, 1e-6)
    target = rate * budget_s
    pp = int(min(p, max(cal, (1 + math.sqrt(1 + 8 * target)) / 2)))
    t0 = time.perf_counter()
    out = run(w.X[:pp])
    dt = time.perf_counter() - t0
    pairs = pp * (pp - 1) // 2
    assert len(out) == pairs
    return {"value": pairs / dt, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"all {pairs} pairs of the first {pp} of the {p} c1 variables "
                      f"(run_analysis, workers={cores}), {dt:.1f} s"}


# ---------------------------------------------------------------------------
def run_reference(args, world, rank):
    if rank != 0:
        return
    w, p = workload(world)
    cores = os.cpu_count() or 1
    per_step = max(2.0, min(20.0, 150.0 / max(args.steps + args.warmup, 1)))
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference(w, p, per_step, cores)
        if i >= args.warmup:
            vals.append(r["value"])
    v = statistics.median(vals)
    total = p * (p - 1) // 2
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / v * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded c1 generator, numpy PCG64 seed 43)",
        "config": config_dict(w, p, world, total),
        "cpu_baseline": {**r, "value": v},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import torch
    from paper_1208_4271_b200 import Engine, Parameters
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    w, p = workload(world)
    n = w.n
    total = p * (p - 1) // 2
    first = rank * total // world
    count = (rank + 1) * total // world - first
    params = Parameters(w.alpha, w.c, 0)
    eng = Engine(local)

    dv = torch.from_numpy(w.X).to(dev).contiguous()
    outs = {k: torch.empty(count, dtype=torch.float64, device=dev) for k in ("mic", "tic")}
    ptrs = {k: t.data_ptr() for k, t in outs.items()}
    stream = torch.cuda.Stream(dev)  # a real stream: the engine enqueues on it
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step(kb=None, ke=None):
        eng.pairwise_device(dv.data_ptr(), p, n, params, ptrs, stream=stream.cuda_stream,
                            first=first, count=count, ev_begin=kb or 0, ev_end=ke or 0)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    # untimed instrumented pass: realised algorithmic work of one step
    work = eng.pairwise_device(dv.data_ptr(), p, n, params, ptrs, stream=stream.cuda_stream,
                               first=first, count=count, counters=True)
    launches = eng.last_launches
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    kern_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    for a, b in kern_ev:  # materialise the events so their handles exist
        a.record(stream)
        b.record(stream)
    torch.cuda.synchronize()

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            step_ev[i][0].record(stream)
            step(kern_ev[i][0].cuda_event, kern_ev[i][1].cuda_event)
            step_ev[i][1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in step_ev]
    kern_ms = [a.elapsed_time(b) for a, b in kern_ev]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot.item())
    value = total * args.steps / (total_ms / 1e3)

    # ---- e2e: the C-ABI call with pinned host buffers -----------------------
    xin = torch.from_numpy(w.X).pin_memory().numpy()
    hout = {k: torch.empty(count, dtype=torch.float64).pin_memory().numpy() for k in ("mic", "tic")}
    for _ in range(max(1, args.warmup)):
        eng.pairwise_host(xin, params, hout, first, count)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        eng.pairwise_host(xin, params, hout, first, count)
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = total * args.steps / float(e2e_s.item())
    same = bool(np.array_equal(hout["mic"].view(np.int64), outs["mic"].cpu().numpy().view(np.int64)))

    if rank == 0:
        dadd, lds, lds2 = probe_peaks(local)
        kern_s = statistics.mean(kern_ms) / 1e3
        g8, g2 = work["gathers"], work["rank_gathers"]
        gathers = g8 + g2
        achieved = gathers / kern_s / 1e9
        # mixed-width peak: the rate at which the LSU would serve this exact
        # mix of 8-byte and 2-byte gathers (time-weighted harmonic mean)
        lds = gathers / (g8 / lds + g2 / lds2) if lds and lds2 and gathers else None
        traffic = None
        try:
            t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))["k_memo_pairs"]
            traffic = int(t["dram_bytes_read"] + t["dram_bytes_write"])
        except Exception:
            pass
        roof = {"bound": "lsu", "achieved": achieved, "peak": lds / 1e9 if lds else None,
                "unit": "Ggather/s", "frac": achieved / (lds / 1e9) if lds else None,
                "traffic": traffic,
                "traffic_source": "profiles/ncu_traffic.json (dram read+write bytes per launch, ncu)",
                "kernel": "k_memo_pairs (the pair-scoring launch of a step)",
                "per_launch_work": {k: int(v) * world for k, v in work.items()},
                "work_unit": "shared-memory table gathers the memo-tier algorithm needs "
                             "(one 2 B dense candidate rank per F(t,2) candidate, 2 x 8 B per "
                             "level-3 span term, 2 B rank per standard 3-row candidate, 7 x 8 B "
                             "per other 3-row candidate), counted by the kernel; DESIGN.md "
                             "'Roofline'",
                "gathers_8b": int(g8) * world, "gathers_rank": int(g2) * world,
                "peak_source": "measured live: probes.cu k_lds (random 8 B gathers, 561-entry "
                               "table) and k_lds2 (random 2 B gathers, 16K-entry table), 8 "
                               "streams/thread, all SMs; peak = time-weighted mix of the two",
                "kernel_ms": statistics.mean(kern_ms),
                # the HBM roofline for the same launch, for completeness: the
                # algorithmic bytes are the outputs (MIC + TIC, 16 B per pair)
                # plus the per-variable records read (96 B per variable)
                "hbm": hbm_line(16 * count + 96 * p, kern_s),
                "secondary": {"bound": "fp64", "achieved": work["fp64_ops"] / kern_s / 1e12,
                              "peak": dadd / 1e12 if dadd else None, "unit": "TFLOP/s",
                              "frac": (work["fp64_ops"] / kern_s) / dadd if dadd else None,
                              "work_unit": "FP64 ops the reference's entropy/DP arithmetic "
                                           "executes for the same pairs (memoised here)",
                              "peak_source": "measured live: probes.cu k_dadd"}}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded c1 generator, numpy PCG64 seed 43)",
            "config": config_dict(w, p, world, total),
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(w.X.nbytes) * world,
                    "d2h_bytes_per_step": int(total * 8 * 2),
                    "matches_value_leg": same},
            "gpu_launches": int(launches) * args.steps * world,
            "clocks": clk.summary(),
            "roofline": roof,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_reference(w, p, args.cpu_seconds, os.cpu_count() or 1)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_config(args):
    """Secondary measurement on another BASELINE config (not the headline):
    device-resident pairs/s over a bounded window of the config's pair space,
    plus the reference CPU engine on a subsample of the same window."""
    import torch
    from paper_1208_4271_b200 import Engine, Parameters, datagen
    w = datagen.make(args.config)
    eng = Engine(0)
    params = Parameters(w.alpha, w.c, w.est)
    total = w.npairs
    count = min(total, args.pairs) if args.pairs else total
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    cnt = None

    def call():
        if w.call == "pairwise":
            return eng.pairwise(w.X, params, first=0, count=count, stats=("mic", "tic"))
        if w.call == "cross":
            return eng.cross(w.X, w.Y, params, first=0, count=count, stats=("mic", "tic"))
        return eng.pairs(w.X, w.xi[:count], w.yi[:count], params, stats=("mic", "tic"))

    call()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    dt = statistics.median(times)
    line = {"config": args.config, "call": w.call, "pairs": count, "n": w.n, "alpha": w.alpha,
            "c": w.c, "est": w.est, "e2e_pairs_per_s": count / dt, "e2e_s": dt,
            "launches": eng.last_launches}
    # FP64 roofline of the whole call: the FP64 ops the
    # reference's op sequence needs for these pairs (entropy sums with the
    # p*log(p) terms as lookups, span terms, and DMUL + DADD + DSETP per DP
    # candidate), counted by the kernels, at the measured DADD issue rate
    eng.count_work = True
    call()
    eng.count_work = False
    work = eng.last_work
    dadd = probe_peaks(0)[0]
    if dadd:
        line["roofline"] = {"bound": "fp64", "achieved": work["fp64_ops"] / dt / 1e12,
                            "peak": dadd / 1e12, "unit": "TFLOP/s",
                            "frac": work["fp64_ops"] / dadd / dt,
                            "work": {k: int(work[k]) for k in ("fp64_ops", "dp_candidates",
                                                               "span_entries", "point_visits",
                                                               "subproblems")},
                            "work_unit": "FP64 ops of the reference's arithmetic (p log p terms "
                                         "as lookups; DMUL+DADD+DSETP per DP candidate), counted "
                                         "by the kernels; time = the whole call (e2e_s)",
                            "peak_source": "measured live: probes.cu k_dadd"}
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        orc = O.Oracle()
        sub = max(1, min(count, args.cpu_pairs))
        t0 = time.perf_counter()
        if w.call == "pairwise":
            ref = orc.pairwise(w.X, w.alpha, w.c, w.est, first=0, count=sub)
        elif w.call == "cross":
            idx = np.arange(sub)
            ref = orc.pairs(np.concatenate([w.X, w.Y]), idx // w.Y.shape[0],
                            w.X.shape[0] + idx % w.Y.shape[0], w.alpha, w.c, w.est)
        else:
            ref = orc.pairs(w.X, w.xi[:sub], w.yi[:sub], w.alpha, w.c, w.est)
        cdt = time.perf_counter() - t0
        got = call()
        line["cpu_port_pairs_per_s"] = sub / cdt
        line["cpu_sample_pairs"] = sub
        line["cpu_cores"] = os.cpu_count()
        line["bit_exact_on_sample"] = bool(np.array_equal(got["mic"][:sub].view(np.int64),
                                                          ref[:, 0].view(np.int64)))
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1,
                    help="1 = the headline (c1); 0/2/3/4 = secondary timing of that config")
    ap.add_argument("--pairs", type=int, default=0, help="secondary configs: pairs to time (0 = all)")
    ap.add_argument("--cpu-pairs", type=int, default=200)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world == 1 and args.gpus > 1:
        log(f"--gpus {args.gpus} without torchrun: running one rank")
    if args.config != 1:
        run_config(args)
    elif args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
