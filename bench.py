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
Multi-GPU (torchrun): strong scaling by default -- the unchanged c1 (all
9,594,390 pairs) is sharded by contiguous condensed-index range, each rank
scores its slice and the slices are gathered to rank 0 inside the timed
region (the only collective; none on the data path).  `--scaling weak` grows
the dataset to p = round(4381 sqrt(N)) so every GPU keeps ~9.59M pairs.
`--impl reference` times the reference's own CPU engine (oracle/_ref, built
from /root/reference/proj/src) with all host threads: whole c1 steps (all
9.59M pairs each), at most 1 warm-up + 3 timed steps so the arm ends in
about a minute.
The default line also carries `secondary`: the other BASELINE configs (c0 all
256 pairs, c2 a 20k-pair window, c3 a 4k-pair window, c4 148 pairs) with
device and end-to-end pairs/s, SURVEY 8(d)'s roofline, the reference engine's
CPU rate on a sample and a bit-exact-on-sample flag.
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


def workload(n_gpus: int, scaling: str = "strong"):
    from paper_1208_4271_b200 import datagen
    p = BASE_P if (n_gpus == 1 or scaling == "strong") else int(round(BASE_P * math.sqrt(n_gpus)))
    return datagen.config1(p=p), p


def config_dict(w, p, n_gpus, total, scaling="strong"):
    weak = n_gpus > 1 and scaling == "weak"
    return {
        "workload": f"c1: all pairs of p={p} variables x n={w.n} samples (BASELINE configs[1]"
                    f"{', weak-scaled p=round(4381*sqrt(N))' if weak else ''}), "
                    f"alpha={w.alpha}, c={w.c}, est=MIC_approx",
        "p": p, "n": w.n, "pairs_per_step": total,
        "stats_written": ["mic", "tic"],
        "l2": "flushed (256 MiB write) before every timed step",
        "inputs": "HBM-resident (value); pinned host (e2e)",
        "parallelism": f"pairs sharded by condensed-index range over {n_gpus} GPU(s); "
                       + ("slices gathered to rank 0 inside the timed region (NCCL all_gather)"
                          if n_gpus > 1 else "no collective"),
    }


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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


def probe_general(device: int, table_bytes: float):
    """Random 8-byte L2 gathers/s from a table of `table_bytes` (the span
    terms' p*log(p) lookups) and exact DP candidates/s (probes.cu)."""
    import ctypes
    from paper_1208_4271_b200 import _build
    L = ctypes.CDLL(_build.PROBES)
    D = ctypes.POINTER(ctypes.c_double)
    L.mine_b200_probe_general.argtypes = [ctypes.c_int, ctypes.c_double, D, D]
    a, b = ctypes.c_double(0), ctypes.c_double(0)
    if L.mine_b200_probe_general(device, float(table_bytes), ctypes.byref(a), ctypes.byref(b)) != 0:
        return None, None
    return a.value, b.value


def roofline_8d(work: dict, t_s: float, out_bytes: int, peaks: dict) -> dict:
    """T_roof = max(2 C / R_fp64, N_pv / R_lsu, bytes_out / BW)
    with C = every DP candidate of levels l = 2 .. l_max (F(t,2) included),
    N_pv = the partition's point visits; fraction = T_roof / t_s."""
    C = int(work["dp_candidates"]) + int(work.get("f2_candidates", 0))
    npv = int(work["point_visits"])
    terms = {"fp64": 2 * C / peaks["fp64_per_s"],
             "lsu": npv / peaks["lsu_per_s"],
             "hbm": out_bytes / (peaks["hbm_gbs"] * 1e9)}
    bound = max(terms, key=terms.get)
    return {"t_roof_s": terms[bound], "bound": bound, "terms_s": terms, "t_measured_s": t_s,
            "frac": terms[bound] / t_s, "C": C, "N_pv": npv, "bytes_out": int(out_bytes),
            "peaks": {"R_fp64 (DADD/s, probes.cu k_dadd)": peaks["fp64_per_s"],
                      "R_lsu (random 8 B shared gathers/s, probes.cu k_lds)": peaks["lsu_per_s"],
                      "BW_hbm (GB/s, MEASURED_PEAKS.json)": peaks["hbm_gbs"]}}


def measured_peaks(device: int) -> dict:
    dadd, lds, lds2 = probe_peaks(device)
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm = 6650.0
    return {"fp64_per_s": dadd, "lsu_per_s": lds, "lsu2_per_s": lds2, "hbm_gbs": hbm}


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
            "cpu_model": cpu_model(),
            "sample": f"all {pairs} pairs of the first {pp} of the {p} c1 variables "
                      f"(run_analysis, workers={cores}), {dt:.1f} s"}


# ---------------------------------------------------------------------------
def run_reference(args, world, rank):
    """The reference's own run_analysis (oracle/_ref: the unmodified
    reference sources) over ALL c1 pairs per step, all host threads.  A step
    takes ~18 s on 16 cores, so at most 1 warm-up + 3 timed steps run (the
    JSON says how many; steps_requested keeps the driver's K / W)."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    w, p = workload(world, args.scaling)
    cores = os.cpu_count() or 1
    try:
        R = O.Reference()
        kind = "reference"
        run = lambda: R.run_analysis(w.X, w.alpha, w.c, workers=cores)  # noqa: E731
    except FileNotFoundError:
        Or = O.Oracle()
        kind = "port"
        run = lambda: Or.pairwise(w.X, w.alpha, w.c, threads=cores)  # noqa: E731
    total = p * (p - 1) // 2
    warm, steps = min(args.warmup, 1), max(1, min(args.steps, 3))
    for _ in range(warm):
        run()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        out = run()
        times.append(time.perf_counter() - t0)
        assert len(out) == total
    dt = sum(times)
    v = total * steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": warm,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": dt / steps * 1e3,
        "higher_is_better": True, "scaling": args.scaling if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded c1 generator, numpy PCG64 seed 43)",
        "config": config_dict(w, p, world, total, args.scaling),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"whole c1 steps: all {total} pairs per step "
                                   f"(run_analysis, workers={cores}); {warm} warm-up + "
                                   f"{steps} timed steps, {dt:.1f} s timed"},
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

    w, p = workload(world, args.scaling)
    n = w.n
    total = p * (p - 1) // 2
    first = rank * total // world
    count = (rank + 1) * total // world - first
    slot = (total + world - 1) // world  # equal gather slots (the last ones padded)
    params = Parameters(w.alpha, w.c, 0)
    eng = Engine(local)

    dv = torch.from_numpy(w.X).to(dev).contiguous()
    outs = {k: torch.empty(slot, dtype=torch.float64, device=dev) for k in ("mic", "tic")}
    ptrs = {k: t.data_ptr() for k, t in outs.items()}
    gathered = ({k: torch.empty(slot * world, dtype=torch.float64, device=dev) for k in outs}
                if dist else None)
    stream = torch.cuda.Stream(dev)  # a real stream: the engine enqueues on it
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step(kb=None, ke=None):
        eng.pairwise_device(dv.data_ptr(), p, n, params, ptrs, stream=stream.cuda_stream,
                            first=first, count=count, ev_begin=kb or 0, ev_end=ke or 0)
        if dist:  # the final gather of the condensed slices (strong and weak)
            for k in outs:
                dist.all_gather_into_tensor(gathered[k], outs[k])

    # the first call pays the per-n constants (host-built glibc p*log(p)
    # triangle, memo tables, kernel attributes), cached on the context for
    # every later call: reported as setup, outside the steps
    torch.cuda.synchronize()
    first_call_ms = None
    t_setup = time.perf_counter()
    for i in range(args.warmup):
        flush.zero_()
        step()
        if i == 0:
            torch.cuda.synchronize()
            first_call_ms = (time.perf_counter() - t_setup) * 1e3
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
    same = bool(np.array_equal(hout["mic"].view(np.int64),
                               outs["mic"][:count].cpu().numpy().view(np.int64)))

    if rank == 0:
        peaks = measured_peaks(local)
        dadd, lds, lds2 = peaks["fp64_per_s"], peaks["lsu_per_s"], peaks["lsu2_per_s"]
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
        ncu_pipe = None
        try:
            pp = json.load(open(os.path.join(ROOT, "profiles", "ncu_pipes.json")))["c1"]
            ncu_pipe = {"limiting_pipe": pp.get("limiting_pipe"), "pct_of_peak": pp.get("limiting_pipe_pct"),
                        "pipes_pct_of_peak": pp["pipes_pct_of_peak"], "capture": pp.get("capture"),
                        "source": "profiles/ncu_pipes.json (ncu --set full, committed capture; not this run)"}
        except Exception:
            pass
        roof = {"bound": "lsu", "ncu_limiting_pipe": ncu_pipe, "achieved": achieved, "peak": lds / 1e9 if lds else None,
                "unit": "Ggather/s", "frac": achieved / (lds / 1e9) if lds else None,
                "traffic": traffic,
                "traffic_source": "profiles/ncu_traffic.json (dram read+write bytes per launch, ncu)",
                "kernel": "k_memo_pairs (the pair-scoring launch of a step)",
                "per_launch_work": {k: int(v) for k, v in work.items()},
                "work_unit": "shared-memory table gathers the memo-tier algorithm needs "
                             "(one 2 B dense candidate rank per F(t,2) candidate, 2 x 8 B per "
                             "level-3 span term, 2 B rank per standard 3-row candidate, 7 x 8 B "
                             "per other 3-row candidate), counted by the kernel; DESIGN.md "
                             "'Roofline'",
                "gathers_8b": int(g8), "gathers_rank": int(g2),
                "peak_source": "measured live: probes.cu k_lds (random 8 B gathers, 561-entry "
                               "table) and k_lds2 (random 2 B gathers, 16K-entry table), 8 "
                               "streams/thread, all SMs; peak = time-weighted mix of the two",
                "kernel_ms": statistics.mean(kern_ms),
                # SURVEY 8(d)'s own T_roof for the same launch (rank 0's slice)
                "survey_8d": roofline_8d(work, kern_s, 16 * count + 96 * p, peaks),
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
            "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded c1 generator, numpy PCG64 seed 43)",
            "config": config_dict(w, p, world, total, args.scaling),
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(w.X.nbytes) * world,
                    "d2h_bytes_per_step": int(total * 8 * 2),
                    "matches_value_leg": same},
            "gpu_launches": int(launches) * args.steps,
            "clocks": clk.summary(),
            "roofline": roof,
            "setup": {"first_call_ms": first_call_ms,
                      "note": "the first call on a context builds the per-n tables (host glibc "
                              "p*log(p) triangle, memo candidate tables) and caches them; later "
                              "calls (every timed step) reuse them"},
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_reference(w, p, args.cpu_seconds, os.cpu_count() or 1)
        if world == 1 and not args.no_secondary:
            line["secondary"] = secondary_block(eng, local, peaks, args)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# Secondary configs: the heavy-DP general tier, observed
# by the driver in the default line.
SECONDARY = (  # (config, pair window, CPU-reference sample pairs)
    (0, 256, 256),
    (2, 20000, 4000),
    (3, 4000, 320),
    (4, 148, 0),  # one pair per SM; CPU rate and parity from the full-size fixture
)


def _ref_stats_parallel(R, X, Y, xi, yi, alpha, c, threads):
    """The reference's compute_statistics per pair (statistics.cpp:53-63) on
    a host thread pool -- run_analysis's own parallelism (analysis.cpp:
    148-190); ctypes releases the GIL inside each call."""
    from concurrent.futures import ThreadPoolExecutor
    out = np.zeros((len(xi), 6))

    def one(i):
        out[i] = R.statistics(X[xi[i]], Y[yi[i]], alpha, c)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, range(len(xi))))
    return out


def secondary_block(eng, device, peaks, args):
    import torch
    from paper_1208_4271_b200 import Parameters, datagen, cell_shapes, grid_bound
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    try:
        R = O.Reference()
    except FileNotFoundError:
        R = None
    cores = os.cpu_count() or 1
    dev = torch.device("cuda", device)
    stream = torch.cuda.current_stream(dev)
    res = []
    l2_rate, cand_rate = probe_general(device, 8.0 * 1341 * 1342 / 2)
    for cfg, window, cpu_pairs in SECONDARY:
        t_start = time.perf_counter()
        w = datagen.make(cfg)
        params = Parameters(w.alpha, w.c, w.est)
        if w.call == "pairwise":
            V = w.X
            total = V.shape[0] * (V.shape[0] - 1) // 2
            count = min(window, total)
            xi = yi = None
        elif w.call == "cross":
            V = np.ascontiguousarray(np.concatenate([w.X, w.Y]))
            count = min(window, w.X.shape[0] * w.Y.shape[0])
            xi = np.arange(count, dtype=np.int32) // w.Y.shape[0]
            yi = (w.X.shape[0] + np.arange(count) % w.Y.shape[0]).astype(np.int32)
        else:
            V = w.X
            xi, yi = w.xi.astype(np.int32), w.yi.astype(np.int32)
            count = xi.size
        dV = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
        douts = {k: torch.empty(count, dtype=torch.float64, device=dev)
                 for k in ("mic", "mas", "mev", "mcn", "tic")}
        dptr = {k: t.data_ptr() for k, t in douts.items()}
        kind = "pairwise" if xi is None else "pairs"
        dxi = torch.from_numpy(xi).to(dev) if xi is not None else None
        dyi = torch.from_numpy(yi).to(dev) if yi is not None else None

        def dcall(counters=False, kb=0, ke=0):
            return eng.device_call(kind, params, dptr, vars_ptr=dV.data_ptr(), p=V.shape[0],
                                   n=V.shape[1], xi_ptr=dxi.data_ptr() if dxi is not None else 0,
                                   yi_ptr=dyi.data_ptr() if dyi is not None else 0,
                                   npairs=count, first=0, count=count if kind == "pairwise" else 0,
                                   stream=stream.cuda_stream, counters=counters,
                                   ev_begin=kb, ev_end=ke)

        def hcall():
            if kind == "pairwise":
                return eng.pairwise(V, params, first=0, count=count, stats=("mic", "tic"))
            return eng.pairs(V, xi, yi, params, stats=("mic", "tic"))

        reps = 1 if cfg == 4 else 3
        dcall()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(reps)]
        for a, b in ev:
            a.record(stream)
            dcall()
            b.record(stream)
        torch.cuda.synchronize()
        dev_s = statistics.median([a.elapsed_time(b) for a, b in ev]) / 1e3
        hcall()
        ht = []
        for _ in range(reps):
            t0 = time.perf_counter()
            hcall()
            ht.append(time.perf_counter() - t0)
        e2e_s = statistics.median(ht)
        work = dcall(counters=True)
        r8 = roofline_8d(work, dev_s, 40 * count, peaks)
        entry = {"config": cfg, "call": w.call, "pairs": count, "n": w.n, "alpha": w.alpha,
                 "c": w.c, "est": w.est, "device_pairs_per_s": count / dev_s, "device_s": dev_s,
                 "e2e_pairs_per_s": count / e2e_s, "e2e_s": e2e_s, "launches": eng.last_launches,
                 "survey_8d": r8,
                 "fp64_ops_frac": work["fp64_ops"] / peaks["fp64_per_s"] / dev_s,
                 "work": {k: int(v) for k, v in work.items()}}
        # extended bound: exact DP candidates at the measured candidate rate
        # (DMUL + DADD + DSETP each) and the span terms' p*log(p) lookups at the
        # measured random L2 gather rate
        if l2_rate and cand_rate:
            C = r8["C"]
            terms = {"dp_candidates": C / cand_rate,
                     "span_lookups_l2": int(work["span_lookups"]) / l2_rate}
            b = max(terms, key=terms.get)
            entry["extended_roofline"] = {
                "t_roof_s": terms[b], "bound": b, "terms_s": terms, "frac": terms[b] / dev_s,
                "peaks": {"candidates_per_s (probes.cu k_dcand)": cand_rate,
                          "l2_gathers_per_s (probes.cu k_ldg_rand, 7.2 MB table)": l2_rate},
                "note": "C = every exact DP candidate (levels 2 .. l_max) at the measured "
                        "candidate rate; span_lookups = the span terms' p*log(p) lookups (rows "
                        "m = c_t - c_s scattered over the table) at the measured random L2 "
                        "gather rate (= one divergent lane per clock per SM through the L1/TEX "
                        "pipe, the pipe ncu shows busiest: ncu_top_kernel)"}
        # the config's top kernel under ncu (a committed capture, not this run):
        # which pipe is busiest and how busy -- the limiting-pipe fraction
        try:
            pp = json.load(open(os.path.join(ROOT, "profiles", "ncu_pipes.json"))).get(f"c{cfg}")
        except (OSError, ValueError):
            pp = None
        if pp:
            entry["ncu_top_kernel"] = {
                "kernel": pp["kernel"], "limiting_pipe": pp.get("limiting_pipe"),
                "limiting_pipe_pct": pp.get("limiting_pipe_pct"),
                "pipes_pct_of_peak": pp["pipes_pct_of_peak"], "capture": pp.get("capture"),
                "source": "profiles/ncu_pipes.json (ncu --set full --clock-control none, "
                          "tools/refresh_profiles.sh + tools/ncu_pipes.py); not measured in this run"}
        got = {k: t.cpu().numpy() for k, t in douts.items()}
        if cfg == 4:
            # the 32 pairs of the full-size reference fixture, scored separately
            g = np.load(os.path.join(ROOT, "tests", "golden", "ref_c4_full.npz"))
            fx = eng.pairs(V, g["xi"].astype(np.int32), (w.X.shape[0] + g["yi"]).astype(np.int32),
                           params, stats=("mic", "mas", "mev", "mcn"))
            n_s = int(g["xi"].size)
            ok = all(np.array_equal(fx[k].view(np.int64), g["stats"][:, c].view(np.int64))
                     for c, k in enumerate(("mic", "mas", "mev", "mcn")))
            secs = g["cpu_seconds"][:n_s]
            entry["cpu_reference"] = {
                "value": n_s / float(secs.sum()), "unit": "pairs/s", "cores": 1,
                "kind": "reference", "cpu_model": "build container (fixture generation)",
                "sample": f"the {n_s} fixture pairs (tests/golden/ref_c4_full.npz), reference "
                          f"compute_score, one thread per pair, {secs.sum():.0f} s CPU total; "
                          "not re-run here (minutes per pair)"}
            entry["bit_exact_on_sample"] = bool(ok)
        elif R is not None and cpu_pairs:
            n_s = min(cpu_pairs, count)
            if kind == "pairwise":
                orc = O.Oracle()
                idx = np.array([orc.pair_at(V.shape[0], t) for t in range(n_s)], dtype=np.int32)
                sxi, syi = idx[:, 0], idx[:, 1]
            else:
                sxi, syi = xi[:n_s], yi[:n_s]
            t0 = time.perf_counter()
            ref = _ref_stats_parallel(R, V, V, sxi, syi, w.alpha, w.c, cores)
            cdt = time.perf_counter() - t0
            ok = all(np.array_equal(got[k][:n_s].view(np.int64), ref[:, c].view(np.int64))
                     for c, k in enumerate(("mic", "mas", "mev", "mcn")))
            entry["cpu_reference"] = {"value": n_s / cdt, "unit": "pairs/s", "cores": cores,
                                      "kind": "reference", "cpu_model": cpu_model(),
                                      "sample": f"the first {n_s} pairs of the window, the "
                                                f"reference's compute_statistics on {cores} "
                                                f"threads, {cdt:.1f} s"}
            entry["bit_exact_on_sample"] = bool(ok)
        entry["wall_s"] = time.perf_counter() - t_start
        log(f"secondary c{cfg}: {entry['device_pairs_per_s']:.4g} pairs/s, 8d frac "
            f"{r8['frac']:.3f}, {entry['wall_s']:.1f} s")
        res.append(entry)
    return res


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
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="N > 1: strong = the unchanged c1 sharded over N GPUs; weak = p grows "
                         "to round(4381 sqrt(N))")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the secondary-config block of the default line")
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
