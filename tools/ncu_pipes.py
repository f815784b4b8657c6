#!/usr/bin/env python3
"""Which pipe limits a kernel, from ncu captures already converted to CSV:

    python tools/ncu_pipes.py OUT.json "TAG=RAW.csv[:SOURCE.csv][@what was captured]" ...

RAW.csv is `ncu -i X.ncu-rep --page raw --csv`, SOURCE.csv the matching
`--page source --csv` (SASS view).  For every capture the summary keeps the
launch's duration, the busy fraction of each candidate pipe (L1/TEX data
pipe wavefronts, FP64, issue slots, L2, DRAM), the split of the L1 wavefronts
into shared-memory and global (LGDS) ones, the shared bank-conflict replays,
and -- with a source page -- the instructions that issue the most shared
wavefronts.  bench.py attaches the entry of a config's top kernel to its
`secondary` line (profiles/ncu_pipes.json)."""
import csv
import json
import sys


def raw_metrics(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"__units__": dict(zip(hdr, units))}
    for h, v in zip(hdr, vals):
        try:
            out[h] = float(v.replace(",", ""))
        except ValueError:
            out[h] = v
    return out


def first(m, *names):
    for n in names:
        if n in m and m[n] != "":
            return m[n]
    return None


def source_top(path, k=8):
    rd = csv.reader(open(path))
    next(rd)
    hdr = next(rd)
    ix = {h: i for i, h in enumerate(hdr)}
    rows = [r for r in rd if len(r) > ix["L1 Wavefronts Shared"]]

    def num(r, key):
        try:
            return float(r[ix[key]])
        except ValueError:
            return 0.0

    tot = sum(num(r, "L1 Wavefronts Shared") for r in rows) or 1.0
    by_op = {}
    for r in rows:
        op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
        if op.startswith("@"):
            op = r[ix["Source"]].split()[1]
        by_op[op] = by_op.get(op, 0.0) + num(r, "L1 Wavefronts Shared")
    top = sorted(rows, key=lambda r: -num(r, "L1 Wavefronts Shared"))[:k]
    return {
        "shared_wavefronts_by_opcode_pct": {o: round(100 * v / tot, 1)
                                            for o, v in sorted(by_op.items(), key=lambda kv: -kv[1])[:6]},
        "top_instructions": [{"sass": " ".join(r[ix["Source"]].split())[:60],
                              "shared_wavefronts_pct": round(100 * num(r, "L1 Wavefronts Shared") / tot, 1),
                              "ideal_pct": round(100 * num(r, "L1 Wavefronts Shared Ideal") / tot, 1)}
                             for r in top]}


def summarise(raw, src=None):
    m = raw_metrics(raw)
    wf = first(m, "l1tex__data_pipe_lsu_wavefronts.sum")
    wf_sh = first(m, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    wf_avg = first(m, "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg")
    wf_avg_sh = first(m, "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg")
    wf_avg_gl = first(m, "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg")
    cyc = first(m, "sm__cycles_active.avg")
    e = {
        "kernel": m.get("Kernel Name"),
        "duration_ms": (first(m, "gpu__time_duration.sum") or 0.0) *
        {"s": 1e3, "ms": 1.0, "us": 1e-3, "ns": 1e-6}.get(m["__units__"].get("gpu__time_duration.sum", "ns"), 1e-6),
        "registers": first(m, "launch__registers_per_thread"),
        "pipes_pct_of_peak": {
            "l1tex (SOL: busiest of the L1/TEX data and tag stages)": first(
                m, "l1tex__throughput.avg.pct_of_peak_sustained_active",
                "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
            "l1tex_data_pipe_wavefronts_busiest_sm": first(
                m, "l1tex__data_pipe_lsu_wavefronts.max.pct_of_peak_sustained_elapsed"),
            "fp64": first(m, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_slots": first(m, "sm__inst_issued.avg.pct_of_peak_sustained_active",
                                 "smsp__issue_active.avg.pct"),
            "l2": first(m, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "dram": first(m, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                          "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        },
        "l1_wavefronts_per_sm_avg": {"all": wf_avg, "shared": wf_avg_sh, "global": wf_avg_gl,
                                     "per_active_cycle": (wf_avg / cyc) if wf_avg and cyc else None},
        "shared_wavefronts": wf_sh if wf_sh is not None else wf,
        "shared_bank_conflict_replays": first(m, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "global_load_requests": first(m, "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
        "global_load_sectors": first(m, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
        "active_threads_per_warp": first(m, "smsp__thread_inst_executed_per_inst_executed.ratio"),
        "source": raw,
    }
    pipes = {k: v for k, v in e["pipes_pct_of_peak"].items() if isinstance(v, float)}
    if pipes:
        e["limiting_pipe"] = max(pipes, key=pipes.get)
        e["limiting_pipe_pct"] = pipes[e["limiting_pipe"]]
    if src:
        e["source_view"] = source_top(src)
    return e


def main():
    out = sys.argv[1]
    res = {}
    for a in sys.argv[2:]:
        tag, paths = a.split("=", 1)
        paths, _, capture = paths.partition("@")
        raw, _, src = paths.partition(":")
        res[tag] = summarise(raw, src or None)
        res[tag]["capture"] = capture or None
    json.dump(res, open(out, "w"), indent=1)
    for t, e in res.items():
        print(t, e.get("limiting_pipe"), e.get("limiting_pipe_pct"), f"{e['duration_ms']:.3f} ms")


if __name__ == "__main__":
    main()
