#!/usr/bin/env python3
"""Summarise an ncu --csv launch list (tools/gen_profile.sh): per kernel
name, launches, total device ms and mean FP64-pipe / issue activity, for the
LAST timed call (between the last two k_sort_vars launches) or all."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Grid Size", "Block Size")}
    L = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        d = L.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]].split("(")[0], "grid": r[ix["Grid Size"]],
                                       "block": r[ix["Block Size"]]})
        try:
            d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:
            pass
    return list(L.values())


def main():
    ks = load(sys.argv[1])
    mode = sys.argv[2] if len(sys.argv) > 2 else "last"
    if mode == "last":
        idx = [i for i, d in enumerate(ks) if "sort_vars" in d["name"]]
        ks = ks[idx[-1]:] if idx else ks
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for d in ks:
        t = d.get("gpu__time_duration.sum", 0.0)
        a = agg[d["name"]]
        a[0] += 1
        a[1] += t
        a[2] += t * d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
        a[3] += t * d.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"total {tot / 1e3:.1f} us over {len(ks)} launches")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k[-60:]:60s} n={a[0]:4d} {a[1] / 1e3:10.1f} us {100 * a[1] / tot:5.1f}%  "
              f"fp64 {a[2] / max(a[1], 1):5.1f}%  issue {a[3] / max(a[1], 1):5.1f}%")


if __name__ == "__main__":
    main()
