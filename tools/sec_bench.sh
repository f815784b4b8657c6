#!/bin/bash
# Secondary-config timing sweep (general tier): one JSON line per config.
# usage: tools/sec_bench.sh OUT.jsonl [steps]
out=${1:-gpurun_out/sec.jsonl}; steps=${2:-3}
for a in "0 256" "2 20000" "3 4000" "4 64"; do
  set -- $a
  timeout 300 python bench.py --config $1 --pairs $2 --steps $steps --no-cpu-baseline >> "$out" 2>>"$out.err"
done
