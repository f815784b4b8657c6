#!/bin/bash
# General-tier ncu captures (full set + source) of the top kernels on c2 / c3.
# usage (under gpurun): tools/prof_general.sh OUTDIR
out=${1:-gpurun_out/pg}; mkdir -p $out
for a in "0 256" "2 20000" "3 2000"; do
  set -- $a
  timeout 300 python tools/gen_timing.py $1 $2 5 > $out/c$1_timing.json 2> $out/c$1_timing.err
done
cap() {  # cap NAME CONFIG PAIRS KERNEL_REGEX
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$4" -c 1 \
    -o $out/$1 python tools/gen_timing.py $2 $3 1 > $out/$1.log 2>&1
}
cap c2_pf2 2 4000 k_part_f2
cap c2_dpw 2 4000 k_dp_warp
cap c3_dp 3 500 'k_dp<'
cap c3_pf2 3 500 k_part_f2
