#!/bin/bash
# General-tier timing + launch list for one config window (run under gpurun).
# usage: tools/gen_profile.sh OUTDIR CONFIG PAIRS
out=${1:-gpurun_out/gen}; cfg=${2:-3}; pairs=${3:-2000}
mkdir -p $out
timeout 600 python tools/gen_timing.py $cfg $pairs 5 > $out/c${cfg}_timing.json 2> $out/c${cfg}_timing.err &&
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file $out/c${cfg}_launches.csv \
  python tools/gen_timing.py $cfg $pairs 1 > $out/c${cfg}_ncu.log 2>&1
