#!/bin/bash
# per-kernel durations of one general-tier call (under gpurun): tools/launch_times.sh OUT CFG PAIRS [ENV=VAL ...]
out=$1; cfg=$2; pairs=$3; shift 3
mkdir -p $(dirname $out)
env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $out \
  python tools/gen_timing.py $cfg $pairs 1 > /dev/null 2>&1
