#!/bin/bash
# A/B of an environment switch (under gpurun): tools/ab_env.sh OUTDIR VAR "cfg:pairs:reps ..." value1 value2 ...
out=$1; var=$2; cfgs=$3; shift 3; mkdir -p $out
for v in "$@"; do
  for c in $cfgs; do
    IFS=: read cfg pairs reps <<< "$c"
    env $var=$v timeout 600 python tools/gen_timing.py $cfg $pairs $reps > $out/c${cfg}_$var$v.json 2>> $out/err.log
  done
done
