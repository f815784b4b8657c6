#!/bin/bash
# A/B of engine builds (under gpurun): tools/ab_libs.sh OUTDIR "cfg:pairs:reps ..." lib1.so lib2.so ...
# (the default in-tree library is "default")
out=$1; shift; cfgs=$1; shift; mkdir -p $out
for lib in "$@"; do
  tag=$(basename $lib .so)
  for c in $cfgs; do
    IFS=: read cfg pairs reps <<< "$c"
    if [ "$lib" = default ]; then
      timeout 600 python tools/gen_timing.py $cfg $pairs $reps > $out/c${cfg}_$tag.json 2>> $out/err.log
    else
      MINE_B200_LIB=$PWD/$lib timeout 600 python tools/gen_timing.py $cfg $pairs $reps > $out/c${cfg}_$tag.json 2>> $out/err.log
    fi
  done
done
