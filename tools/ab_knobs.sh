#!/bin/bash
out=gpurun_out/knob; mkdir -p $out
for c in "0:256:7" "3:2000:3"; do
  IFS=: read cfg pairs reps <<< "$c"
  timeout 600 python tools/gen_timing.py $cfg $pairs $reps > $out/c${cfg}_base.json 2>>$out/err
  MINE_B200_DP_INPLACE=1 timeout 600 python tools/gen_timing.py $cfg $pairs $reps > $out/c${cfg}_inplace.json 2>>$out/err
  for cv in 40 58 75 100; do
    MINE_B200_DP_CARVEOUT=$cv timeout 600 python tools/gen_timing.py $cfg $pairs $reps > $out/c${cfg}_cv$cv.json 2>>$out/err
  done
done
