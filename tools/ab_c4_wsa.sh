#!/bin/bash
out=gpurun_out/wsa; mkdir -p $out
for cv in 58 72 86; do
  MINE_B200_LIB=$PWD/ab/wsa.so MINE_B200_DP_CARVEOUT=$cv timeout 600 python tools/gen_timing.py 4 148 2 > $out/c4_wsa$cv.json 2>>$out/err
done
MINE_B200_LIB=$PWD/ab/cur.so timeout 600 python tools/gen_timing.py 4 148 2 > $out/c4_cur.json 2>>$out/err
MINE_B200_LIB=$PWD/ab/wsa.so timeout 600 python tools/gen_timing.py 3 2000 3 > $out/c3_wsa.json 2>>$out/err
MINE_B200_LIB=$PWD/ab/cur.so timeout 600 python tools/gen_timing.py 3 2000 3 > $out/c3_cur.json 2>>$out/err
