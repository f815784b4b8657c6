#!/bin/bash
# ncu full-set captures of k_dp on c3 and c0 (under gpurun): gpurun_out/pd/
out=${1:-gpurun_out/pd}; mkdir -p $out
timeout 600 ncu --set full --import-source on --clock-control none -k k_dp -c 1 \
  -o $out/c3_dp python tools/gen_timing.py 3 500 1 > $out/c3_dp.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k k_dp -c 1 \
  -o $out/c0_dp python tools/gen_timing.py 0 256 1 > $out/c0_dp.log 2>&1
