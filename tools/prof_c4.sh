#!/bin/bash
# ncu full-set captures (with source counters) of the general tier's DP kernel
# on c4 (first k_dp launch = the y = 2.. group, ring variant) and c3: gpurun_out/p4/
out=${1:-gpurun_out/p4}; mkdir -p $out
timeout 300 python tools/gen_timing.py 4 ${2:-16} 1 > $out/c4_plain.log 2>&1 || exit 1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:^k_dp$ -c 1 \
  -o $out/c4_dp python tools/gen_timing.py 4 ${2:-16} 1 > $out/c4_dp.log 2>&1
ncu -i $out/c4_dp.ncu-rep --page details --csv > $out/c4_k_dp_details.csv 2>/dev/null
ncu -i $out/c4_dp.ncu-rep --page raw --csv > $out/c4_k_dp_raw.csv 2>/dev/null
ncu -i $out/c4_dp.ncu-rep --page source --csv > $out/c4_k_dp_source.csv 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:^k_dp$ -c 1 \
  -o $out/c3_dp python tools/gen_timing.py 3 500 1 > $out/c3_dp.log 2>&1
ncu -i $out/c3_dp.ncu-rep --page raw --csv > $out/c3_k_dp_raw.csv 2>/dev/null
ncu -i $out/c3_dp.ncu-rep --page source --csv > $out/c3_k_dp_source.csv 2>/dev/null
rm -f $out/*.ncu-rep.tmp
ls -la $out
