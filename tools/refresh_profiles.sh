#!/bin/bash
# Round profile refresh on a GPU box: bench lines (ours incl. the secondary
# block, reference arm), the launch list of the bench command, an ncu --set
# full capture of the c1 pair kernel, and the general-tier launch lists.
# Writes under gpurun_out/prof/.  Every ncu command runs after the same
# command has exited 0 without ncu (profiling recipe).
set -x
P=gpurun_out/prof; mkdir -p $P
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $P/gpu.txt
lscpu > $P/lscpu.txt
timeout 900 python bench.py > $P/bench.json 2> $P/bench.err
timeout 900 python bench.py --impl reference > $P/bench_ref.json 2> $P/bench_ref.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary"
timeout 400 $B > $P/plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $P/launches.csv $B > $P/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  -k regex:^k_memo_pairs$ -s 4 -c 1 -o $P/memo_full $B > $P/ncu_full.log 2>&1
ncu -i $P/memo_full.ncu-rep --page raw --csv > $P/k_memo_pairs_raw.csv 2>/dev/null
ncu -i $P/memo_full.ncu-rep --page details --csv > $P/k_memo_pairs_details.csv 2>/dev/null
for a in "0 256" "2 20000" "3 2000"; do
  set -- $a
  tools/gen_profile.sh $P $1 $2
done
# general-tier top kernels: ncu full set (after the timing runs above exited 0)
timeout 600 ncu --set full --import-source on --clock-control none -k k_dp -c 1 \
  -o $P/c3_k_dp python tools/gen_timing.py 3 500 1 > $P/ncu_c3_dp.log 2>&1
ncu -i $P/c3_k_dp.ncu-rep --page details --csv > $P/c3_k_dp_details.csv 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k k_part_warp -c 1 \
  -o $P/c2_k_part_warp python tools/gen_timing.py 2 4000 1 > $P/ncu_c2_pw.log 2>&1
ncu -i $P/c2_k_part_warp.ncu-rep --page details --csv > $P/c2_k_part_warp_details.csv 2>/dev/null
