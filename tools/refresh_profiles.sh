#!/bin/bash
# Round profile refresh on a GPU box: pytest -m gpu, the launch list of the
# bench command, an ncu --set full capture of the c1 pair kernel, the
# general-tier launch lists and top-kernel captures with their limiting-pipe
# summary (ncu_pipes.json), then the bench lines (ours incl. the secondary
# block, reference arm).
# Writes under gpurun_out/prof/.  Every ncu command runs after the same
# command has exited 0 without ncu (profiling recipe).
set -x
P=gpurun_out/prof; mkdir -p $P
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $P/gpu.txt
lscpu > $P/lscpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $P/pytest_gpu_full.log 2>&1
tail -3 $P/pytest_gpu_full.log > $P/pytest_gpu.log
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
cap() {  # cap TAG KERNEL_REGEX CONFIG PAIRS
  timeout 1500 ncu --set full --import-source on --clock-control none --kernel-name-base function \
    -k regex:^$2\$ -c 1 -o $P/$1 python tools/gen_timing.py $3 $4 1 > $P/ncu_$1.log 2>&1
  ncu -i $P/$1.ncu-rep --page details --csv > $P/$1_details.csv 2>/dev/null
  ncu -i $P/$1.ncu-rep --page raw --csv > $P/$1_raw.csv 2>/dev/null
  ncu -i $P/$1.ncu-rep --page source --csv > $P/$1_source.csv 2>/dev/null
}
cap c3_k_dp k_dp 3 500
cap c3_k_part_f2 k_part_f2 3 500
cap c2_k_part_warp k_part_warp 2 4000
cap c0_k_dp k_dp 0 256
cap c4_k_dp k_dp 4 148
# which pipe limits each config's top kernel (bench.py attaches these to the secondary block)
python tools/ncu_pipes.py $P/ncu_pipes.json \
  "c1=$P/k_memo_pairs_raw.csv@k_memo_pairs, launch 5 of bench.py --steps 2 --warmup 3 (all 9,594,390 c1 pairs)" \
  "c0=$P/c0_k_dp_raw.csv:$P/c0_k_dp_source.csv@k_dp, first launch of a c0 call (256 pairs)" \
  "c2=$P/c2_k_part_warp_raw.csv:$P/c2_k_part_warp_source.csv@k_part_warp, first launch of a c2 call (4,000 pairs)" \
  "c3=$P/c3_k_dp_raw.csv:$P/c3_k_dp_source.csv@k_dp, first launch of a c3 call (500 pairs)" \
  "c3_k_part_f2=$P/c3_k_part_f2_raw.csv:$P/c3_k_part_f2_source.csv@k_part_f2, first launch of a c3 call (500 pairs)" \
  "c4=$P/c4_k_dp_raw.csv:$P/c4_k_dp_source.csv@k_dp (ring variant), first launch of a c4 call (148 pairs)" > $P/ncu_pipes.log 2>&1
rm -f $P/*_source.csv $P/*.ncu-rep
# the bench lines last: the secondary block cites the pipe summary just made
sed -e "s#$P/#profiles/r02/#g" $P/ncu_pipes.json > profiles/ncu_pipes.json
timeout 900 python bench.py > $P/bench.json 2> $P/bench.err
timeout 900 python bench.py --impl reference > $P/bench_ref.json 2> $P/bench_ref.err
cp profiles/ncu_pipes.json $P/ncu_pipes_final.json
