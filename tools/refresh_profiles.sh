#!/bin/bash
# Round profile refresh on a GPU box: bench lines, launch list, ncu capture of
# the pair kernel, secondary configs.  Writes under gpurun_out/prof/.
set -x
P=gpurun_out/prof; mkdir -p $P
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $P/gpu.txt
timeout 400 python bench.py > $P/bench.json 2> $P/bench.err
timeout 600 python bench.py --impl reference > $P/bench_ref.json 2> $P/bench_ref.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $P/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $P/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  -k regex:^k_memo_pairs$ -s 4 -c 1 -o $P/memo_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $P/ncu_full.log 2>&1
ncu -i $P/memo_full.ncu-rep --page raw --csv > $P/k_memo_pairs_raw.csv 2>/dev/null
ncu -i $P/memo_full.ncu-rep --page details --csv > $P/k_memo_pairs_details.csv 2>/dev/null
for a in "0 256 256" "2 20000 2000" "3 4000 160"; do
  set -- $a
  timeout 600 python bench.py --config $1 --pairs $2 --cpu-pairs $3 --steps 3 >> $P/secondary.jsonl 2>> $P/secondary.err
done
timeout 600 python bench.py --config 4 --pairs 128 --steps 2 --no-cpu-baseline >> $P/secondary.jsonl 2>> $P/secondary.err
