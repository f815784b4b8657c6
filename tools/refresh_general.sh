#!/bin/bash
# General-tier profile refresh: secondary configs (with CPU port samples) and
# the c3 launch list with FP64-pipe activity.  Writes under gpurun_out/gen/.
P=gpurun_out/gen; mkdir -p $P
for a in "0 256 256" "2 20000 2000" "3 4000 160"; do
  set -- $a
  timeout 600 python bench.py --config $1 --pairs $2 --cpu-pairs $3 --steps 3 >> $P/secondary.jsonl 2>> $P/secondary.err
done
timeout 600 python bench.py --config 4 --pairs 128 --steps 2 --no-cpu-baseline >> $P/secondary.jsonl 2>> $P/secondary.err
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic \
  --clock-control none --csv --log-file $P/c3_launches.csv \
  python bench.py --config 3 --pairs 2000 --steps 1 --warmup 3 --no-cpu-baseline > $P/c3_ncu.log 2>&1
