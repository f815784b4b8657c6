#!/bin/bash
# Row-map dedup A/B + parity (under gpurun): writes gpurun_out/dd/
out=${1:-gpurun_out/dd}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "dedup or c2 or c0 or general or golden or randomized or debug" > $out/pytest.log 2>&1
for cfg in "0 256" "2 20000" "3 2000"; do
  set -- $cfg
  for f in 1 0; do
    MINE_B200_ROW_DEDUP=$f timeout 300 python tools/gen_timing.py $1 $2 5 > $out/c$1_dd$f.json 2>> $out/err.log
  done
done
