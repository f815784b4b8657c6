#!/bin/bash
# A/B timing of engine builds on the secondary configs.
# usage: tools/ab.sh OUT ROUNDS LIB...
out=$1; rounds=$2; shift 2
for r in $(seq $rounds); do
  for lib in "$@"; do
    for a in ${AB_CONFIGS:-"0:256" "2:20000" "3:4000" "4:32"}; do
      c=${a%%:*}; p=${a##*:}
      MINE_B200_LIB=$lib timeout 300 python bench.py --config $c --pairs $p --steps 3 --no-cpu-baseline \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['config'], round(d['e2e_pairs_per_s'],1))" >> "$out"
    done
  done
done
