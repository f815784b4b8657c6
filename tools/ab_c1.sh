#!/bin/bash
# c1 headline A/B over environment settings: tools/ab_c1.sh OUT "ENV=.." "ENV=.." ...
out=$1; shift
for r in 1 2; do
  for e in "$@"; do
    env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['value']/1e9,4), round(d['roofline']['frac'],4), round(d['e2e']['value']/1e9,4), d['e2e']['matches_value_leg'])" >> "$out"
  done
done
