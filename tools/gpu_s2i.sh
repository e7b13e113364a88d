#!/bin/bash
# cfg5 fused consumer: bench value vs run length (power cap), clocks and per-step best/median.
for n in 5 20 50 200; do
  python bench.py --workload cfg5 --steps $n --warmup 3 --no-cpu-baseline --e2e-steps 0 --sustained-s 0 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
ps = d['per_step']
print('steps', $n, 'value', round(d['value'], 1), 'best-step', round(ps['value_at_best'], 1), 'median-step', round(ps['value_at_median'], 1), 'clocks', d['clocks']['sm_mhz'], d['clocks']['reasons'], d['clocks'].get('power_w_max'))"
  sleep 5
done
