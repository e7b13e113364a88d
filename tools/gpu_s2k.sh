#!/bin/bash
# Fused consumer warps per SM (PRNGD_CONS_SEG_WARPS 16 product / 18 / 20 variants): cfg5, short runs
# (10 steps, little power capping) and 50-step runs, value and best step.
run() {
  env $1 python bench.py --workload cfg5 --steps $2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --sustained-s 0 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); ps = d['per_step']
print('$3', 'steps', $2, 'value', round(d['value'], 1), 'best', round(ps['value_at_best'], 1), d['clocks']['reasons'])"
}
for i in 1 2; do
  for v in product cw18 cw20; do
    if [ $v = product ]; then L="X=1"; else L="PRNGD_LIB=$PWD/variants/lib_$v.so"; fi
    run "$L" 10 $v; sleep 3
  done
done
for v in product cw18 cw20; do
  if [ $v = product ]; then L="X=1"; else L="PRNGD_LIB=$PWD/variants/lib_$v.so"; fi
  run "$L" 50 $v; sleep 5
done
