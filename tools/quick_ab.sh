#!/bin/bash
# Quick bench lines (value, kernel, clocks) for a list of "workload:store[:extra args]" cases.
for c in "$@"; do
  IFS=: read wl st extra <<< "$c"
  out=$(timeout 300 python bench.py --workload $wl --store $st --steps ${STEPS:-100} --no-cpu-baseline --e2e-steps 0 $extra 2>&1 | tail -1)
  echo "$out" | python -c "
import sys,json
s=sys.stdin.read()
try:
    d=json.loads(s); print('$c', '${TAG:-}', round(d['value'],1), d['roofline'].get('kernel'), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'), d['clocks']['reasons'])
except Exception: print('$c', '${TAG:-}', 'FAILED:', s[-300:])"
done
