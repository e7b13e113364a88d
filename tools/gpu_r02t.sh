#!/bin/bash
for rep in 1 2; do for v in default ps4 ps1; do
  if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
  for wl in "cfg5" "cfg3 --consume"; do
    PRNGD_LIB=$L timeout 300 python bench.py --workload $wl --steps 50 --sustained-s 0 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', '$wl', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done; done
