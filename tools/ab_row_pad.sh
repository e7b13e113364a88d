#!/bin/bash
# A/B: ROW generator tile alignment 1024 B (12 one-warp CTAs per SM) vs 16 B (13 per SM).
for rep in 1 2 3; do for v in default rowpad16; do for wl in cfg3 cfg4; do
  if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
  PRNGD_LIB=$L timeout 300 python bench.py --workload $wl --steps 200 --no-cpu-baseline --e2e-steps 0 --sustained-s 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v $wl', round(d['value'],1), d['roofline'].get('kernel'), round(d['roofline']['frac'],3), d['clocks']['reasons'])"
done; done; done
