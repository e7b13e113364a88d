#!/bin/bash
# A/B library variants on one B200: tools/ab_variants.sh "bench args" name1 name2 ...
# (name "default" = the in-tree library, else variants/lib_<name>.so)
args=$1; shift
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L=variants/lib_$v.so; fi
  PRNGD_LIB=$L timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 $args 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
