#!/bin/bash
# A/B: jump kernel byte-permute composition for w = 8 / 16 (PRNGD_JUMP_NARROW=1, default) vs the
# generic MODE 1 composition (variants/lib_narrow0.so), cfg2, alternating; comppos = the narrow
# modes with the position-indexed compaction stores (before the byte-address walk).
for rep in 1 2 3; do for v in default comppos narrow0; do
  if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
  PRNGD_LIB=$L timeout 300 python bench.py --workload cfg2 --steps 300 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v cfg2', round(d['value'],1), d['per_step']['step_ms_median'])"
done; done
