#!/bin/bash
# A/B: MRG32k3a output tile row length (PRNGD_MRG_RC outputs per row flush: 16 default, 32, 64)
for rep in 1 2; do for v in default mrgrc32 mrgrc64; do
  if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
  PRNGD_LIB=$L timeout 300 python bench.py --workload mrg26 --steps 30 --sustained-s 0 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v mrg26', round(d['value'],1), round(d['roofline']['kernel_ms'],4), d['clocks']['sm_mhz'])"
done; done
