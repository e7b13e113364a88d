#!/bin/bash
# A/B: MRG32k3a ring reads as 16-byte loads from XOR-swizzled rings + hi/lo composition + fused
# ring-address LOP3 (default) vs without the swizzle (mrgswz0) vs the code before all three
# (mrgbase); mrg26 write and fused write + statistics, alternating.
for rep in 1 2 3; do for v in default mrgswz0 mrgbase; do
  if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
  for args in "" "--consume"; do
  PRNGD_LIB=$L timeout 300 python bench.py --workload mrg26 --steps 30 --sustained-s 0 --no-cpu-baseline --e2e-steps 0 $args 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v mrg26 $args', round(d['value'],1), round(d['roofline']['kernel_ms'],4), d['clocks']['sm_mhz'])"
  done
done; done
