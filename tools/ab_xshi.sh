#!/bin/bash
# A/B: xorshift128 right shifts on the FMA pipe (IMAD.HI) vs the ALU pipe (SHF), PRNGD_XS_HI
# variants (variants/lib_xshi{1,2,3}.so) against the in-tree library, alternating.
mkdir -p gpurun_out; out=gpurun_out/s3b_xshi_ab.txt; : > $out
one() {  # variant workload steps [extra]
  v=$1; wl=$2; st=$3; shift 3
  if [ "$v" = default ]; then L=""; else L=variants/lib_$v.so; fi
  PRNGD_LIB=$L timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --sustained-s 0 \
      --workload $wl --steps $st "$@" 2>/dev/null | tail -1 | python -c "
import sys,json
try:
    d=json.loads(sys.stdin.read()); p=d.get('per_step') or {}
    print('$wl $* $v', round(d['value'],1), 'best', round(p.get('value_at_best',0),1), 'kern_ms', round(d['roofline'].get('kernel_ms',0),5), d['clocks']['sm_mhz'], d['clocks']['reasons'])
except Exception as e: print('$wl $v FAILED', e)" | tee -a $out
}
for rep in 1 2 3; do
  for v in default xshi1 xshi2 xshi3; do one $v cfg5 20; done
  for v in default xshi1 xshi2 xshi3; do one $v cfg2 100; done
  for v in default xshi1 xshi2 xshi3; do one $v cfg1 100; done
done
for rep in 1 2; do
  for v in default xshi3; do one $v cfg3 20; done
  for v in default xshi3; do one $v cfg4 20 --consume; done
done
echo done
