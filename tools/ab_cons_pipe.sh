#!/bin/bash
# A/B: software-pipelined row-segment consumer (PRNGD_CONS_PIPE=1, variants/lib_pipe.so) vs the
# in-tree library; then the GPU consumer parity tests on the variant.
mkdir -p gpurun_out; out=gpurun_out/s3e_cons_pipe_ab.txt; : > $out
one() {
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
  for v in default pipe2; do one $v cfg5 20; done
  for v in default pipe2; do one $v cfg4 20 --consume; done
  for v in default pipe2; do one $v cfg3 20 --consume; done
done
PRNGD_LIB=variants/lib_pipe2.so timeout 900 python -m pytest tests -q -m gpu -x -k "consum or fullsize or statistic or pairs" > gpurun_out/s3e_pipe_tests.log 2>&1
echo "variant tests rc=$?" | tee -a $out; tail -2 gpurun_out/s3e_pipe_tests.log | tee -a $out
echo done
