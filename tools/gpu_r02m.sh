#!/bin/bash
timeout 600 python -m pytest tests -q -m gpu -x -k "jump" > gpurun_out/gputests_m.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gputests_m.log
for rep in 1 2; do for v in default jp33m4 jp33m5; do
  if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
  PRNGD_LIB=$L timeout 300 python bench.py --workload cfg2 --steps 300 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v cfg2', round(d['value'],1), d['per_step']['step_ms_median'])"
done; done
