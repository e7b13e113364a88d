#!/bin/bash
PRNGD_LIB=variants/lib_inc1.so timeout 900 python -m pytest tests -q -m gpu -x -k "consume or hist or segments" > gpurun_out/gputests_x.log 2>&1; echo "tests(inc1) rc=$?"; tail -1 gpurun_out/gputests_x.log
for rep in 1 2 3; do for v in default inc1; do
  if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
  for wl in "cfg5" "cfg3 --consume"; do
    PRNGD_LIB=$L timeout 300 python bench.py --workload $wl --steps 50 --sustained-s 0 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', '$wl', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done; done
