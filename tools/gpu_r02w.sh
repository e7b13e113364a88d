#!/bin/bash
timeout 900 python -m pytest tests -q -m gpu -x -k "consume or hist or fullsize or segments or pairs or random or peer" > gpurun_out/gputests_w.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gputests_w.log
for rep in 1 2; do for v in default h16; do
  if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
  for wl in "cfg5" "cfg3 --consume" "cfg4 --consume"; do
    PRNGD_LIB=$L timeout 300 python bench.py --workload $wl --steps 50 --sustained-s 0 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', '$wl', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done; done
bash tools/prof_one.sh r02w_cfg5_consume8 consume_seg8_kernel --workload cfg5
