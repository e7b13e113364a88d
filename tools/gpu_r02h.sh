#!/bin/bash
# Row-segment fused consumer: parity, then A/B against ROW tiles (variant PRNGD_CONS_SEG=0).
timeout 900 python -m pytest tests -q -m gpu -x -k "consume or fullsize or segments or random or hist" > gpurun_out/gputests_h.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests_h.log
for rep in 1 2; do for v in default consrow; do
  if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
  for wl in "cfg5" "cfg4 --consume" "cfg3 --consume"; do
    PRNGD_LIB=$L timeout 300 python bench.py --workload $wl --steps 50 --sustained-s 0 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', '$wl', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done; done > gpurun_out/cons_seg_ab.txt 2>&1
cat gpurun_out/cons_seg_ab.txt
bash tools/prof_one.sh r02h_cfg5_consume_seg consume_kernel --workload cfg5
echo done
