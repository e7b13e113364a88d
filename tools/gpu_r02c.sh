#!/bin/bash
# Round 2: fused consumer A/B (bin via RZ DADD, split power sums, 12 vs 16 warps) + ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "consume or fullsize or hist or random" > gpurun_out/gputests_c.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_c.log
for rep in 1 2; do for v in default ps2 w16 ps2w16; do
  if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
  for wl in "cfg5" "cfg4 --consume"; do
    PRNGD_LIB=$L timeout 300 python bench.py --workload $wl --steps 50 --sustained-s 0 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', '$wl', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done; done > gpurun_out/cons_ab.txt 2>&1
cat gpurun_out/cons_ab.txt
bash tools/prof_one.sh r02c_cfg5_consume consume_kernel --workload cfg5
echo done
