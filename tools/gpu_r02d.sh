#!/bin/bash
# Round 2: fused MRG32k3a consumer (tests, A/B against generate + read-back), bin A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "mrg" > gpurun_out/gputests_d.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_d.log
for rep in 1 2; do
  for v in default mrgold mrgw8; do
    if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
    for wl in "mrg26 --consume" "mrg26 --consume --no-write"; do
      PRNGD_LIB=$L timeout 300 python bench.py --workload $wl --steps 20 --sustained-s 0 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', '$wl', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
  for v in default bin0; do
    if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
    PRNGD_LIB=$L timeout 300 python bench.py --workload cfg5 --steps 50 --sustained-s 0 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', 'cfg5', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done > gpurun_out/mrg_ab.txt 2>&1
cat gpurun_out/mrg_ab.txt
bash tools/prof_one.sh r02d_mrg26_consume consume_mrg_kernel --workload mrg26 --consume
echo done
