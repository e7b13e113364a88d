#!/bin/bash
# ncu evidence for every kernel family (run under gpurun; one ncu tool per call).
set -e
run() { tag=$1; shift; python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 "$@" > gpurun_out/${tag}_plain.log 2>&1; }
run cfg3 ; run cfg1 --workload cfg1 ; run cfg5 --workload cfg5 ; run mrg --workload mrg26
NCU="ncu --set full --clock-control none --import-source on -c 1"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0"
ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/r01_final_cfg3_launches.csv $B > /dev/null 2>&1
$NCU -k regex:gen_jump -s 2 -o gpurun_out/r01_cfg1_jump -f $B --workload cfg1 > /dev/null 2>&1
$NCU -k regex:consume_kernel -s 2 -o gpurun_out/r01_cfg5_consume_write -f $B --workload cfg5 > /dev/null 2>&1
$NCU -k regex:gen_mrg -s 2 -o gpurun_out/r01_mrg26 -f $B --workload mrg26 > /dev/null 2>&1
echo profiled
