#!/bin/bash
# ncu evidence for the current kernels (run under gpurun; one GPU).  Each capture runs only
# after the same command exited 0 without ncu.
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0"
NCU="ncu --set full --clock-control none --import-source on -c 1"
mkdir -p gpurun_out
run() { tag=$1; shift; $B "$@" > gpurun_out/r01b_${tag}_plain.log 2>&1 || echo "plain run $tag failed"; }
run cfg3; run cfg5 --workload cfg5; run cfg4 --workload cfg4; run mrg --workload mrg26; run cfg1 --workload cfg1
# launch list of the default bench command (cold-cache, serialised per-launch times)
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/r01b_cfg3_launches.csv python bench.py --steps 20 --warmup 3 \
    --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/r01b_cfg5_launches.csv $B --workload cfg5 > /dev/null 2>&1
$NCU -k regex:gen_kernel -s 2 -o gpurun_out/r01b_cfg3_row -f $B > /dev/null 2>&1
$NCU -k regex:consume_kernel -s 2 -o gpurun_out/r01b_cfg5_consume -f $B --workload cfg5 > /dev/null 2>&1
$NCU -k regex:gen_kernel -s 2 -o gpurun_out/r01b_cfg4_row -f $B --workload cfg4 > /dev/null 2>&1
$NCU -k regex:gen_mrg -s 2 -o gpurun_out/r01b_mrg26 -f $B --workload mrg26 > /dev/null 2>&1
$NCU -k regex:gen_seg -s 2 -o gpurun_out/r01b_cfg1_seg -f $B --workload cfg1 > /dev/null 2>&1


# export on the box (the .ncu-rep files are too large to bring back), keep the CSVs
for f in gpurun_out/r01b_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${b}_details.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > ${b}_sass.csv 2>/dev/null
  rm -f $f
done
du -sh gpurun_out
echo profiled
