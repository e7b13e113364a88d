#!/bin/bash
B="python bench.py --workload cfg1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --sustained-s 0 --warm-l2"
$B > /dev/null 2>&1
ncu --set full --cache-control none --clock-control none -k regex:gen_seg_kernel -s 4 -c 1 -o gpurun_out/r02y_cfg1_warm -f $B > /dev/null 2>&1
ncu -i gpurun_out/r02y_cfg1_warm.ncu-rep --page raw --csv > gpurun_out/r02y_cfg1_warm_raw.csv 2>/dev/null
ncu -i gpurun_out/r02y_cfg1_warm.ncu-rep --page details --csv > gpurun_out/r02y_cfg1_warm_details.csv 2>/dev/null
rm -f gpurun_out/r02y_cfg1_warm.ncu-rep
echo done
