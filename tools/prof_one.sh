#!/bin/bash
# One ncu --set full capture of a kernel (regex) in a bench command, exported to CSV on the box.
# usage: tools/prof_one.sh tag kernel_regex [bench args...]
tag=$1; re=$2; shift 2
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 $*"
$B > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$re -s 2 -c 1 -o gpurun_out/${tag} -f $B > /dev/null 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
rm -f gpurun_out/${tag}.ncu-rep
echo "profiled $tag"
