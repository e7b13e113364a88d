#!/bin/bash
# Profile the bench's dominant kernel on one B200 (run under gpurun).  Args: tag [bench args...]
tag=$1; shift
cmd="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 $*"
$cmd > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv \
    --log-file gpurun_out/${tag}_launches.csv $cmd > gpurun_out/${tag}_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gen_kernel|gen_seg_kernel|gen_segc_kernel|consume_kernel" -s 2 -c 1 \
    -o gpurun_out/${tag}_prof -f $cmd > gpurun_out/${tag}_ncu_full.log 2>&1
echo "profile rc=$?"
