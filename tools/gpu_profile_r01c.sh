#!/bin/bash
# Round-1 final captures (run under gpurun): the launch list of the DEFAULT bench command, and
# ncu --set full of the kernels changed since r01b (exported to CSV on the box).
mkdir -p gpurun_out
python bench.py > gpurun_out/r01c_default_plain.log 2>&1 || { echo "default bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r01c_default_launches.csv python bench.py > gpurun_out/r01c_default_ncu.log 2>&1
bash tools/prof_one.sh r01c_cfg5_consume consume_kernel --workload cfg5
bash tools/prof_one.sh r01c_mrg26 gen_mrg --workload mrg26
bash tools/prof_one.sh r01c_cfg4_row gen_kernel --workload cfg4
bash tools/prof_one.sh r01c_cfg3_row gen_kernel
du -sh gpurun_out
echo profiled
