#!/bin/bash
# Final round-1 captures of the kernels changed after r01c (consume task order, MRG32k3a,
# jump kernel, SEG) plus the benchmark sweep.
mkdir -p gpurun_out
bash tools/prof_one.sh r01d_cfg5_consume consume_kernel --workload cfg5
bash tools/prof_one.sh r01d_mrg26 gen_mrg --workload mrg26
bash tools/prof_one.sh r01d_cfg2_jump gen_jump --workload cfg2
bash tools/prof_one.sh r01d_cfg1_seg gen_seg --workload cfg1
bash tools/bench_all.sh
echo profiled
