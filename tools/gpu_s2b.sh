#!/bin/bash
# Narrow jump kernel: parity (jump tests) and cfg2 A/B against the previous narrow path.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "jump or narrow or cfg2 or pairs" > gpurun_out/s2b_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s2b_tests.log
for i in 1 2; do
STEPS=300 TAG=new bash tools/quick_ab.sh cfg2:auto
PRNGD_LIB=$PWD/variants/lib_jn0.so STEPS=300 TAG=old bash tools/quick_ab.sh cfg2:auto
done
ncu --set full --clock-control none -k regex:gen_jump -c 1 -o gpurun_out/s2b_cfg2_jumpn python bench.py --workload cfg2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --sustained-s 0 > /dev/null 2>&1; echo "ncu rc=$?"
