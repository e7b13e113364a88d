#!/bin/bash
# MRG32k3a floor-mode reduction: parity (every MRG test) and mrg26 A/B against the nearest-mode build.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "mrg or MRG" > gpurun_out/s2c_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s2c_tests.log
for i in 1 2; do
STEPS=50 TAG=floor bash tools/quick_ab.sh mrg26:auto mrg26:auto:--consume mrg26:auto:--consume\ --no-write
PRNGD_LIB=$PWD/variants/lib_mf0.so STEPS=50 TAG=nearest bash tools/quick_ab.sh mrg26:auto mrg26:auto:--consume mrg26:auto:--consume\ --no-write
done
ncu --set full --clock-control none -k regex:gen_mrg -c 1 -o gpurun_out/s2c_mrg26 python bench.py --workload mrg26 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --sustained-s 0 > /dev/null 2>&1; echo "ncu rc=$?"
