#!/bin/bash
# MRG32k3a output staging A/B: ROW tile beside the rings (0, default) vs in-ring staging (2)
V=$PWD/paper_1401_8230_b200/libprngd_stage2.so
PRNGD_LIB=$V timeout 600 python -m pytest tests -x -q -m gpu -k "mrg" > gpurun_out/gputests_stage2.log 2>&1; echo tests_stage2=$?
for i in 1 2; do
TAG=stage0 STEPS=50 bash tools/quick_ab.sh mrg26:auto
PRNGD_LIB=$V TAG=stage2 STEPS=50 bash tools/quick_ab.sh mrg26:auto
done
