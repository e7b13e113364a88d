#!/bin/bash
# A/B: pairs per lane per round of the jump kernel (PRNGD_JUMP_PAIRS; 16 = default)
for v in p17 p24; do
PRNGD_LIB=$PWD/paper_1401_8230_b200/libprngd_$v.so timeout 900 python -m pytest tests -x -q -m gpu -k "jump" > gpurun_out/gputests_$v.log 2>&1; echo tests_$v=$?
done
for i in 1 2; do
TAG=p16 STEPS=200 bash tools/quick_ab.sh cfg2:auto
for v in p17 p18 p24; do PRNGD_LIB=$PWD/paper_1401_8230_b200/libprngd_$v.so TAG=$v STEPS=200 bash tools/quick_ab.sh cfg2:auto; done
done
