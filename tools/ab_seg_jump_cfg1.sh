#!/bin/bash
# cfg1 (cold L2 every step): SEG lane-start jump variants (PRNGD_SEG_JUMP 4 = default byte tables
# with the lane innermost; 0 byte tables; 1 nibble tables; 2 nibble tables by binary decomposition)
for v in sj0 sj1 sj2; do
PRNGD_LIB=$PWD/paper_1401_8230_b200/libprngd_$v.so timeout 600 python -m pytest tests -x -q -m gpu -k "seg and cfg1" > gpurun_out/gputests_$v.log 2>&1; echo tests_$v=$?
done
for i in 1 2; do
TAG=sj4 STEPS=300 bash tools/quick_ab.sh cfg1:auto
for v in sj0 sj1 sj2; do PRNGD_LIB=$PWD/paper_1401_8230_b200/libprngd_$v.so TAG=$v STEPS=300 bash tools/quick_ab.sh cfg1:auto; done
done
