#!/bin/bash
# MRG32k3a fill-loop step A/B (draws per lane per step; 3: 304, 6: 326, 9: 330 Gd/s)
for i in 1 2; do
for v in step9 step12 step15 step18 step24; do PRNGD_LIB=$PWD/paper_1401_8230_b200/libprngd_$v.so TAG=$v STEPS=50 bash tools/quick_ab.sh mrg26:auto; done
done
