#!/bin/bash
# Fused consumer warps per SM / tile columns A/B (default 16 warps x 16 columns)
for i in 1 2; do
TAG=w16 STEPS=50 bash tools/quick_ab.sh cfg5:auto "cfg4:auto:--consume"
for v in w8 w10 w12 w12c32; do PRNGD_LIB=$PWD/paper_1401_8230_b200/libprngd_$v.so TAG=$v STEPS=50 bash tools/quick_ab.sh cfg5:auto "cfg4:auto:--consume"; done
done
