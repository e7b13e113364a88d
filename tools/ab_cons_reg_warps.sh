#!/bin/bash
# Consume-only (no output) kernel: warps per SM A/B (default 24)
for i in 1 2; do
TAG=r24 STEPS=50 bash tools/quick_ab.sh "cfg5:auto:--no-write"
for v in r12 r16 r20 r28 r32; do PRNGD_LIB=$PWD/paper_1401_8230_b200/libprngd_$v.so TAG=$v STEPS=50 bash tools/quick_ab.sh "cfg5:auto:--no-write"; done
done
