#!/bin/bash
# Jump-ahead kernel warps (streams) per CTA A/B on cfg2 (default 4)
for i in 1 2; do
TAG=jw4 STEPS=200 bash tools/quick_ab.sh cfg2:auto
for v in jw2 jw8; do PRNGD_LIB=$PWD/paper_1401_8230_b200/libprngd_$v.so TAG=$v STEPS=200 bash tools/quick_ab.sh cfg2:auto; done
done
