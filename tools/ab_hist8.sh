#!/bin/bash
# Timing-only A/B (wrong histograms): 64 KiB 8-bit-field histogram simulation with longer bursts
# or more warps, against the current consumer (cfg5 write + histogram + moments).
for i in 1 2; do
TAG=cur STEPS=50 bash tools/quick_ab.sh cfg5:auto
for v in h8_16 h8_32 h8_w20 h8_w24; do
PRNGD_LIB=$PWD/paper_1401_8230_b200/libprngd_$v.so TAG=$v STEPS=50 bash tools/quick_ab.sh cfg5:auto
done
done
