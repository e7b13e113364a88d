#!/bin/bash
# A/B: jump kernel compaction run padded by 8 bytes per 16 outputs (current) vs unpadded (head)
timeout 900 python -m pytest tests -x -q -m gpu -k "jump or cfg2 or random" > gpurun_out/gputests.log 2>&1; echo tests=$?
H=$PWD/paper_1401_8230_b200/libprngd_head.so
for i in 1 2; do
TAG=pad STEPS=200 bash tools/quick_ab.sh cfg2:auto "cfg1:auto:--flags 512"
PRNGD_LIB=$H TAG=head STEPS=200 bash tools/quick_ab.sh cfg2:auto "cfg1:auto:--flags 512"
done
