#!/bin/bash
# Consumer A/B: the current library vs libprngd_head.so (the previous commit), cfg5 / cfg4 fused
timeout 900 python -m pytest tests -x -q -m gpu -k "consume or hist or cfg5 or random or wrap or exact or next_workloads" > gpurun_out/gputests.log 2>&1; echo tests=$?
H=$PWD/paper_1401_8230_b200/libprngd_head.so
for i in 1 2; do
TAG=new STEPS=50 bash tools/quick_ab.sh cfg5:auto "cfg5:auto:--no-write" "cfg4:auto:--consume"
PRNGD_LIB=$H TAG=head STEPS=50 bash tools/quick_ab.sh cfg5:auto "cfg5:auto:--no-write" "cfg4:auto:--consume"
done
