#!/bin/bash
# MRG32k3a parity + bench A/B (current library).  Ring sizes must hold a batch plus one 3-draw
# step (static_assert in prngd_kernels.cu; kMrgRing = 16 would never finish filling).
timeout 600 python -m pytest tests -x -q -m gpu -k "mrg" > gpurun_out/gputests.log 2>&1; echo tests=$?
for i in 1 2; do TAG=r32 STEPS=50 bash tools/quick_ab.sh mrg26:auto; done
