#!/bin/bash
# A/B: MRG32k3a kernel with the shared-memory ROW tile (default) vs register stores (PRNGD_MRG_STAGE=1)
V=$PWD/paper_1401_8230_b200/libprngd_mrgdirect.so
PRNGD_LIB=$V timeout 600 python -m pytest tests -x -q -m gpu -k "mrg" > gpurun_out/gputests_direct.log 2>&1; echo tests_direct=$?
for i in 1 2; do
TAG=tile STEPS=50 bash tools/quick_ab.sh mrg26:auto
PRNGD_LIB=$V TAG=direct STEPS=50 bash tools/quick_ab.sh mrg26:auto
done
