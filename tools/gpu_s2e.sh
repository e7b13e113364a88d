#!/bin/bash
# MRG32k3a constants pinned in registers (PRNGD_MRG_REGCONST=1, variants/lib_mrc1.so) vs product.
mkdir -p gpurun_out
PRNGD_LIB=$PWD/variants/lib_mrc1.so timeout 900 python -m pytest tests -q -m gpu -x -k "mrg or MRG" 2>&1 | tail -2
for i in 1 2; do
PRNGD_LIB=$PWD/variants/lib_mrc1.so STEPS=50 TAG=regconst bash tools/quick_ab.sh mrg26:auto mrg26:auto:--consume mrg26:auto:--consume\ --no-write
STEPS=50 TAG=product bash tools/quick_ab.sh mrg26:auto mrg26:auto:--consume mrg26:auto:--consume\ --no-write
done
