#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (every product kernel family, small ragged shapes)
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
python tools/sanitize_cases.py > gpurun_out/san_plain.txt 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py \
      > gpurun_out/san_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_$tool.txt
  tail -3 gpurun_out/san_$tool.txt
done
