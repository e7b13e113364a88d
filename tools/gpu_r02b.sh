#!/bin/bash
# Round 2, second pass: GPU suite after the A/B-path gating, per-lane row-store pattern sweep,
# jump-kernel occupancy A/B (cfg2), ncu of the few-stream kernels (cfg1 SEG, cfg2 jump).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -rs -x > gpurun_out/gputests_b.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gputests_b.log
timeout 600 python tools/lane_rows_sweep.py > gpurun_out/lane_rows.json 2>&1; echo "sweep rc=$?"
for v in default jmin1 default jmin1; do
  if [ $v = default ]; then L=""; else L=variants/lib_$v.so; fi
  for wl in cfg2 cfg1; do
    PRNGD_LIB=$L timeout 300 python bench.py --workload $wl --steps 300 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v $wl', round(d['value'],1), d['per_step'])"
  done
done > gpurun_out/jump_ab.txt 2>&1
bash tools/prof_one.sh r02b_cfg1_seg gen_seg_kernel --workload cfg1
bash tools/prof_one.sh r02b_cfg2_jump gen_jump_kernel --workload cfg2
echo done
