#!/bin/bash
timeout 900 python -m pytest tests -q -m gpu -x -k "seg or jump or cfg1 or random or misaligned or guard" > gpurun_out/gputests_r.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gputests_r.log
for rep in 1 2; do
  timeout 300 python bench.py --workload cfg1 --steps 300 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg1', round(d['value'],1), d['per_step']['step_ms_median'], d['roofline']['kernel'])"
done
bash tools/prof_one.sh r02r_cfg1_segw gen_segw_kernel --workload cfg1
