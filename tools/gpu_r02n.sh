#!/bin/bash
timeout 900 python -m pytest tests -q -m gpu -x -k "jump or cfg2 or random" > gpurun_out/gputests_n.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gputests_n.log
for rep in 1 2; do
  timeout 300 python bench.py --workload cfg2 --steps 300 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg2', round(d['value'],1), d['per_step']['step_ms_median'], d['roofline']['kernel'])"
done
bash tools/prof_one.sh r02n_cfg2_jump gen_jump_kernel --workload cfg2
