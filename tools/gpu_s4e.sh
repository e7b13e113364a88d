#!/bin/bash
# Session-4: same-box A/B of the default (histogram + moments) consumer before / after the
# histogram-only branch: variants/lib_head.so = the previous commit's sources.
mkdir -p gpurun_out
run() { timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline --sustained-s 0 "$@" 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$TAG', d['config']['workload'][:5], 'steps', d['steps'], 'val %.1f'%d['value'], 'best %.1f'%d['per_step']['value_at_best'], 'median %.1f'%d['per_step']['value_at_median'], d['clocks']['reasons'])"; }
for rep in 1 2 3; do
  TAG=new run --workload cfg5 --steps 20
  TAG=head PRNGD_LIB=$PWD/variants/lib_head.so run --workload cfg5 --steps 20
  TAG=new run --workload cfg4 --consume --steps 20
  TAG=head PRNGD_LIB=$PWD/variants/lib_head.so run --workload cfg4 --consume --steps 20
done 2>&1 | tee gpurun_out/s4e_cons_branch_ab.txt
