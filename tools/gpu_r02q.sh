#!/bin/bash
for wl in cfg1 cfg2; do for f in "--graph on --warm-l2"; do
  timeout 300 python bench.py --workload $wl --steps 300 --no-cpu-baseline --e2e-steps 0 $f 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$wl $f', round(d['value'],1), d['ms_per_step'], d['config']['cuda_graph'])"
done; done
