#!/bin/bash
timeout 900 python -m pytest tests -q -m gpu -x -k "consume or fullsize or segments or hist" > gpurun_out/gputests_j.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_j.log
for rep in 1 2; do
  for wl in "cfg5" "cfg3 --consume" "cfg4 --consume"; do
    timeout 300 python bench.py --workload $wl --steps 50 --sustained-s 1.5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$wl', round(d['value'],1), 'sus', round(d['sustained']['value'],1), d['clocks']['sm_mhz'], d['sustained']['clocks']['sm_mhz'])"
  done
  for st in auto seg; do for wl in cfg3 cfg4; do
    timeout 300 python bench.py --workload $wl --store $st --steps 50 --sustained-s 1.5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$wl $st', round(d['value'],1), 'sus', round(d['sustained']['value'],1), d['clocks']['sm_mhz'], d['sustained']['clocks']['sm_mhz'])"
  done; done
done
