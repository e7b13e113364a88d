#!/bin/bash
# Session-4 re-entry check: GPU suite, smoke (+ launch list), default bench line (+ launch list).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rs -x > gpurun_out/s4a_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4a_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4a_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/s4a_bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s4a_bench_default.log | cut -c1-400
for w in cfg1 cfg2 cfg5; do timeout 600 python bench.py --workload $w --e2e-steps 0 --no-cpu-baseline --steps 50 2>/dev/null | tail -1 | cut -c1-300; done
echo done
