#!/bin/bash
# Session-4: histogram-only consumer (d_pow = NULL): new tests, full GPU suite, smoke, A/B bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hist_only.py -q -x > gpurun_out/s4d_histonly_tests.log 2>&1; echo "hist-only tests rc=$?"; tail -5 gpurun_out/s4d_histonly_tests.log
timeout 1500 python -m pytest tests -q -m gpu -rs > gpurun_out/s4d_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4d_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4d_smoke.log 2>&1; echo "smoke rc=$?"
out=gpurun_out/s4d_bench.jsonl; : > $out
run() { timeout 900 python bench.py --e2e-steps 0 --no-cpu-baseline "$@" 2>/dev/null | tail -1 >> $out; }
for rep in 1 2; do
run --workload cfg4 --steps 50 --consume
run --workload cfg4 --steps 50 --consume --hist-only
run --workload cfg5 --steps 50
run --workload cfg5 --steps 50 --hist-only
run --workload cfg5 --steps 50 --no-write
run --workload cfg5 --steps 50 --no-write --hist-only
done
run --workload cfg4 --steps 5 --consume --hist-only --sustained-s 0
run --workload mrg26 --steps 20 --consume
run --workload mrg26 --steps 20 --consume --hist-only
python bench.py --steps 20 --warmup 5 > gpurun_out/s4d_default20.log 2>&1; tail -1 gpurun_out/s4d_default20.log | cut -c1-200
python - <<'P'
import json
for l in open('gpurun_out/s4d_bench.jsonl'):
    try: d=json.loads(l)
    except Exception: print('bad line', l[:100]); continue
    c=d['config']; s=d.get('sustained') or {}
    print(c['workload'][:6], c.get('statistics'), 'write' if c['write_outputs'] else 'nowrite', 'steps', d['steps'], 'val %.1f'%d['value'], 'best %.1f'%d['per_step']['value_at_best'], 'sust %.1f'%s.get('value',0), d['clocks']['reasons'])
P
