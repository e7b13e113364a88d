#!/bin/bash
# Run bench.py over every BASELINE config on one B200 (under gpurun); JSON lines -> gpurun_out/
out=gpurun_out/bench_all.jsonl; : > $out
run() { timeout 600 python bench.py --e2e-steps 0 "$@" 2>/dev/null | tail -1 >> $out; }
run --workload cfg1 --steps 200
run --workload cfg2 --steps 200
run --workload cfg3 --steps 200
run --workload cfg4 --steps 50
run --workload cfg4 --steps 50 --consume
run --workload cfg5 --steps 50
run --workload cfg5 --steps 50 --no-write
run --workload mrg26 --steps 50
echo done
