#!/bin/bash
# Run bench.py over every BASELINE config and the NEXT workloads on one B200 (under gpurun);
# JSON lines -> gpurun_out/bench_all.jsonl.  Write workloads carry the >= 1.5 s sustained record.
out=gpurun_out/bench_all.jsonl; : > $out
run() { timeout 900 python bench.py --e2e-steps 0 --no-cpu-baseline "$@" 2>/dev/null | tail -1 >> $out; }
run --workload cfg1 --steps 200
run --workload cfg2 --steps 200
run --workload cfg3 --steps 200
run --workload cfg3 --steps 200 --store seg
run --workload cfg3 --steps 50 --consume
run --workload cfg4 --steps 50
run --workload cfg4 --steps 50 --consume
run --workload cfg5 --steps 50
run --workload cfg5 --steps 50 --store row
run --workload cfg5 --steps 50 --no-write
run --workload mrg26 --steps 50
run --workload mrg26 --steps 20 --consume
run --workload mrg26 --steps 20 --consume --no-write
run --workload eq5 --steps 100
run --workload eq6 --steps 100
run --workload open4 --steps 100
python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log >> $out
python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1 >> $out
echo done
