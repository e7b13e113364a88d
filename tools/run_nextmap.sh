set -x
python -m paper_1401_8230_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "mappings or random or parity" > gpurun_out/gputests.log 2>&1; echo tests=$?
out=gpurun_out/nextmap.jsonl; : > $out
for w in cfg3 eq5 eq6 open4 cfg3; do timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline --workload $w --steps 100 2>/dev/null | tail -1 >> $out; done
