# MRG32k3a: parity tests + bench on the mrg26 workload (one B200)
python -m paper_1401_8230_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "mrg" > gpurun_out/gputests.log 2>&1; echo tests=$?
out=gpurun_out/mrg_ab.jsonl; : > $out
for i in 1 2; do timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline --workload mrg26 --steps 50 2>/dev/null | tail -1 >> $out; done
