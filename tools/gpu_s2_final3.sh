#!/bin/bash
# Session-2 final evidence: build, GPU suite, smoke (+ launch list), bench sweep of every workload,
# default line (+ launch list) and a 20-step line, ncu of the MRG32k3a kernels after the last changes.
mkdir -p gpurun_out
python -m paper_1401_8230_b200.build > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -rs > gpurun_out/s2x_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s2x_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2x_smoke.log 2>&1; echo "smoke rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2x_smoke_launches.csv \
    python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
bash tools/bench_all.sh
cp gpurun_out/bench_all.jsonl gpurun_out/s2x_bench_all.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/s2x_default_launches.csv python bench.py --steps 20 --warmup 5 --sustained-s 0 > /dev/null 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s2x_default20.log 2>&1; tail -1 gpurun_out/s2x_default20.log | cut -c1-160
bash tools/prof_one.sh s2x_mrg26 gen_mrg_kernel --workload mrg26
bash tools/prof_one.sh s2x_mrg26_consume consume_mrg_kernel --workload mrg26 --consume
echo done
