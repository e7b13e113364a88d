#!/bin/bash
# Round-2 closing evidence (session 4, re-created container): GPU suite, smoke (+ launch list), bench sweep of every
# workload (with sustained records), default line (+ launch list), a 20-step line, reference arm.
mkdir -p gpurun_out
python -m paper_1401_8230_b200.build > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -rs > gpurun_out/s4f_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4f_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4f_smoke.log 2>&1; echo "smoke rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4f_smoke_launches.csv \
    python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
bash tools/bench_all.sh
cp gpurun_out/bench_all.jsonl gpurun_out/s4f_bench_all.jsonl
cp gpurun_out/bench_default.log gpurun_out/s4f_bench_default.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/s4f_default_launches.csv python bench.py --steps 20 --warmup 5 --sustained-s 0 > /dev/null 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s4f_default20.log 2>&1; tail -1 gpurun_out/s4f_default20.log | cut -c1-160

# ncu --set full of the two dominant kernels on the final code (after their plain runs exit 0)
bash tools/prof_one.sh s4f_cfg3_row gen_kernel --workload cfg3
bash tools/prof_one.sh s4f_cfg5_consume consume_kernel --workload cfg5
rm -f gpurun_out/s4f_*_sass.csv
echo final done
