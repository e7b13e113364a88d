#!/bin/bash
# Round-2 session-2 evidence sweep: GPU suite, smoke (+ launch list), default bench line (+ launch list),
# bench sweep, ncu --set full of the dominant kernels.  Tag = $1 (e.g. s2z).
tag=${1:-s2z}
mkdir -p gpurun_out
python -m paper_1401_8230_b200.build > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -rs > gpurun_out/${tag}_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${tag}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_smoke_launches.csv \
    python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
python bench.py > gpurun_out/${tag}_default.log 2>&1; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_default_launches.csv python bench.py --steps 20 --warmup 5 --sustained-s 0 > /dev/null 2>&1
bash tools/bench_all.sh
bash tools/prof_one.sh ${tag}_cfg3_row gen_kernel --workload cfg3
bash tools/prof_one.sh ${tag}_cfg5_consume consume_kernel --workload cfg5
bash tools/prof_one.sh ${tag}_mrg26_consume consume_mrg_kernel --workload mrg26 --consume
bash tools/prof_one.sh ${tag}_mrg26 gen_mrg_kernel --workload mrg26
bash tools/prof_one.sh ${tag}_cfg2_jump gen_jump --workload cfg2
bash tools/prof_one.sh ${tag}_cfg1_seg gen_seg_kernel --workload cfg1
echo done
