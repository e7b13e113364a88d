#!/bin/bash
# Round-1 closing sweep after the 12-warp consumer: full GPU suite, smoke, default bench line
# + launch list, bench sweep.
mkdir -p gpurun_out
python -m paper_1401_8230_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gputests_full.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/r01l_default_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/r01l_default_launches.csv python bench.py > /dev/null 2>&1
bash tools/prof_one.sh r01l_cfg5_consume consume_kernel --workload cfg5
bash tools/bench_all.sh
echo done
