#!/bin/bash
# Round-2 first GPU pass: full GPU suite, smoke (with its launch list), default bench line,
# bench sweep over the configs.
mkdir -p gpurun_out
python -m paper_1401_8230_b200.build > gpurun_out/build.log 2>&1
nvidia-smi -L > gpurun_out/devices.txt
timeout 1800 python -m pytest tests -q -m gpu -rs > gpurun_out/gputests_full.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv \
    python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
python bench.py > gpurun_out/r02a_default.log 2>&1; echo "bench rc=$?"
bash tools/bench_all.sh
echo done
