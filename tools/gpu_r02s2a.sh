#!/bin/bash
# Session-2 re-entry check: GPU suite, smoke, default bench line, quick lines for the weak rows.
mkdir -p gpurun_out
python -m paper_1401_8230_b200.build > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -x -rs > gpurun_out/s2a_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s2a_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/s2a_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s2a_default.log
STEPS=50 bash tools/quick_ab.sh cfg5:auto cfg4:auto:--consume mrg26:auto mrg26:auto:--consume 
STEPS=200 bash tools/quick_ab.sh cfg1:auto cfg2:auto
