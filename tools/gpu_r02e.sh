#!/bin/bash
# Round 2: full GPU suite after NEXT-4 + fused MRG consumer, smoke, bench lines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rs > gpurun_out/gputests_e.log 2>&1; echo "tests rc=$?"; tail -8 gpurun_out/gputests_e.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_e.log 2>&1; echo "smoke rc=$?"
python -c "
from paper_1401_8230_b200 import prngd as P, dist as D
import torch
torch.cuda.set_device(0)
print('mc supported attr:', P.prngd_mc_supported())
try:
    m = D.McStats(); print('McStats OK'); m.close()
except Exception as e: print('McStats refused:', e)
" > gpurun_out/mc_probe_e.log 2>&1
cat gpurun_out/mc_probe_e.log
PRNGD_BENCH_SAME_GPU=1 PRNGD_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --sustained-s 0 > gpurun_out/bench_n2_samegpu.log 2>&1; echo "n2 rc=$?"; tail -1 gpurun_out/bench_n2_samegpu.log | cut -c1-600
python bench.py > gpurun_out/r02e_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02e_default.log | cut -c1-300
echo done
