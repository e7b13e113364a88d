#!/bin/bash
# Small configs: device time per step vs an empty kernel under the same event timing, and the
# ncu duration of each small-config kernel (cfg1 SEG, cfg2 jump-ahead).
python - <<'PY' > gpurun_out/small_probe.txt 2>&1
import torch, time
torch.cuda.init()
x = torch.empty(1, device="cuda")
s = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def evt(fn, n=200, fl=True):
    ts = []
    for _ in range(n):
        if fl: flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    ts.sort(); return ts[len(ts)//2], ts[0]
print("empty (x.add_ 1 elem) median/best us:", evt(lambda: x.add_(1)))
import sys; sys.path.insert(0, ".")
from paper_1401_8230_b200 import prngd as P, workloads as W
for name in ("cfg1", "cfg2"):
    g = P.Generator(**W.config(name))
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    print(name, P.prngd_get_info(g.handle), "median/best us:", evt(lambda: P.prngd_generate(g.handle, out, s)))
PY
ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gen_ -c 6 python bench.py --workload cfg1 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/small_ncu_cfg1.txt 2>&1
ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gen_ -c 6 python bench.py --workload cfg2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/small_ncu_cfg2.txt 2>&1
echo done
