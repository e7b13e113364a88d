"""Host-side cost of one prngd_generate call vs the device time per step (small configs)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1401_8230_b200 import prngd as P  # noqa: E402
from paper_1401_8230_b200 import workloads as W  # noqa: E402

for name in ("cfg1", "cfg2"):
    g = P.Generator(**W.config(name))
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(10):
        P.prngd_generate(g.handle, out, st)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        P.prngd_generate(g.handle, out, st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        P.prngd_generate(g.handle, out, st)
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: host enqueue {1e6 * (t1 - t0) / n:.2f} us/call, wall {1e6 * (t2 - t0) / n:.2f} "
          f"us/call, device {1e3 * a.elapsed_time(b) / n:.2f} us/step")
