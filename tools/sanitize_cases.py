"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_8230_b200 import prngd as P  # noqa: E402
from paper_1401_8230_b200 import workloads as W  # noqa: E402

cases = []
for store in ("row", "tma", "tile", "direct", "row1k"):
    cases.append(("gen " + store, W.config("cfg1", n_streams=300, n_per_stream=200,
                                            flags=P.STORE_FLAGS[store] | P.PRNGD_FLAG_NO_JUMP)))
cases.append(("gen cfg2", W.config("cfg2", n_streams=100, n_per_stream=130, flags=P.PRNGD_FLAG_NO_JUMP)))
cases.append(("jump", W.config("cfg2", n_streams=50, n_per_stream=1500, flags=P.PRNGD_FLAG_JUMP)))
cases.append(("eq5 open", W.config("cfg4", n_streams=64, n_per_stream=96,
                                   flags=P.PRNGD_FLAG_MAP_EQ5 | P.PRNGD_FLAG_OPEN)))
cases.append(("mrg", dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1, seed=1, n_streams=70,
                          n_per_stream=100, flags=P.PRNGD_FLAG_MRG32K3A)))
for name, p in cases:
    g = P.Generator(**p)
    out = g.generate()
    torch.cuda.synchronize()
    print("ok", name, out.shape, flush=True)
for store in ("row", "tma", "tile", "direct"):
    g = P.Generator(**W.config("cfg1", n_streams=400, n_per_stream=100, flags=P.STORE_FLAGS[store]))
    g.generate_consume(torch.empty(g.shape, dtype=torch.float64, device="cuda"))
    g.generate_consume()
    torch.cuda.synchronize()
    print("ok consume", store, flush=True)
g = P.Generator(**W.config("cfg1", n_streams=64, n_per_stream=64))
g.raw(10), g.pairs(), g.generate_host()
torch.cuda.synchronize()
print("ok debug/host", flush=True)
