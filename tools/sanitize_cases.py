"""Small invocations of every product kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck):  compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_cases.py

Shapes are small (the sanitizer slows kernels 10-100x) but ragged, and each case names the
kernel the host plan should pick for it (checked through prngd_get_info where it reports one).
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_8230_b200 import prngd as P  # noqa: E402
from paper_1401_8230_b200 import workloads as W  # noqa: E402

MRG = dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1, seed=1, stream_begin=0)
only = sys.argv[1:]  # optional case-name filter (substring)


def want(name):
    return not only or any(o in name for o in only)


gen_cases = [
    ("gen row", W.config("cfg1", n_streams=300, n_per_stream=200, flags=P.PRNGD_FLAG_STORE_ROW)),
    ("gen row cfg2 (w=8)", W.config("cfg2", n_streams=100, n_per_stream=130,
                                    flags=P.PRNGD_FLAG_NO_JUMP)),
    ("gen row cfg4 (asym)", W.config("cfg4", n_streams=150, n_per_stream=96)),
    ("gen seg 32-output segments", W.config("cfg1", n_streams=40, n_per_stream=1024)),
    ("gen seg 128-output segments", W.config("cfg1", n_streams=37, n_per_stream=4096,
                                             flags=P.PRNGD_FLAG_STORE_SEG)),
    ("jump 17 pairs", W.config("cfg2", n_streams=50, n_per_stream=700, flags=P.PRNGD_FLAG_JUMP)),
    ("jump 33 pairs", W.config("cfg2", n_streams=50, n_per_stream=1500, flags=P.PRNGD_FLAG_JUMP)),
    ("eq5 open", W.config("cfg4", n_streams=64, n_per_stream=96,
                          flags=P.PRNGD_FLAG_MAP_EQ5 | P.PRNGD_FLAG_OPEN)),
    ("eq6", W.config("cfg3", n_streams=64, n_per_stream=96, flags=P.PRNGD_FLAG_MAP_EQ6)),
    ("alg1", W.config("cfg4", n_streams=70, n_per_stream=90, flags=P.PRNGD_FLAG_ALG1)),
    ("ieee div", W.config("cfg1", n_streams=70, n_per_stream=90, flags=P.PRNGD_FLAG_IEEE_DIV)),
    ("mrg", dict(MRG, n_streams=70, n_per_stream=100, flags=P.PRNGD_FLAG_MRG32K3A)),
]
for name, p in gen_cases:
    if not want(name):
        continue
    g = P.Generator(**p)
    out = g.generate()
    torch.cuda.synchronize()
    print("ok", name, tuple(out.shape), "kernel", g.info.get("kernel"), flush=True)

consume_cases = [
    ("consume row tile", W.config("cfg1", n_streams=400, n_per_stream=100)),
    ("consume row segments", W.config("cfg5", n_streams=600, n_per_stream=256)),
    ("consume exact pass", W.config("cfg1", n_streams=300, n_per_stream=64,
                                    flags=P.PRNGD_FLAG_EXACT_HIST)),
    ("consume mrg fused", dict(MRG, n_streams=300, n_per_stream=96, flags=P.PRNGD_FLAG_MRG32K3A)),
    ("consume jump config", W.config("cfg2", n_streams=40, n_per_stream=1100)),
]
for name, p in consume_cases:
    if not want(name):
        continue
    g = P.Generator(**p)
    g.generate_consume(torch.empty(g.shape, dtype=torch.float64, device="cuda"))
    g.generate_consume()  # statistics only
    torch.cuda.synchronize()
    print("ok", name, flush=True)

if want("host"):
    g = P.Generator(**W.config("cfg1", n_streams=90, n_per_stream=300))
    g.generate_host()
    torch.cuda.synchronize()
    print("ok generate_host", flush=True)
if want("pairs"):
    g = P.Generator(**W.config("cfg2", n_streams=33, n_per_stream=1030))
    g.pairs()
    torch.cuda.synchronize()
    print("ok debug_pairs", flush=True)
print("all cases ran", flush=True)
