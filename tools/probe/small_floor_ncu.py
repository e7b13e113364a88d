"""One launch of each small-floor probe kernel and of the library's cfg1 / cfg2 steps, for an ncu
launch list (gpu__time_duration, sm__cycles_active): python tools/probe/small_floor_ncu.py"""
import ctypes, os, subprocess, sys
import torch
here = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(here)))
from paper_1401_8230_b200 import prngd as P  # noqa: E402
from paper_1401_8230_b200 import workloads as W  # noqa: E402
so = os.path.join(here, "libsmallfloor.so")
if not os.path.exists(so):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-O3", "-shared", "-Xcompiler", "-fPIC", "-o", so,
                           os.path.join(here, "small_floor.cu")])
L = ctypes.CDLL(so)
L.probe_empty.argtypes = [ctypes.c_uint, ctypes.c_uint, ctypes.c_void_p]
L.probe_rows.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint, ctypes.c_void_p]
S = torch.cuda.current_stream().cuda_stream
for name in ("cfg1", "cfg2"):
    cfg = W.config(name)
    nout = cfg["n_streams"] * cfg["n_per_stream"]
    out = torch.empty(nout, dtype=torch.float64, device="cuda")
    g = P.Generator(**cfg)
    for _ in range(3):
        P.prngd_generate(g.handle, out, torch.cuda.current_stream())
        L.probe_empty(1024, 32, S)
        L.probe_rows(out.data_ptr(), cfg["n_per_stream"] // 2, cfg["n_streams"], 1, S)
    torch.cuda.synchronize()
print("done")
