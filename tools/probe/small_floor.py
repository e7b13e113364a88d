"""What a step of the small configs costs at the floor: empty launches and plain store kernels
of cfg1 / cfg2's output size, timed exactly as bench.py times those configs (256 MiB written
and another 256 MiB read between steps, CUDA events around the step alone), next to the
library's own cfg1 / cfg2 steps."""
import ctypes, json, os, statistics, subprocess, sys
import torch
here = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(here)))
from paper_1401_8230_b200 import prngd as P  # noqa: E402
from paper_1401_8230_b200 import workloads as W  # noqa: E402

so = os.path.join(here, "libsmallfloor.so")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                       "-O3", "-shared", "-Xcompiler", "-fPIC", "-o", so,
                       os.path.join(here, "small_floor.cu")])
L = ctypes.CDLL(so)
L.probe_empty.argtypes = [ctypes.c_uint, ctypes.c_uint, ctypes.c_void_p]
L.probe_rows.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint,
                         ctypes.c_void_p]
L.probe_flat.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint, ctypes.c_uint,
                         ctypes.c_void_p]
scratch = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
scratch_rd = torch.zeros(32 << 20, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
S = st.cuda_stream


def timed(fn, steps=300, warm=5, flush=True):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    for k in range(steps):
        if flush:
            scratch.fill_(float(k))
            scratch_rd.sum()
        ev[k][0].record(st)
        fn()
        ev[k][1].record(st)
    torch.cuda.synchronize()
    per = [a.elapsed_time(b) * 1e3 for a, b in ev]
    return round(statistics.median(per), 2), round(min(per), 2)


res = {}
for name in ("cfg1", "cfg2"):
    cfg = W.config(name)
    nout = cfg["n_streams"] * cfg["n_per_stream"]
    out = torch.empty(nout, dtype=torch.float64, device="cuda")
    g = P.Generator(**cfg)
    rows, rd2 = cfg["n_streams"], cfg["n_per_stream"] // 2
    cases = {
        "prngd": lambda: P.prngd_generate(g.handle, out, st),
        "empty 1024x32": lambda: L.probe_empty(1024, 32, S),
        "empty 148x128": lambda: L.probe_empty(148, 128, S),
        "rows 1 warp/CTA": lambda: L.probe_rows(out.data_ptr(), rd2, rows, 1, S),
        "rows 4 warps/CTA": lambda: L.probe_rows(out.data_ptr(), rd2, rows, 4, S),
        "flat 148x1024": lambda: L.probe_flat(out.data_ptr(), nout // 2, 148, 1024, S),
        "flat 592x512": lambda: L.probe_flat(out.data_ptr(), nout // 2, 592, 512, S),
    }
    for k, fn in cases.items():
        for flush in (True, False):
            med, best = timed(fn, flush=flush)
            key = f"{name} {k} {'flush' if flush else 'warm'}"
            res[key] = {"us_median": med, "us_best": best,
                        "Gd_s_median": round(nout / (med * 1e-6) / 1e9, 1)}
            print(key, res[key], flush=True)
print(json.dumps(res))
