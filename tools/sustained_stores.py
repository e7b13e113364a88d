"""Pure-store HBM write bandwidth vs run length (power-cap behaviour) on one B200.
python tools/sustained_stores.py -> JSON {pattern: {reps: GB/s}} plus SM clock / power medians."""
import ctypes
import json
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_1401_8230_b200 import build as B  # noqa: E402

L = ctypes.CDLL(B.build_tools())
L.wc_segments.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                          ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64]
L.wc_store.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                       ctypes.c_void_p]
import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
n = 1 << 30
out = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()


def run(fn, reps):
    for k in range(3):
        fn(k)
    torch.cuda.synchronize()
    clk, pw, stop = [], [], threading.Event()

    def sample():
        while not stop.is_set():
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000)
            time.sleep(0.005)
    t = threading.Thread(target=sample)
    t.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(reps):
        fn(10 + k)
    b.record()
    torch.cuda.synchronize()
    stop.set()
    t.join()
    return {"GBs": round(reps * 8 * n / (a.elapsed_time(b) * 1e-3) / 1e9),
            "sm_mhz": statistics.median(clk) if clk else None,
            "power_w": round(statistics.median(pw)) if pw else None}


pats = {
    "row_pattern": lambda k: L.wc_segments(out.data_ptr(), n, 1, 512, 16384, k, st.cuda_stream, 1024),
    "seg_1KiB": lambda k: L.wc_segments(out.data_ptr(), n, 8, 512, 16384, k, st.cuda_stream, 1024),
    "contig_stg32": lambda k: L.wc_store(out.data_ptr(), n, 1, k, st.cuda_stream),
}
res = {}
for name, fn in pats.items():
    res[name] = {reps: run(fn, reps) for reps in (50, 1000)}
    time.sleep(2)
print(json.dumps(res))
