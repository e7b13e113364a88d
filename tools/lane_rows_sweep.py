"""Per-lane row-store pattern (tools/write_ceiling.cu wc_lane_rows) vs the ROW kernel's
warp-coalesced row bursts (wc_segments S=1, chunk 512) on one B200: is a lane writing its own
row in 512-byte+ bursts (32-byte stores) as DRAM-friendly as the coalesced ROW flush?"""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_8230_b200 import build as B  # noqa: E402

L = ctypes.CDLL(B.build_tools())
L.wc_lane_rows.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                           ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64]
L.wc_segments.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                          ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64]
n = 1 << 30
out = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()


def timeit(fn, reps=20):
    for k in range(3):
        fn(k)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(reps):
        fn(10 + k)
    b.record()
    torch.cuda.synchronize()
    return reps * 8 * n / (a.elapsed_time(b) * 1e-3) / 1e9


res = {}
for cols in (1024, 2048):
    for pad_kb in (0, 8, 16):   # one-warp CTAs: 0 -> up to 32/SM (threads), 16 KiB -> 12-13/SM
        res[f"row512_cols{cols}_pad{pad_kb}k"] = timeit(
            lambda k: L.wc_segments(out.data_ptr(), n, 1, 512, pad_kb * 1024, k, st.cuda_stream, cols))
        for burst in (128, 256, 512, 1024):
            res[f"lane{burst}_cols{cols}_pad{pad_kb}k"] = timeit(
                lambda k: L.wc_lane_rows(out.data_ptr(), n, burst, pad_kb * 1024, k,
                                         st.cuda_stream, cols))
print(json.dumps({k: round(v) for k, v in res.items()}))
