"""Sweep the segmented-row write pattern (tools/write_ceiling.cu wc_segments) on one B200.

Question: does splitting each row across S lanes (intra-stream parallelism via jump-ahead)
raise the HBM write ceiling above the ROW kernel's pattern (S = 1, 512 B chunks, 16 KiB smem)?
Usage: python tools/segment_sweep.py [cols ...]"""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_8230_b200 import build as B  # noqa: E402

L = ctypes.CDLL(B.build_tools())
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
for cols in [int(c) for c in sys.argv[1:]] or [1024]:
    for pad_kb in (16, 8):
        for S in (1, 2, 4, 8, 16, 32):
            for chunk in (256, 512, 1024):
                if cols * 8 // S < chunk:
                    continue
                res[f"c{cols}_S{S}_chunk{chunk}_pad{pad_kb}k"] = timeit(
                    lambda k: L.wc_segments(out.data_ptr(), n, S, chunk, pad_kb * 1024, k,
                                            st.cuda_stream, cols))
print(json.dumps({k: round(v) for k, v in res.items()}))
