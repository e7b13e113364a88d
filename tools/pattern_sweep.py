"""Sweep the write-pattern microbenchmark (tools/write_ceiling.cu wc_pattern) on one B200."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_8230_b200 import build as B  # noqa: E402

L = ctypes.CDLL(B.build_tools())
L.wc_pattern.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                         ctypes.c_uint64, ctypes.c_void_p]
L.wc_store.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                       ctypes.c_void_p]
n = 1 << 30
out = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()


def timeit(fn, reps=10):
    for k in range(2):
        fn(k)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(reps):
        fn(10 + k)
    b.record()
    torch.cuda.synchronize()
    return reps * 8 * n / (a.elapsed_time(b) * 1e-3) / 1e9


res = {}
res["contig_stg32"] = timeit(lambda k: L.wc_store(out.data_ptr(), n, 1, k, st.cuda_stream))
for pad_kb in (0, 20, 28, 50, 100):  # 0: full occupancy; 50 KB pad -> 4 CTAs/SM, 100 -> 2
    for burst in (128, 256, 512, 1024, 2048, 8192):
        res[f"burst{burst}_pad{pad_kb}k"] = timeit(
            lambda k: L.wc_pattern(out.data_ptr(), n, burst, pad_kb * 1024, k, st.cuda_stream))
print(json.dumps({k: round(v) for k, v in res.items()}))
