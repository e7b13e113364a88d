"""Pure-store ceilings of candidate fused-consumer layouts (cfg5 rows of 2048 doubles, 128-byte
chunks per lane per flush, one-warp CTAs whose number per SM is set by a shared-memory pad):
S lanes per row (row segments by jump-ahead) and W warps per SM.  Question: does sharing rows
between lanes (fewer rows in flight per SM) raise the 5.2 TB/s ceiling of the current layout
(S = 1, 12 warps)?  tools/write_ceiling.cu wc_segments."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_8230_b200 import build as B  # noqa: E402

L = ctypes.CDLL(B.build_tools())
L.wc_segments.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                          ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64]
n = 1 << 31
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
pads = {8: 27000, 12: 18000, 16: 13500, 20: 10800, 24: 9000}   # bytes -> one-warp CTAs per SM
for S in (1, 2, 4, 16):
    for w, pad in pads.items():
        for chunk in (128, 256):
            res[f"S{S}_w{w}_chunk{chunk}"] = timeit(
                lambda k: L.wc_segments(out.data_ptr(), n, S, chunk, pad, k, st.cuda_stream, 2048))
print(json.dumps({k: round(v) for k, v in res.items()}))
