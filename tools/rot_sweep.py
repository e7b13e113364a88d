"""Sweep the rotated-row write pattern (tools/write_ceiling.cu wc_rot) on one B200: does giving
each lane of the ROW kernel a column phase (d_r = r * skew mod chunks-per-row) raise the HBM
write ceiling the way 1 KiB segments do?  Usage: python tools/rot_sweep.py [cols ...]"""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_8230_b200 import build as B  # noqa: E402

L = ctypes.CDLL(B.build_tools())
L.wc_rot.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                     ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64]
L.wc_blockcol.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                          ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32]
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
    pad = 16 * 1024
    res[f"c{cols}_seg_S1"] = timeit(lambda k: L.wc_segments(out.data_ptr(), n, 1, 512, pad, k, st.cuda_stream, cols))
    res[f"c{cols}_seg_1KiB"] = timeit(lambda k: L.wc_segments(out.data_ptr(), n, cols // 128, 512, pad, k, st.cuda_stream, cols))
    for S, chunk, padk in ((8, 512, 150), (8, 512, 185), (8, 256, 88), (8, 256, 120), (8, 256, 60),
                           (16, 256, 150), (16, 512, 210), (4, 512, 72)):
        res[f"c{cols}_blockcol_S{S}_chunk{chunk}_pad{padk}k"] = timeit(
            lambda k: L.wc_blockcol(out.data_ptr(), n, S, padk * 1024, k, st.cuda_stream, cols, chunk))
    for M in ():
        for skew in (0, 1, 2, 3, 5, 7):
            res[f"c{cols}_rot_M{M}_skew{skew}"] = timeit(
                lambda k: L.wc_rot(out.data_ptr(), n, M, skew, pad, k, st.cuda_stream, cols))
print(json.dumps({k: round(v) for k, v in res.items()}))
