"""Cluster-split (distributed shared memory) histogram add rate vs the per-SM histogram
(tools/write_ceiling.cu wc_dsmem_hist / wc_smem_hist) on one B200."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_8230_b200 import build as B  # noqa: E402

L = ctypes.CDLL(B.build_tools())
L.wc_dsmem_hist.argtypes = [ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                            ctypes.c_void_p]
L.wc_smem_hist.argtypes = [ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                           ctypes.c_void_p]
sink = torch.zeros(1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
sms = torch.cuda.get_device_properties(0).multi_processor_count
res = {}


def rate(fn, grid_ctas, warps, iters=2048):
    for _ in range(2):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(5 * grid_ctas * warps * 32 * iters * 8 / (a.elapsed_time(b) * 1e-3) / 1e9, 1)


for warps in (16, 24):
    res[f"local_red_w{warps}"] = rate(lambda: L.wc_smem_hist(2048, 1, warps, st.cuda_stream, sink.data_ptr()), sms, warps)
    for c in (1, 2, 4):
        res[f"cluster{c}_w{warps}"] = rate(lambda: L.wc_dsmem_hist(2048, c, warps, st.cuda_stream, sink.data_ptr()), sms // c * c, warps)
print(json.dumps({"G_adds_per_s": res}))
