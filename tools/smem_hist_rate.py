"""Shared-memory packed-histogram increment rate on one B200 (tools/write_ceiling.cu
wc_smem_hist): the peak the fused consumer's histogram path is measured against."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1401_8230_b200 import build as B  # noqa: E402

L = ctypes.CDLL(B.build_tools())
L.wc_smem_hist.argtypes = [ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                           ctypes.c_void_p]
sink = torch.zeros(1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
sms = torch.cuda.get_device_properties(0).multi_processor_count
res = {}
for red in (1, 0):
    for warps in (8, 16, 24, 32):
        iters = 2048
        for _ in range(2):
            L.wc_smem_hist(iters, red, warps, st.cuda_stream, sink.data_ptr())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            L.wc_smem_hist(iters, red, warps, st.cuda_stream, sink.data_ptr())
        b.record()
        torch.cuda.synchronize()
        ops = 5 * sms * warps * 32 * iters * 8
        res[f"{'red' if red else 'atomic_ret'}_w{warps}"] = round(ops / (a.elapsed_time(b) * 1e-3) / 1e9, 1)
print(json.dumps({"G_adds_per_s": res, "sms": sms}))
