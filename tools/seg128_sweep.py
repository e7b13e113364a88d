import ctypes, json, sys, torch
sys.path.insert(0, ".")
from paper_1401_8230_b200 import build as B
L = ctypes.CDLL(B.build_tools())
L.wc_segments.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64]
n = 1 << 30
out = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
def timeit(fn, reps=20):
    for k in range(3): fn(k)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(reps): fn(10 + k)
    b.record(); torch.cuda.synchronize()
    return round(reps * 8 * n / (a.elapsed_time(b) * 1e-3) / 1e9)
res = {}
for cols in (2048, 4096):
    for S in (1, cols // 128):
        for chunk in (128, 256):
            for pad in (14, 12):
                res[f"c{cols}_S{S}_chunk{chunk}_pad{pad}k"] = timeit(lambda k: L.wc_segments(out.data_ptr(), n, S, chunk, pad * 1024, k, st.cuda_stream, cols))
print(json.dumps(res))
