"""Sustained store bandwidth vs number of SMs issuing stores (tools/probe/sm_count_stores.cu)."""
import ctypes, json, os, statistics, subprocess, threading, time
import torch
import pynvml
here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "libsmstores.so")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                       "-shared", "-Xcompiler", "-fPIC", "-o", so, os.path.join(here, "sm_count_stores.cu")])
L = ctypes.CDLL(so)
L.sm_stores.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p]
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
n = 1 << 30
out = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
def run(S, reps):
    for k in range(3): L.sm_stores(out.data_ptr(), n, S, k, st.cuda_stream)
    torch.cuda.synchronize()
    clk, pw, stop = [], [], threading.Event()
    def sample():
        while not stop.is_set():
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)); pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000); time.sleep(0.005)
    t = threading.Thread(target=sample); t.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(reps): L.sm_stores(out.data_ptr(), n, S, 10 + k, st.cuda_stream)
    b.record(); torch.cuda.synchronize(); stop.set(); t.join()
    return {"GBs": round(reps * 8 * n / (a.elapsed_time(b) * 1e-3) / 1e9), "sm_mhz": statistics.median(clk), "power_w": round(statistics.median(pw))}
res = {}
for S in (148, 128, 111, 96, 74):
    res[S] = {"50": run(S, 50), "600": run(S, 600)}
    print(S, res[S], flush=True)
print(json.dumps(res))
