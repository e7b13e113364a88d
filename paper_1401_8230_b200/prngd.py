"""Thin ctypes binding of libprngd_b200.so (include/prngd.h).

Argument marshalling only: every step of the PRNGD path runs in the library's sm_100a kernels.
Functions carry the C names; ``Generator`` is a convenience wrapper over them.  There is no CPU
fallback: if the library is missing this module raises on import of the library.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# PRNGD_LIB: load an alternative build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("PRNGD_LIB") or os.path.join(PKG, "libprngd_b200.so")

PRNGD_OK, PRNGD_EINVAL, PRNGD_ECUDA, PRNGD_ENOMEM, PRNGD_EUNSUPPORTED = range(5)
PRNGD_FLAG_IEEE_DIV = 0x1
PRNGD_FLAG_ALG1 = 0x4
PRNGD_FLAG_STORE_AUTO = 0 << 3
PRNGD_FLAG_STORE_ROW = 5 << 3
PRNGD_FLAG_STORE_SEG = 6 << 3
PRNGD_FLAG_STORE_SEGC = 7 << 3
PRNGD_FLAG_STORE_TMA = 1 << 3
PRNGD_FLAG_STORE_TILE = 2 << 3
PRNGD_FLAG_STORE_DIRECT = 3 << 3
PRNGD_FLAG_STORE_ROW1K = 4 << 3
PRNGD_FLAG_MAP_EQ4 = 0 << 6
PRNGD_FLAG_MAP_EQ5 = 1 << 6
PRNGD_FLAG_MAP_EQ6 = 2 << 6
PRNGD_FLAG_OPEN = 0x100
PRNGD_FLAG_JUMP = 0x200
PRNGD_FLAG_MRG32K3A = 0x800
PRNGD_FLAG_EXACT_HIST = 0x1000
PRNGD_FLAG_NO_JUMP = 0x400
MAP_FLAGS = {4: PRNGD_FLAG_MAP_EQ4, 5: PRNGD_FLAG_MAP_EQ5, 6: PRNGD_FLAG_MAP_EQ6}
STORE_FLAGS = {"auto": PRNGD_FLAG_STORE_AUTO, "seg": PRNGD_FLAG_STORE_SEG,
               "segc": PRNGD_FLAG_STORE_SEGC,
               "row": PRNGD_FLAG_STORE_ROW, "tma": PRNGD_FLAG_STORE_TMA,
               "tile": PRNGD_FLAG_STORE_TILE, "direct": PRNGD_FLAG_STORE_DIRECT,
               "row1k": PRNGD_FLAG_STORE_ROW1K}

# A/B store paths present only in the variant build (-DPRNGD_AB_STORES=1, include/prngd.h)
AB_STORES = ("tma", "tile", "direct", "row1k", "segc")
_store_ok: dict[str, bool] = {}


def store_supported(name: str) -> bool:
    """Whether the loaded library implements store path `name` (host-only probe)."""
    if name not in _store_ok:
        p = prngd_params(w=32, flags=STORE_FLAGS[name], a0=0, a=2**32 - 1, b0=0, b=2**32 - 1,
                         seed=1, stream_begin=0, n_streams=1, n_per_stream=1)
        h = C.c_void_p()
        st = lib().prngd_create(C.byref(p), C.byref(h))
        if st == PRNGD_OK:
            lib().prngd_destroy(h)
        _store_ok[name] = st == PRNGD_OK
    return _store_ok[name]


def stores_available(names) -> list:
    """The subset of store-path names the loaded library implements (test parametrisation;
    the product set if the library cannot be loaded here)."""
    try:
        return [n for n in names if store_supported(n)]
    except Exception:
        return [n for n in names if n not in AB_STORES]


EXPORTS = (
    "prngd_create", "prngd_destroy", "prngd_get_info", "prngd_generate", "prngd_generate_consume",
    "prngd_generate_host", "prngd_last_launches", "prngd_status_string", "prngd_last_error",
    "prngd_abi_version", "prngd_debug_raw", "prngd_debug_pairs", "prngd_debug_map",
    "prngd_debug_div_check", "prngd_debug_jump",
    "prngd_peer_alloc", "prngd_peer_free", "prngd_ipc_export", "prngd_ipc_open",
    "prngd_ipc_close", "prngd_copy", "prngd_zero", "prngd_generate_consume_ex",
    "prngd_wait_arrivals", "prngd_generate_consume_mc", "prngd_mc_supported", "prngd_mc_create",
    "prngd_mc_import", "prngd_mc_bytes", "prngd_mc_add_device", "prngd_mc_bind_map",
    "prngd_mc_destroy",
)


class prngd_params(C.Structure):
    _fields_ = [("w", C.c_uint32), ("flags", C.c_uint32), ("a0", C.c_uint64), ("a", C.c_uint64),
                ("b0", C.c_uint64), ("b", C.c_uint64), ("seed", C.c_uint64),
                ("stream_begin", C.c_uint64), ("n_streams", C.c_uint64),
                ("n_per_stream", C.c_uint64)]


class prngd_info(C.Structure):
    _fields_ = [("C", C.c_double), ("D", C.c_double), ("C_s", C.c_double), ("D_s", C.c_double),
                ("y", C.c_double), ("sh1", C.c_uint32), ("sh2", C.c_uint32),
                ("clamp", C.c_uint32), ("speculative", C.c_uint32), ("n_outputs", C.c_uint64),
                ("out_bytes", C.c_uint64), ("kernel", C.c_uint32), ("store", C.c_uint32)]


class PrngdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} [status {status}]")
        self.status = status


_lib = None


def lib():
    """Load the native library (build it first with paper_1401_8230_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1401_8230_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, u64, u32, st = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
        sig = {
            "prngd_create": (st, [C.POINTER(prngd_params), C.POINTER(vp)]),
            "prngd_destroy": (st, [vp]),
            "prngd_get_info": (st, [vp, C.POINTER(prngd_info)]),
            "prngd_generate": (st, [vp, vp, vp]),
            "prngd_generate_consume": (st, [vp, vp, vp, vp, vp, vp]),
            "prngd_generate_consume_ex": (st, [vp, vp, vp, vp, vp, vp, vp]),
            "prngd_wait_arrivals": (st, [vp, u64, u64, vp]),
            "prngd_generate_consume_mc": (st, [vp, vp, vp, vp]),
            "prngd_mc_supported": (st, [C.POINTER(C.c_int)]),
            "prngd_mc_create": (st, [u64, u32, C.POINTER(vp), C.POINTER(C.c_int)]),
            "prngd_mc_import": (st, [C.c_int, C.c_int, u64, C.POINTER(vp)]),
            "prngd_mc_bytes": (u64, [vp]),
            "prngd_mc_add_device": (st, [vp]),
            "prngd_mc_bind_map": (st, [vp, C.POINTER(vp), C.POINTER(vp)]),
            "prngd_mc_destroy": (st, [vp]),
            "prngd_generate_host": (st, [vp, vp, vp]),
            "prngd_last_launches": (u32, [vp]),
            "prngd_status_string": (C.c_char_p, [st]),
            "prngd_last_error": (C.c_char_p, []),
            "prngd_abi_version": (C.c_int, []),
            "prngd_debug_raw": (st, [vp, vp, u64, vp]),
            "prngd_debug_pairs": (st, [vp, vp, vp, vp]),
            "prngd_debug_map": (st, [vp, vp, vp, vp, u64, vp]),
            "prngd_debug_div_check": (st, [vp, u64, u64, vp, vp]),
            "prngd_debug_jump": (st, [u64, vp, vp, C.c_int]),
            "prngd_peer_alloc": (st, [u64, C.POINTER(vp)]),
            "prngd_peer_free": (st, [vp]),
            "prngd_ipc_export": (st, [vp, vp]),
            "prngd_ipc_open": (st, [vp, C.POINTER(vp)]),
            "prngd_ipc_close": (st, [vp]),
            "prngd_copy": (st, [vp, vp, u64, vp]),
            "prngd_zero": (st, [vp, u64, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != PRNGD_OK:
        detail = lib().prngd_last_error().decode(errors="replace")
        name = lib().prngd_status_string(status).decode()
        raise PrngdError(status, f"{what}: {name}: {detail}")


def _ptr(t):
    """Device/host pointer of a torch tensor or numpy array (None -> NULL, int -> itself)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def _check_buf(t, name: str, dtype: str, numel: int, device: str):
    """Guard the raw pointer handed to the library: a torch tensor / numpy array must have the
    dtype the C ABI expects, be contiguous, live on the right device and hold >= numel elements
    (the kernels write that many).  Raw integer pointers (peer-mapped buffers) pass unchecked."""
    if t is None or isinstance(t, int):
        return
    if hasattr(t, "data_ptr"):  # torch
        import torch
        want = {"f64": torch.float64, "i64": torch.int64, "i32": (torch.int32,),
                "u32": (torch.int32,)}[dtype]
        ok_dtype = t.dtype in want if isinstance(want, tuple) else t.dtype == want
        if not ok_dtype:
            raise ValueError(f"{name}: dtype {t.dtype}, the C ABI expects {dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name}: must be contiguous")
        if device == "cuda":
            if not t.is_cuda:
                raise ValueError(f"{name}: must be CUDA device memory, got {t.device}")
            if t.device.index != torch.cuda.current_device():
                raise ValueError(f"{name}: on {t.device}, not the current device "
                                 f"cuda:{torch.cuda.current_device()}")
        elif t.is_cuda:
            raise ValueError(f"{name}: must be host memory, got {t.device}")
        n = t.numel()
    else:  # numpy (host only)
        if device == "cuda":
            raise ValueError(f"{name}: a numpy array is host memory; the call needs device memory")
        want = {"f64": "float64", "i64": "int64", "i32": "int32", "u32": "uint32"}[dtype]
        if t.dtype.name not in (want, "int32" if dtype == "u32" else want):
            raise ValueError(f"{name}: dtype {t.dtype}, the C ABI expects {dtype}")
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name}: must be C-contiguous")
        n = t.size
    if n < numel:
        raise ValueError(f"{name}: {n} elements, the call writes {numel}")


_n_outputs: dict[int, int] = {}


def _params_of(h: int) -> tuple[int, int]:
    """(n_outputs, 0) of a handle, cached (the handle is immutable)."""
    n = _n_outputs.get(h)
    if n is None:
        n = _n_outputs[h] = prngd_get_info(h)["n_outputs"]
    return n, 0


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------------- C-named entry points

def prngd_create(**kw) -> int:
    p = prngd_params(**{k: int(v) for k, v in kw.items() if k in dict(prngd_params._fields_)})
    h = C.c_void_p()
    _check(lib().prngd_create(C.byref(p), C.byref(h)), "prngd_create")
    return h.value


def prngd_destroy(h: int):
    _n_outputs.pop(h, None)
    _check(lib().prngd_destroy(h), "prngd_destroy")


def prngd_get_info(h: int) -> dict:
    i = prngd_info()
    _check(lib().prngd_get_info(h, C.byref(i)), "prngd_get_info")
    return {k: getattr(i, k) for k, _ in prngd_info._fields_}


def _check_stats(hist, pw, count, arrive=None):
    _check_buf(hist, "hist", "i64", 65536, "cuda")
    _check_buf(pw, "pw", "f64", 4, "cuda")
    _check_buf(count, "count", "i64", 1, "cuda")
    _check_buf(arrive, "arrive", "i64", 1, "cuda")


def prngd_generate(h: int, out, stream=None):
    _check_buf(out, "out", "f64", _params_of(h)[0], "cuda")
    _check(lib().prngd_generate(h, _ptr(out), _stream_ptr(stream)), "prngd_generate")


def prngd_generate_consume(h: int, out, hist, pw, count, stream=None):
    _check_buf(out, "out", "f64", _params_of(h)[0], "cuda")
    _check_stats(hist, pw, count)
    _check(lib().prngd_generate_consume(h, _ptr(out), _ptr(hist), _ptr(pw), _ptr(count),
                                        _stream_ptr(stream)), "prngd_generate_consume")


def prngd_generate_consume_ex(h: int, out, hist, pw, count, arrive, stream=None):
    _check_buf(out, "out", "f64", _params_of(h)[0], "cuda")
    _check_stats(hist, pw, count, arrive)
    _check(lib().prngd_generate_consume_ex(h, _ptr(out), _ptr(hist), _ptr(pw), _ptr(count),
                                           _ptr(arrive), _stream_ptr(stream)),
           "prngd_generate_consume_ex")


def prngd_wait_arrivals(arrive, target: int, timeout_ns: int = 0, stream=None):
    _check_buf(arrive, "arrive", "i64", 1, "cuda")
    _check(lib().prngd_wait_arrivals(_ptr(arrive), target, timeout_ns, _stream_ptr(stream)),
           "prngd_wait_arrivals")


def prngd_generate_host(h: int, host_out, stream=None):
    _check_buf(host_out, "host_out", "f64", _params_of(h)[0], "cpu")
    _check(lib().prngd_generate_host(h, _ptr(host_out), _stream_ptr(stream)),
           "prngd_generate_host")


def prngd_last_launches(h: int) -> int:
    return int(lib().prngd_last_launches(h))


def prngd_debug_raw(h: int, raw, draws_per_stream: int, stream=None):
    _check(lib().prngd_debug_raw(h, _ptr(raw), draws_per_stream, _stream_ptr(stream)),
           "prngd_debug_raw")


def prngd_debug_pairs(h: int, pair_index, consumed, stream=None):
    _check(lib().prngd_debug_pairs(h, _ptr(pair_index), _ptr(consumed), _stream_ptr(stream)),
           "prngd_debug_pairs")


def prngd_debug_map(h: int, x1, x2, z, stream=None):
    n = z.numel() if hasattr(z, "numel") else z.size
    _check(lib().prngd_debug_map(h, _ptr(x1), _ptr(x2), _ptr(z), n, _stream_ptr(stream)),
           "prngd_debug_map")


def prngd_debug_div_check(h: int, n: int, seed: int, mismatch, stream=None):
    _check(lib().prngd_debug_div_check(h, n, seed, _ptr(mismatch), _stream_ptr(stream)),
           "prngd_debug_div_check")


def prngd_generate_consume_mc(h: int, out, mc_stats: int, stream=None):
    _check_buf(out, "out", "f64", _params_of(h)[0], "cuda")
    _check(lib().prngd_generate_consume_mc(h, _ptr(out), mc_stats, _stream_ptr(stream)),
           "prngd_generate_consume_mc")


# statistics buffer layout (include/prngd.h PRNGD_STATS_*)
STATS_COUNT_OFFSET, STATS_POW_OFFSET, STATS_ARRIVE_OFFSET = 65536 * 8, 65537 * 8, 65541 * 8
STATS_BYTES = 65542 * 8


def prngd_mc_supported() -> bool:
    v = C.c_int(0)
    _check(lib().prngd_mc_supported(C.byref(v)), "prngd_mc_supported")
    return bool(v.value)


def prngd_mc_create(nbytes: int, n_devices: int) -> tuple[int, int]:
    """Owner: (handle, exported POSIX fd) of a new multicast object."""
    m, fd = C.c_void_p(), C.c_int(-1)
    _check(lib().prngd_mc_create(nbytes, n_devices, C.byref(m), C.byref(fd)), "prngd_mc_create")
    return m.value, fd.value


def prngd_mc_import(owner_pid: int, owner_fd: int, nbytes: int) -> int:
    m = C.c_void_p()
    _check(lib().prngd_mc_import(owner_pid, owner_fd, nbytes, C.byref(m)), "prngd_mc_import")
    return m.value


def prngd_mc_bytes(m: int) -> int:
    return int(lib().prngd_mc_bytes(m))


def prngd_mc_add_device(m: int):
    _check(lib().prngd_mc_add_device(m), "prngd_mc_add_device")


def prngd_mc_bind_map(m: int) -> tuple[int, int]:
    """(multicast address, local copy address) of this rank's bound buffer (zeroed)."""
    mc, local = C.c_void_p(), C.c_void_p()
    _check(lib().prngd_mc_bind_map(m, C.byref(mc), C.byref(local)), "prngd_mc_bind_map")
    return mc.value, local.value


def prngd_mc_destroy(m: int):
    _check(lib().prngd_mc_destroy(m), "prngd_mc_destroy")


IPC_HANDLE_BYTES = 64


def prngd_peer_alloc(nbytes: int) -> int:
    """Zeroed device allocation of the current device (raw pointer) for peer sharing."""
    p = C.c_void_p()
    _check(lib().prngd_peer_alloc(nbytes, C.byref(p)), "prngd_peer_alloc")
    return p.value


def prngd_peer_free(ptr: int):
    _check(lib().prngd_peer_free(ptr), "prngd_peer_free")


def prngd_ipc_export(ptr: int) -> bytes:
    buf = C.create_string_buffer(IPC_HANDLE_BYTES)
    _check(lib().prngd_ipc_export(ptr, buf), "prngd_ipc_export")
    return buf.raw


def prngd_ipc_open(handle: bytes) -> int:
    buf = C.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES)
    p = C.c_void_p()
    _check(lib().prngd_ipc_open(buf, C.byref(p)), "prngd_ipc_open")
    return p.value


def prngd_ipc_close(ptr: int):
    _check(lib().prngd_ipc_close(ptr), "prngd_ipc_close")


def prngd_copy(dst, src, nbytes: int, stream=None):
    _check(lib().prngd_copy(_ptr(dst), _ptr(src), nbytes, _stream_ptr(stream)), "prngd_copy")


def prngd_zero(ptr, nbytes: int, stream=None):
    _check(lib().prngd_zero(_ptr(ptr), nbytes, _stream_ptr(stream)), "prngd_zero")


def prngd_debug_jump(n_draws: int, state, lane_table: int = -1):
    import numpy as np
    a = np.ascontiguousarray(state, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    _check(lib().prngd_debug_jump(n_draws, a.ctypes.data, o.ctypes.data, lane_table),
           "prngd_debug_jump")
    return tuple(int(v) for v in o)


# ---------------------------------------------------------------- convenience wrapper

class Generator:
    """PRNGD(k = 2^-w, [a0;a], [b0;b]) over streams [stream_begin, stream_begin + n_streams)."""

    def __init__(self, w, a0, a, b0, b, seed, n_streams, n_per_stream, stream_begin=0, flags=0,
                 **_ignored):
        self.params = dict(w=w, a0=a0, a=a, b0=b0, b=b, seed=seed, n_streams=n_streams,
                           n_per_stream=n_per_stream, stream_begin=stream_begin, flags=flags)
        self.handle = prngd_create(**self.params)
        self.info = prngd_get_info(self.handle)

    @classmethod
    def from_params(cls, p: dict, **over):
        q = dict(p)
        q.update(over)
        return cls(**q)

    @property
    def shape(self):
        return (self.params["n_streams"], self.params["n_per_stream"])

    def generate(self, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty(self.shape, dtype=torch.float64, device="cuda")
        prngd_generate(self.handle, out, stream)
        return out

    def generate_consume(self, out=None, hist=None, pw=None, count=None, stream=None,
                         moments=True):
        """moments=False: histogram-only call (d_pow = NULL in the C ABI); pw is returned as None."""
        import torch
        dev = "cuda"
        hist = torch.zeros(65536, dtype=torch.int64, device=dev) if hist is None else hist
        if moments:
            pw = torch.zeros(4, dtype=torch.float64, device=dev) if pw is None else pw
        else:
            pw = None
        count = torch.zeros(1, dtype=torch.int64, device=dev) if count is None else count
        prngd_generate_consume(self.handle, out, hist, pw, count, stream)
        return out, hist, pw, count

    def generate_host(self, host_out=None, stream=None):
        import torch
        if host_out is None:
            host_out = torch.empty(self.shape, dtype=torch.float64, pin_memory=True)
        prngd_generate_host(self.handle, host_out, stream)
        return host_out

    def raw(self, draws_per_stream, stream=None):
        import torch
        r = torch.empty((self.params["n_streams"], draws_per_stream), dtype=torch.int32,
                        device="cuda")
        prngd_debug_raw(self.handle, r, draws_per_stream, stream)
        return r

    def pairs(self, stream=None):
        import torch
        pidx = torch.empty(self.shape, dtype=torch.int32, device="cuda")
        cons = torch.empty(self.params["n_streams"], dtype=torch.int64, device="cuda")
        prngd_debug_pairs(self.handle, pidx, cons, stream)
        return pidx, cons

    def map(self, x1, x2, stream=None):
        import torch
        z = torch.empty(x1.shape, dtype=torch.float64, device="cuda")
        prngd_debug_map(self.handle, x1, x2, z, stream)
        return z

    @property
    def last_launches(self) -> int:
        return prngd_last_launches(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            prngd_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
