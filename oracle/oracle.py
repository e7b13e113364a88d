"""ctypes marshalling for ``liboracle_prngd.so`` (TEST INFRASTRUCTURE ONLY, see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "prngd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_prngd.so")
_CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]

__all__ = [
    "build", "lib", "mix64", "splitmix64_output", "xs128_sequence", "stream_state", "constants",
    "map_pairs", "map_pairs_noclamp", "accept", "generate", "raw", "enumerate_pairs",
    "map_eq5", "map_eq6", "map_kind", "mrg_sequence", "mrg_stream_state", "mrg_reduced",
    "generate_chunk", "GAMMA",
]

GAMMA = 0x9E3779B97F4A7C15
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no GPU involved).  Returns the .so path."""
    stale = (not os.path.exists(_LIB)) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "prngd_oracle.h")))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        u32, u64, i32, dbl = C.c_uint32, C.c_uint64, C.c_int, C.c_double
        vp = C.c_void_p
        L.oracle_mix64.restype = u64
        L.oracle_mix64.argtypes = [u64]
        L.oracle_splitmix64_output.restype = u64
        L.oracle_splitmix64_output.argtypes = [u64, u64]
        L.oracle_xs128_next.restype = u32
        L.oracle_xs128_next.argtypes = [vp]
        L.oracle_stream_state.restype = None
        L.oracle_stream_state.argtypes = [u64, u64, vp]
        L.oracle_constants.restype = i32
        L.oracle_constants.argtypes = [u32, u64, u64, u64, u64, vp, vp]
        for f in (L.oracle_map, L.oracle_map_noclamp, L.oracle_map_eq5):
            f.restype = dbl
            f.argtypes = [u32, u64, u64, u64, u64, u32, u32]
        L.oracle_map_array.restype = None
        L.oracle_map_array.argtypes = [u32, u64, u64, u64, u64, vp, vp, u64, i32, vp]
        L.oracle_map_eq6.restype = dbl
        L.oracle_map_eq6.argtypes = [u32, u32, u32]
        L.oracle_accept.restype = i32
        L.oracle_accept.argtypes = [u64, u64, u32]
        L.oracle_generate.restype = i32
        L.oracle_generate.argtypes = [u32, u64, u64, u64, u64, u64, u64, u64, u64,
                                      vp, vp, vp, vp, vp, vp]
        L.oracle_generate_ex.restype = i32
        L.oracle_generate_ex.argtypes = [u32, u64, u64, u64, u64, u64, u64, u64, u64, i32, i32, i32,
                                         vp, vp, vp, vp, vp, vp]
        L.oracle_generate_gen.restype = i32
        L.oracle_generate_gen.argtypes = [u32, u64, u64, u64, u64, u64, u64, u64, u64, i32, i32,
                                          i32, i32, vp, vp, vp, vp, vp, vp]
        L.oracle_mrg_next.restype = u32
        L.oracle_mrg_next.argtypes = [vp]
        L.oracle_mrg_stream_state.restype = None
        L.oracle_mrg_stream_state.argtypes = [u64, u64, vp]
        L.oracle_mrg_reduced.restype = u32
        L.oracle_mrg_reduced.argtypes = [vp, i32, vp]
        L.oracle_map_kind.restype = dbl
        L.oracle_map_kind.argtypes = [i32, i32, u32, u64, u64, u64, u64, u32, u32]
        L.oracle_raw.restype = None
        L.oracle_raw.argtypes = [u64, u64, u64, u64, vp]
        L.oracle_enumerate.restype = i32
        L.oracle_enumerate.argtypes = [u32, u64, u64, u64, u64, vp, vp]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def mix64(z: int) -> int:
    return lib().oracle_mix64(z)


def splitmix64_output(seed: int, i: int) -> int:
    return lib().oracle_splitmix64_output(seed, i)


def xs128_sequence(state, n: int) -> list[int]:
    st = np.array(state, dtype=np.uint32)
    return [lib().oracle_xs128_next(st.ctypes.data) for _ in range(n)]


def stream_state(seed: int, s: int) -> tuple[int, int, int, int]:
    st = np.zeros(4, dtype=np.uint32)
    lib().oracle_stream_state(seed, s, st.ctypes.data)
    return tuple(int(v) for v in st)


def constants(w, a0, a, b0, b):
    c, d = C.c_double(), C.c_double()
    rc = lib().oracle_constants(w, a0, a, b0, b, C.byref(c), C.byref(d))
    if rc:
        raise ValueError("invalid parameters")
    return c.value, d.value


def map_pairs(p: dict, x1, x2, clamp: bool = True) -> np.ndarray:
    x1 = np.ascontiguousarray(x1, dtype=np.uint32).ravel()
    x2 = np.ascontiguousarray(x2, dtype=np.uint32).ravel()
    if x1.size != x2.size:
        raise ValueError("x1 and x2 sizes differ")
    out = np.empty(x1.size, dtype=np.float64)
    lib().oracle_map_array(p["w"], p["a0"], p["a"], p["b0"], p["b"], x1.ctypes.data,
                           x2.ctypes.data, x1.size, 1 if clamp else 0, out.ctypes.data)
    return out


def map_pairs_noclamp(p: dict, x1, x2) -> np.ndarray:
    return map_pairs(p, x1, x2, clamp=False)


def accept(p: dict, x1: int) -> bool:
    return bool(lib().oracle_accept(p["a0"], p["a"], x1))


def generate(p: dict, stream_begin: int | None = None, n_streams: int | None = None,
             want_out=True, want_pidx=False, want_consumed=False, want_stats=False,
             kind: int | None = None, alg1: bool | None = None, open_interval: bool | None = None
             ) -> dict:
    """Run the whole oracle path on streams [stream_begin, stream_begin+n_streams).
    kind / alg1 / open_interval default to p["map"] (4), p["alg1"], p["open"] (False)."""
    kind = p.get("map", 4) if kind is None else kind
    mrg = bool(p.get("mrg", False))
    alg1 = p.get("alg1", False) if alg1 is None else alg1
    open_interval = p.get("open", False) if open_interval is None else open_interval
    sb = p.get("stream_begin", 0) if stream_begin is None else stream_begin
    ns = p["n_streams"] if n_streams is None else n_streams
    nps = p["n_per_stream"]
    res = {}
    out = np.empty(ns * nps, dtype=np.float64) if want_out else None
    pidx = np.empty(ns * nps, dtype=np.uint32) if want_pidx else None
    cons = np.empty(ns, dtype=np.uint64) if want_consumed else None
    hist = np.zeros(65536, dtype=np.int64) if want_stats else None
    pw = np.zeros(4, dtype=np.float64) if want_stats else None
    cnt = np.zeros(1, dtype=np.int64) if want_stats else None
    rc = lib().oracle_generate_gen(p["w"], p["a0"], p["a"], p["b0"], p["b"], p["seed"], sb, ns,
                                   nps, int(kind), int(bool(alg1)), int(bool(open_interval)),
                                   int(mrg), _ptr(out), _ptr(pidx), _ptr(cons), _ptr(hist),
                                   _ptr(pw), _ptr(cnt))
    if rc:
        raise ValueError("invalid parameters")
    if want_out:
        res["out"] = out.reshape(ns, nps)
    if want_pidx:
        res["pidx"] = pidx.reshape(ns, nps)
    if want_consumed:
        res["consumed"] = cons
    if want_stats:
        res["hist"], res["pow"], res["count"] = hist, pw, int(cnt[0])
    return res


def raw(seed: int, stream_begin: int, n_streams: int, draws: int) -> np.ndarray:
    out = np.empty(n_streams * draws, dtype=np.uint32)
    lib().oracle_raw(seed, stream_begin, n_streams, draws, out.ctypes.data)
    return out.reshape(n_streams, draws)


def enumerate_pairs(p: dict):
    """All pairs of draw values: returns (q, accepted) shaped [2^bitlen(a), 2^bitlen(b)]."""
    n1, n2 = 1 << int(p["a"]).bit_length(), 1 << int(p["b"]).bit_length()
    q = np.empty(n1 * n2, dtype=np.float64)
    acc = np.empty(n1 * n2, dtype=np.uint8)
    rc = lib().oracle_enumerate(p["w"], p["a0"], p["a"], p["b0"], p["b"], q.ctypes.data,
                                acc.ctypes.data)
    if rc:
        raise ValueError("invalid parameters or widths too large")
    return q.reshape(n1, n2), acc.reshape(n1, n2).astype(bool)


def mrg_sequence(state6, n: int) -> list[int]:
    st = np.array(state6, dtype=np.int64)
    return [lib().oracle_mrg_next(st.ctypes.data) for _ in range(n)]


def mrg_stream_state(seed: int, s: int) -> tuple:
    st = np.zeros(6, dtype=np.int64)
    lib().oracle_mrg_stream_state(seed, s, st.ctypes.data)
    return tuple(int(v) for v in st)


def mrg_reduced(state6, width: int, n: int) -> tuple[list[int], int]:
    """n reduced (R23) values from MRG32k3a state `state6` and the draws they consumed."""
    st = np.array(state6, dtype=np.int64)
    d = C.c_uint64(0)
    vals = [lib().oracle_mrg_reduced(st.ctypes.data, width, C.byref(d)) for _ in range(n)]
    return vals, int(d.value)


def map_kind(p: dict, kind: int, x1, x2, open_interval: bool = False) -> np.ndarray:
    x1 = np.asarray(x1, dtype=np.uint32).ravel()
    x2 = np.asarray(x2, dtype=np.uint32).ravel()
    f = lib().oracle_map_kind
    return np.array([f(kind, int(open_interval), p["w"], p["a0"], p["a"], p["b0"], p["b"],
                       int(a), int(b)) for a, b in zip(x1, x2)], dtype=np.float64)


def map_eq5(p: dict, x1: int, x2: int) -> float:
    return lib().oracle_map_eq5(p["w"], p["a0"], p["a"], p["b0"], p["b"], x1, x2)


def map_eq6(w: int, x1: int, x2: int) -> float:
    return lib().oracle_map_eq6(w, x1, x2)


def generate_chunk(args):
    """generate() over one stream chunk, for a multiprocessing pool (picklable by reference):
    args = (p, stream_begin, n_streams, stats) -> (stream_begin, out or None, hist, pow, count)."""
    p, s0, ns, stats = args
    r = generate(p, stream_begin=s0, n_streams=ns, want_out=not stats, want_stats=stats)
    if stats:
        return s0, None, r["hist"], r["pow"], r["count"]
    return s0, r["out"], None, None, None
