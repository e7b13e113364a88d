"""The C-ABI library builds, loads and exports every symbol include/prngd.h declares; host-side
validation and constants (no GPU needed: prngd_create and prngd_get_info make no CUDA call)."""
import os
import re
import subprocess

import pytest

from paper_1401_8230_b200 import build as B
from paper_1401_8230_b200 import prngd as P
from paper_1401_8230_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return P.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "prngd.h")).read()
    return sorted(set(re.findall(r"PRNGD_API\s+[\w\s\*]+?\b(prngd_\w+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(P.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (prngd_\w+)", out))
    for name in declared_symbols():
        assert name in exported, name
        assert getattr(lib, name) is not None


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_abi_version(lib):
    assert lib.prngd_abi_version() == 1


@pytest.mark.parametrize("bad,fragment", [
    (dict(W.FULL32, w=0), "w=0"),
    (dict(W.FULL32, w=33), "w=33"),
    (dict(W.FULL32, a=2**32), "32 bits"),
    (dict(W.FULL32, a0=2**32 - 2), "a - a0 >= 2"),
    (dict(W.BYTE8, b0=1), "b0 must be 0"),
    (dict(W.BYTE8, b=254), "power of two"),
    (dict(W.BYTE8, b=511), "b < 2^w"),
])
def test_create_rejects_invalid(lib, bad, fragment):
    with pytest.raises(P.PrngdError) as e:
        P.prngd_create(**bad, seed=1, n_streams=1, n_per_stream=2)
    assert e.value.status == P.PRNGD_EINVAL and fragment in str(e.value)


@pytest.mark.parametrize("counts", [(0, 4), (4, 0), (2**40, 2**30), (1, 2**32)])
def test_create_rejects_bad_counts(lib, counts):
    with pytest.raises(P.PrngdError) as e:
        P.prngd_create(**W.FULL32, seed=1, n_streams=counts[0], n_per_stream=counts[1])
    assert e.value.status == P.PRNGD_EINVAL


def test_create_rejects_unknown_flags(lib):
    with pytest.raises(P.PrngdError) as e:
        P.prngd_create(**W.FULL32, seed=1, n_streams=1, n_per_stream=2, flags=0x10000)
    assert e.value.status == P.PRNGD_EUNSUPPORTED


def test_null_arguments(lib):
    assert lib.prngd_create(None, None) == P.PRNGD_EINVAL
    assert lib.prngd_destroy(None) == P.PRNGD_OK
    assert lib.prngd_generate(None, None, None) == P.PRNGD_EINVAL
    assert b"EINVAL" in lib.prngd_status_string(1)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4"])
def test_constants_match_oracle(lib, orc, name):
    p = W.CONFIGS[name]
    h = P.prngd_create(**p)
    try:
        i = P.prngd_get_info(h)
    finally:
        P.prngd_destroy(h)
    C, D = orc.constants(p["w"], p["a0"], p["a"], p["b0"], p["b"])
    assert (i["C"], i["D"]) == (C, D)
    assert i["C_s"] == C * 2.0 ** p["w"] and i["D_s"] == D * 2.0 ** p["w"]
    assert i["y"] == 1.0 / i["D_s"]
    assert i["sh1"] == 32 - p["a"].bit_length() and i["sh2"] == 32 - p["b"].bit_length()
    assert i["n_outputs"] == p["n_streams"] * p["n_per_stream"]


@pytest.mark.parametrize("w,clamp", [(8, 0), (26, 0), (27, 1), (32, 1)])
def test_clamp_flag_follows_R11(lib, w, clamp):
    h = P.prngd_create(w=w, a0=0, a=2**w - 1, b0=0, b=2**w - 1, seed=1, n_streams=1, n_per_stream=2)
    try:
        assert P.prngd_get_info(h)["clamp"] == clamp
    finally:
        P.prngd_destroy(h)


def test_speculation_only_for_rare_rejection(lib):
    for p, spec in [(W.FULL32, 1), (W.ASYM, 1), (W.BYTE8, 0)]:
        h = P.prngd_create(**p, seed=1, n_streams=1, n_per_stream=2)
        assert P.prngd_get_info(h)["speculative"] == spec
        P.prngd_destroy(h)
    h = P.prngd_create(**W.FULL32, seed=1, n_streams=1, n_per_stream=2, flags=P.PRNGD_FLAG_ALG1)
    assert P.prngd_get_info(h)["speculative"] == 0
    P.prngd_destroy(h)


def test_generate_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = P.prngd_create(**W.CONFIGS["cfg1"])
    try:
        st = lib.prngd_generate(h, 0x1000, None)
        assert st in (P.PRNGD_ECUDA, P.PRNGD_EUNSUPPORTED)
    finally:
        P.prngd_destroy(h)


def test_eq6_requires_unit_interval(lib):
    with pytest.raises(P.PrngdError) as e:
        P.prngd_create(**W.ASYM, seed=1, n_streams=1, n_per_stream=2, flags=P.PRNGD_FLAG_MAP_EQ6)
    assert e.value.status == P.PRNGD_EINVAL
    h = P.prngd_create(**W.FULL32, seed=1, n_streams=1, n_per_stream=2, flags=P.PRNGD_FLAG_MAP_EQ6)
    P.prngd_destroy(h)


@pytest.mark.parametrize("kind,w,clamp", [(5, 8, 0), (5, 32, 1), (6, 8, 0), (6, 32, 1)])
def test_clamp_flag_for_eq5_eq6(lib, orc, kind, w, clamp):
    p = dict(w=w, a0=0, a=2**w - 1, b0=0, b=2**w - 1)
    h = P.prngd_create(**p, seed=1, n_streams=1, n_per_stream=2, flags=P.MAP_FLAGS[kind])
    try:
        assert P.prngd_get_info(h)["clamp"] == clamp
    finally:
        P.prngd_destroy(h)
    top = 2**w - 1
    raw = orc.map_eq5(p, top - 1, top) if kind == 5 else orc.map_eq6(w, top - 1, top)
    assert (raw >= 1.0) == bool(clamp)


def test_jump_ahead_matches_sequential_draws(lib, orc):
    """NEXT-3: T^n (GF(2) matrix power) and the GPU's byte tables reproduce n sequential
    xorshift128 draws of the oracle (Marsaglia recurrence)."""
    for seed, s in [(1, 0), (7, 12345), (W.SEED2, 2**40 + 3)]:
        st = orc.stream_state(seed, s)
        seq = orc.xs128_sequence(st, 64 * 31 + 4)   # outputs = successive w words
        for n in (1, 2, 3, 4, 5, 63, 64, 65, 1000, 64 * 31):
            got = P.prngd_debug_jump(n, st)
            # the state after n draws holds the last four outputs (x, y, z, w)
            assert got == tuple(seq[n - 4:n]) if n >= 4 else got[3] == seq[n - 1]
        # NEXT-3 jump kernel tables: lane l of a round starts at draw 34 l (17 pairs per lane)
        for lane in (0, 1, 2, 17, 31):
            if lane:
                assert P.prngd_debug_jump(0, st, lane) == tuple(seq[34 * lane - 4:34 * lane])
            else:
                assert P.prngd_debug_jump(0, st, 0) == st
        # SEG store path tables: lane j of a row starts at draw 256 j (pair 128 j)
        seq = orc.xs128_sequence(st, 256 * 31)
        for lane in (1, 2, 7, 15, 31):
            assert P.prngd_debug_jump(256, st, lane) == tuple(seq[256 * lane - 4:256 * lane])


def test_jump_flag_rules(lib):
    with pytest.raises(P.PrngdError):
        P.prngd_create(**W.FULL32, seed=1, n_streams=1, n_per_stream=2,
                       flags=P.PRNGD_FLAG_JUMP | P.PRNGD_FLAG_ALG1)


def test_mrg_flag_rules(lib):
    with pytest.raises(P.PrngdError) as e:   # 32-bit draws cannot come from MRG32k3a (R23)
        P.prngd_create(**W.FULL32, seed=1, n_streams=1, n_per_stream=2, flags=P.PRNGD_FLAG_MRG32K3A)
    assert e.value.status == P.PRNGD_EINVAL
    p = dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1)
    with pytest.raises(P.PrngdError):   # no jump-ahead for MRG32k3a
        P.prngd_create(**p, seed=1, n_streams=1, n_per_stream=2,
                       flags=P.PRNGD_FLAG_MRG32K3A | P.PRNGD_FLAG_JUMP)
    h = P.prngd_create(**p, seed=1, n_streams=1, n_per_stream=2,
                       flags=P.PRNGD_FLAG_MRG32K3A | P.PRNGD_FLAG_ALG1)   # Alg. 1 on MRG32k3a
    P.prngd_destroy(h)
    h = P.prngd_create(**p, seed=1, n_streams=1, n_per_stream=2, flags=P.PRNGD_FLAG_MRG32K3A)
    assert P.prngd_get_info(h)["speculative"] == 0
    P.prngd_destroy(h)


@pytest.mark.parametrize("name,flags,kernel,store", [
    ("cfg1", 0, 1, 6),                          # AUTO, few streams, rare rejection: SEG
    ("cfg2", 0, 5, 4),                          # AUTO, few streams, w = 8: NEXT-3 narrow jump kernel
    ("cfg3", 0, 0, 4),                          # AUTO, bulk: ROW
    ("cfg4", 0, 0, 4),
    ("cfg3", P.PRNGD_FLAG_STORE_SEG, 1, 6),     # explicit SEG
    ("cfg2", P.PRNGD_FLAG_STORE_SEG, 0, 4),     # SEG ineligible (w = 8 is not speculative): ROW
    ("cfg1", P.PRNGD_FLAG_STORE_ROW, 0, 4),     # an explicit store path is honoured
    ("cfg1", P.PRNGD_FLAG_JUMP, 2, 4),
])
def test_kernel_selection(lib, name, flags, kernel, store):
    """prngd_get_info reports the kernel and store path prngd_generate launches (host logic)."""
    h = P.prngd_create(**{k: v for k, v in W.config(name, flags=flags).items() if k != "mrg"})
    try:
        info = P.prngd_get_info(h)
        assert (info["kernel"], info["store"]) == (kernel, store)
    finally:
        P.prngd_destroy(h)


@pytest.mark.parametrize("store", ["tma", "tile", "direct", "row1k", "segc"])
def test_ab_store_paths_only_in_variant_build(lib, store):
    """The losing A/B store paths are not in the product library."""
    if P.store_supported(store):
        pytest.skip("variant build (-DPRNGD_AB_STORES=1) loaded")
    with pytest.raises(P.PrngdError) as e:
        P.prngd_create(**W.FULL32, seed=1, n_streams=1, n_per_stream=2, flags=P.STORE_FLAGS[store])
    assert e.value.status == P.PRNGD_EUNSUPPORTED and "variant build" in str(e.value)


def test_accept_band_floor(lib):
    """Bands accepting fewer than 2^-16 of the x1 draw values are refused (include/prngd.h)."""
    top = 2**32 - 1
    ok = P.prngd_create(w=32, a0=top - 2**16 - 1, a=top, b0=0, b=top, seed=1, n_streams=1,
                        n_per_stream=2)            # exactly 2^16 of 2^32 values accepted
    P.prngd_destroy(ok)
    with pytest.raises(P.PrngdError) as e:
        P.prngd_create(w=32, a0=top - 2**16, a=top, b0=0, b=top, seed=1, n_streams=1,
                       n_per_stream=2)
    assert e.value.status == P.PRNGD_EINVAL and "acceptance floor" in str(e.value)
    h = P.prngd_create(w=8, a0=0, a=2, b0=0, b=255, seed=1, n_streams=1, n_per_stream=2)
    P.prngd_destroy(h)                             # tiny ranges: 1 of 4 values, fine


def test_binding_checks_buffers_before_the_call(lib):
    """The binding refuses buffers the kernels would overrun (dtype, size, device, layout)."""
    import numpy as np
    torch = pytest.importorskip("torch")
    h = P.prngd_create(**W.FULL32, seed=1, n_streams=4, n_per_stream=8)
    try:
        with pytest.raises(ValueError, match="CUDA device memory"):
            P.prngd_generate(h, torch.empty(32, dtype=torch.float64))
        with pytest.raises(ValueError, match="dtype"):
            P.prngd_generate_host(h, np.empty(32, dtype=np.float32))
        with pytest.raises(ValueError, match="elements"):
            P.prngd_generate_host(h, np.empty(31, dtype=np.float64))
        with pytest.raises(ValueError, match="contiguous"):
            P.prngd_generate_host(h, torch.empty(64, dtype=torch.float64)[::2])
    finally:
        P.prngd_destroy(h)


def test_stream_id_range_reaches_the_top(lib):
    """Streams [stream_begin, stream_begin + n) may end at id 2^64 - 1, not beyond."""
    h = P.prngd_create(**W.FULL32, seed=1, stream_begin=2**64 - 1000, n_streams=1000,
                       n_per_stream=2)
    P.prngd_destroy(h)
    with pytest.raises(P.PrngdError) as e:
        P.prngd_create(**W.FULL32, seed=1, stream_begin=2**64 - 999, n_streams=1000,
                       n_per_stream=2)
    assert e.value.status == P.PRNGD_EINVAL and "overflows" in str(e.value)
