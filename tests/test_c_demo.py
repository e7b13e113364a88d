"""The boundary from plain C: examples/prngd_demo.c is compiled with gcc against include/prngd.h
and linked to libprngd_b200.so (no Python in the caller).  On CPU it exercises the host-side
validation (EINVAL cases, constants, plan); on a B200 its prngd_generate_host output is hashed
and compared with the oracle's outputs for the same parameters."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1401_8230_b200")


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    if not os.path.exists(os.path.join(LIBDIR, "libprngd_b200.so")):
        pytest.skip("libprngd_b200.so not built (python -m paper_1401_8230_b200.build)")
    exe = str(tmp_path_factory.mktemp("cdemo") / "prngd_demo")
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror",
                           "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "prngd_demo.c"),
                           "-L", LIBDIR, "-lprngd_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe])
    return exe


def test_c_caller_host_validation(demo):
    r = subprocess.run([demo, "--validate"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "validate ok" in r.stdout and r.stdout.count("PRNGD_EINVAL") == 4
    # cfg1's constants (hand-derived pins in test_oracle_pins): C = b/2^w, D = a - a0 - b/2^w
    assert "C = 0.99999999976716936 D = 4294967294" in r.stdout


def _fnv1a(a: np.ndarray) -> int:
    h = 0xcbf29ce484222325
    for byte in a.astype("<f8").tobytes():
        h = ((h ^ byte) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


@pytest.mark.gpu
@pytest.mark.parametrize("par", [
    dict(w=32, a0=0, a=2**32 - 1, b=2**32 - 1, seed=1, n_streams=64, n_per_stream=1024),
    dict(w=8, a0=0, a=255, b=255, seed=1, n_streams=48, n_per_stream=1030),
    dict(w=32, a0=1, a=2**32 - 1, b=2**31 - 1, seed=7, n_streams=300, n_per_stream=37),
])
def test_c_caller_generate_host_matches_oracle(demo, par):
    import oracle
    oracle.build()
    args = [str(par[k]) for k in ("w", "a0", "a", "b", "seed", "n_streams", "n_per_stream")]
    r = subprocess.run([demo, *args], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    fields = r.stdout.split()
    got_hash = int(fields[fields.index("fnv1a") + 1], 16)
    p = dict(par, b0=0, stream_begin=0)
    ref = oracle.generate(p)["out"].ravel()
    assert got_hash == _fnv1a(ref), r.stdout
    first = [float(x) for x in fields[fields.index("first") + 1:fields.index("first") + 4]]
    assert first == [float(ref[0]), float(ref[1]), float(ref[2])]
