"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage it follows.  None of them re-types the oracle's own op sequence:
the expected values come from published generator vectors, exact rational arithmetic (Python
integers / fractions), closed forms, counts that follow from the accept-reject rule, or
monotonicity / error-bound arguments written out in DESIGN.md ("Oracle pins").
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_1401_8230_b200 import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def full(w):
    return dict(w=w, a0=0, a=(1 << w) - 1, b0=0, b=(1 << w) - 1)


def exact_eq4(p, x1, x2):
    """Eq.(4) as an exact rational of integer-unit inputs (R1)."""
    k = Fraction(1, 1 << p["w"])
    z = x1 + k * x2
    return (z - (p["a0"] + k * p["b"])) / (p["a"] - p["a0"] - k * (p["b"] - p["b0"]))


# ----------------------------------------------------------------------------- base generators

def test_splitmix64_published_vectors(orc):
    g = _gold("paper_examples.json")["splitmix64_seed0"]
    got = [orc.splitmix64_output(g["seed"], i) for i in range(3)]
    assert got == [int(h, 16) for h in g["outputs_hex"]]


def test_splitmix64_counter_equals_sequential(orc):
    # Counter addressing (R6) must equal the sequential "state += gamma" definition.
    seed, state, mask = 0xDEADBEEF12345678, 0xDEADBEEF12345678, (1 << 64) - 1
    for i in range(50):
        state = (state + orc.GAMMA) & mask
        assert orc.mix64(state) == orc.splitmix64_output(seed, i)


def test_xorshift128_marsaglia_sequence(orc):
    g = _gold("paper_examples.json")["xorshift128_marsaglia"]
    assert orc.xs128_sequence(g["state"], 5) == g["outputs"]


def test_stream_convention_matches_independent_survey_vectors(orc):
    a = _gold("survey_appendix_a.json")
    assert orc.stream_state(1, 0) == tuple(int(h, 16) for h in a["stream0_state"])
    assert orc.stream_state(1, 1) == tuple(int(h, 16) for h in a["stream1_state"])
    r = orc.raw(1, 0, 2, 4)
    assert list(r[0]) == a["stream0_draws"] and list(r[1]) == a["stream1_draws"]


def test_stream_state_never_all_zero(orc):
    # R6: mix64 is a bijection and outputs #2s, #2s+1 differ, so the 128-bit state is nonzero.
    for s in range(2000):
        assert any(orc.stream_state(0, s))


# ----------------------------------------------------------------------------- constants

@pytest.mark.parametrize("key,par", [("w32_constants", W.FULL32), ("cfg4_constants", W.ASYM)])
def test_constants_hand_derived(orc, key, par):
    g = _gold("paper_examples.json")[key]
    C, D = orc.constants(**par)
    assert C == float.fromhex(g["C_hex"]) and D == float.fromhex(g["D_hex"])


@pytest.mark.parametrize("bad", [
    dict(w=0, a0=0, a=1, b0=0, b=0), dict(w=33, a0=0, a=7, b0=0, b=7),
    dict(w=8, a0=0, a=1, b0=0, b=255),          # empty accepted band
    dict(w=8, a0=5, a=4, b0=0, b=255),          # a0 > a
    dict(w=8, a0=0, a=255, b0=1, b=255),        # b0 != 0 (R5)
    dict(w=8, a0=0, a=255, b0=0, b=254),        # x2 does not fill its width (R5)
    dict(w=8, a0=0, a=255, b0=0, b=511),        # k*(b-b0) >= 1
    dict(w=32, a0=0, a=2**32, b0=0, b=255),     # a beyond 32 bits
])
def test_invalid_parameters_rejected(orc, bad):
    with pytest.raises(ValueError):
        orc.constants(**bad)


# ----------------------------------------------------------------------------- Eq.(4) values

def test_paper_worked_examples_w3(orc):
    g = _gold("paper_examples.json")["eq4_w3_examples"]
    for c in g["cases"]:
        q = orc.map_pairs(g["params"], [c["x1"]], [c["x2"]])[0]
        assert q == float(Fraction(c["num"], c["den"]))
        assert exact_eq4(g["params"], c["x1"], c["x2"]) == Fraction(c["num"], c["den"])


@pytest.mark.parametrize("w", [3, 5, 8, 12])
def test_closed_form_exhaustive(orc, w):
    """for w <= 26 on the full range, accepted outputs are exactly
    RN(j / (2^w-1)^2) with j = 2^w x1 + x2 - (2^w-1) -- one correctly-rounded division of two
    integers below 2^53 (numpy's IEEE division is that rounding)."""
    p = full(w)
    q, acc = orc.enumerate_pairs(p)
    n = 1 << w
    x1, x2 = np.meshgrid(np.arange(n, dtype=np.int64), np.arange(n, dtype=np.int64), indexing="ij")
    j = (x1 << w) + x2 - (n - 1)
    M = float((n - 1) ** 2)
    assert np.array_equal(q[acc], j[acc].astype(np.float64) / M)
    # the accepted j cover 1..M-1 exactly once: equally spaced, uniformly weighted (Eq.(3))
    assert np.array_equal(np.sort(j[acc]), np.arange(1, (n - 1) ** 2, dtype=np.int64))


@pytest.mark.parametrize("w", [16, 20, 24, 26])
def test_closed_form_sampled(orc, w):
    p = full(w)
    x1, x2 = W.random_pairs(100 + w, 200_000, w, w)
    e1, e2 = W.edge_pairs(w, w)
    x1, x2 = np.concatenate([x1, e1]), np.concatenate([x2, e2])
    acc = (x1 > 0) & (x1 < (1 << w) - 1)
    x1, x2 = x1[acc].astype(np.int64), x2[acc].astype(np.int64)
    j = (x1 << w) + x2 - ((1 << w) - 1)
    got = orc.map_pairs(p, x1, x2)
    assert np.array_equal(got, j.astype(np.float64) / float(((1 << w) - 1) ** 2))


def test_general_range_exact_rational_w8(orc):
    """w <= 26, any [a0;a], [0;b]: every step of Eq.(4) is exact but the division, so the
    result is RN of the exact rational (2^w(x1-a0) + x2 - b) / (2^w(a-a0) - b)."""
    for (a0, a, b) in [(3, 200, 255), (0, 100, 127), (17, 18 + 2, 15)]:
        p = dict(w=8, a0=a0, a=a, b0=0, b=b)
        q, acc = orc.enumerate_pairs(p)
        for x1 in range(q.shape[0]):
            for x2 in range(0, q.shape[1], 7):
                e = Fraction(256 * (x1 - a0) + x2 - b, 256 * (a - a0) - b)
                if acc[x1, x2]:
                    assert q[x1, x2] == float(e), (p, x1, x2)
                    assert 0 < e < 1


def _ulp(x):
    return np.spacing(np.abs(x))


def test_w32_error_bound(orc):
    """w = 32: Eq.(1) needs 64 bits and is rounded.  DESIGN.md "Oracle pins" derives
    |q - E| <= 2^-53 + 2^-54 + 2^-62 against the exact Eq.(4) value E, and
    |q - E| <= ulp(q)/2 + E*2^-62 when x1 < 2^20 (z and z - C exact)."""
    p = W.FULL32
    x1, x2 = W.random_pairs(7, 4000, 32, 32)
    e1, e2 = W.edge_pairs(32, 32, span=6)
    x1 = np.concatenate([x1, e1, np.arange(1, 2000, dtype=np.uint32)])
    x2 = np.concatenate([x2, e2, np.arange(1, 2000, dtype=np.uint32) * 2147483])
    keep = (x1 > 0) & (x1 < 2**32 - 1)
    x1, x2 = x1[keep], x2[keep]
    q = orc.map_pairs_noclamp(p, x1, x2)
    bound = Fraction(1, 2**53) + Fraction(1, 2**54) + Fraction(1, 2**62)
    for a, b, v in zip(x1.tolist(), x2.tolist(), q.tolist()):
        E = exact_eq4(p, a, b)
        err = abs(Fraction(v) - E)
        assert err <= bound, (a, b)
        if a < 2**20:
            assert err <= Fraction(float(_ulp(v))) / 2 + E / 2**62, (a, b)


def test_cfg4_error_bound_and_extremes(orc):
    p = W.ASYM
    x1, x2 = W.random_pairs(8, 3000, 32, 31)
    keep = (x1 > 1) & (x1 < 2**32 - 1)
    x1, x2 = x1[keep], x2[keep]
    q = orc.map_pairs(p, x1, x2)
    bound = Fraction(1, 2**53) + Fraction(1, 2**54) + Fraction(1, 2**62)
    for a, b, v in zip(x1.tolist(), x2.tolist(), q.tolist()):
        assert abs(Fraction(v) - exact_eq4(p, a, b)) <= bound
    # extremes of the accepted set (x1 in [2, 2^32-2]) stay strictly inside (0, 1)
    lo = orc.map_pairs(p, [2], [0])[0]
    hi = orc.map_pairs(p, [2**32 - 2], [2**31 - 1])[0]
    assert 0.0 < lo < 1e-9 and 1 - 1e-9 < hi < 1.0
    assert abs(Fraction(lo) - exact_eq4(p, 2, 0)) <= bound


def test_map_monotone(orc):
    # Each RN step is monotone non-decreasing, so the literal chain is monotone in z.
    p = W.FULL32
    x1 = np.repeat(np.array([1, 2, 3, 2**31, 2**32 - 3, 2**32 - 2], dtype=np.uint32), 4096)
    x2 = np.tile(np.arange(2**32 - 4096, 2**32, dtype=np.uint64).astype(np.uint32), 6)
    q = orc.map_pairs_noclamp(p, x1, x2)
    assert np.all(np.diff(q) >= 0)


# ----------------------------------------------------------------------------- z' < 1, z' > 0

@pytest.mark.parametrize("w,expected", [(27, 2), (28, 4), (29, 16), (30, 64), (31, 256), (32, 1024)])
def test_literal_one_set_and_clamp(orc, w, expected):
    """DESIGN.md R11: the literal Eq.(4) in RN reaches exactly 1.0 only at x1 = a-1 and the top
    x2 values; by monotonicity the whole set is found in a window at the top of x2."""
    p = full(w)
    top = (1 << w) - 1
    win = 4 * expected + 64
    x2 = np.arange(top - win + 1, top + 1, dtype=np.uint64).astype(np.uint32)
    x1 = np.full(x2.size, top - 1, dtype=np.uint32)
    raw = orc.map_pairs_noclamp(p, x1, x2)
    ones = raw == 1.0
    assert ones.sum() == expected
    assert np.all(ones[-expected:]) and not ones[0]
    # next row down never reaches 1 (monotone in x1, x2): its maximum is < 1
    assert orc.map_pairs_noclamp(p, [top - 2], [top])[0] < 1.0
    clamped = orc.map_pairs(p, x1, x2)
    assert np.all(clamped < 1.0) and clamped.max() == float.fromhex("0x1.fffffffffffffp-1")


@pytest.mark.parametrize("w", [3, 8, 16, 20, 26])
def test_no_one_for_small_w(orc, w):
    p = full(w)
    top = (1 << w) - 1
    assert orc.map_pairs_noclamp(p, [top - 1], [top])[0] < 1.0
    assert orc.map_pairs_noclamp(p, [1], [0])[0] > 0.0


# ----------------------------------------------------------------------------- w = 8 brute force

def test_w8_brute_force(orc):
    """BASELINE north_star: enumerate all 2^16 pairs at w=8."""
    p = W.BYTE8
    g = _gold("paper_examples.json")["eq4_endpoints"]
    q, acc = orc.enumerate_pairs(p)
    # rejection set is exactly x1 in {a0, a}: 2 rows x 256
    assert acc.sum() == 65024 and (~acc).sum() == 512
    assert not acc[0].any() and not acc[255].any() and acc[1:255].all()
    v = np.sort(q[acc])
    assert np.unique(v).size == 65024                      # each lattice point exactly once
    assert v[0] == float.fromhex(g["w8_min_hex"]) and v[-1] == float.fromhex(g["w8_max_hex"])
    assert 0.0 < v[0] and v[-1] < 1.0
    d = np.diff(v)                                         # equally spaced up to rounding
    assert np.all(np.abs(d - 1 / 65025) <= 2 * _ulp(v[1:]))
    # 2^16-bin histogram: bin(j) = floor(65536 j / 65025) (integer arithmetic, R16)
    j = np.arange(1, 65025, dtype=np.int64)
    assert np.array_equal((v * 65536.0).astype(np.int64), (65536 * j) // 65025)
    hist = np.bincount((65536 * j) // 65025, minlength=65536)
    assert (hist == 1).sum() == 65024 and (hist == 0).sum() == 512
    assert hist[0] == 0 and hist[65535] == 0


def test_w8_exact_lattice_moments(orc):
    q, acc = orc.enumerate_pairs(W.BYTE8)
    v = q[acc]
    N, M = 65024, 65025
    for pw in (1, 2, 3, 4):
        exact = Fraction(sum(j**pw for j in range(1, N + 1)), N * M**pw)
        got = float(np.sum(v**pw)) / N
        assert abs(got - float(exact)) <= 1e-12 * float(exact)
    assert Fraction(sum(range(1, N + 1)), N * M) == Fraction(1, 2)   # mean exactly 1/2


# ----------------------------------------------------------------------------- whole path

def test_rejection_rate_cfg2(orc):
    """Per-attempt rejection probability is 2/2^w; empirical within 5 sigma."""
    p = W.config("cfg2", n_streams=256)
    r = orc.generate(p, want_out=False, want_consumed=True)
    att = int(r["consumed"].sum())
    rej = att - 256 * 1024
    pr = 2 / 256
    assert abs(rej / att - pr) < 5 * np.sqrt(pr * (1 - pr) / att)


def test_generate_pair_indices_consistent_with_raw_draws(orc):
    """Output j of a stream is the j-th accepted pair; pair p = draws (2p, 2p+1) (R2)."""
    p = W.config("cfg2", n_streams=8, n_per_stream=300)
    r = orc.generate(p, want_pidx=True, want_consumed=True)
    raw = orc.raw(p["seed"], 0, 8, 2 * int(r["consumed"].max()))
    for s in range(8):
        x1 = raw[s, 0::2] >> 24
        x2 = raw[s, 1::2] >> 24
        accepted = np.nonzero((x1 > 0) & (x1 < 255))[0][:300]
        assert np.array_equal(r["pidx"][s], accepted)
        assert r["consumed"][s] == accepted[-1] + 1
        # outputs are the closed-form lattice values of the accepted pairs (P3)
        j = (x1[accepted].astype(np.int64) << 8) + x2[accepted] - 255
        assert np.array_equal(r["out"][s], j / 65025.0)


def test_shard_invariance(orc):
    p = W.config("cfg1", n_streams=16, n_per_stream=64)
    whole = orc.generate(p)["out"]
    parts = [orc.generate(W.shard(p, r, 4))["out"] for r in range(4)]
    assert np.array_equal(whole, np.concatenate(parts))


def test_determinism_and_seed_dependence(orc):
    p = W.config("cfg1", n_streams=4, n_per_stream=32)
    a, b = orc.generate(p)["out"], orc.generate(p)["out"]
    c = orc.generate(dict(p, seed=W.SEED2))["out"]
    assert np.array_equal(a, b) and not np.array_equal(a, c)


def test_cfg1_cfg2_against_independent_survey_vectors(orc):
    a = _gold("survey_appendix_a.json")
    r = orc.generate(W.config("cfg1"), want_consumed=True, want_stats=True)
    out = r["out"]
    assert [v.hex() for v in out[0, :4]] == a["cfg1_stream0_q"]
    assert [v.hex() for v in out[1023, :4]] == a["cfg1_stream1023_q"]
    assert int(r["consumed"].sum()) - out.size == a["cfg1_rejected_pairs"]
    assert (r["hist"] > 0).sum() == a["cfg1_nonempty_bins"] and r["hist"].max() == a["cfg1_max_bin"]
    assert r["count"] == out.size and np.all(out < 1.0) and np.all(out > 0.0)
    r2 = orc.generate(W.config("cfg2"), want_consumed=True, want_stats=True)
    assert [v.hex() for v in r2["out"][0, :6]] == a["cfg2_stream0_q"]
    assert int(r2["consumed"].sum()) == a["cfg2_attempts"]
    assert int(r2["consumed"].sum()) - r2["out"].size == a["cfg2_rejected_pairs"]
    assert (r2["hist"] > 0).sum() == a["cfg2_nonempty_bins"]


def test_stats_consistent_with_outputs(orc):
    p = W.config("cfg4", n_streams=64, n_per_stream=256)
    r = orc.generate(p, want_stats=True)
    v = r["out"].ravel()
    assert np.array_equal(r["hist"], np.bincount(np.floor(v * 65536).astype(np.int64), minlength=65536))
    for k in range(4):
        assert abs(r["pow"][k] - np.sum(v ** (k + 1))) <= 1e-12 * r["pow"][k]
    assert r["count"] == v.size


# ----------------------------------------------------------------------------- NEXT-1: Eq.(5)/(6)

def test_eq5_paper_endpoints_and_example(orc):
    """Endpoints are exact; interior values carry the literal order's two roundings
    (num/den, then *(1-k')), so they sit within one ulp of the exact rational."""
    g = _gold("paper_examples.json")["eq5_w3_examples"]
    for c in g["cases"]:
        q = orc.map_eq5(g["params"], c["x1"], c["x2"])
        E = Fraction(c["num"], c["den"])
        if c["num"] in (0, c["den"] - 1):
            assert q == float(E)
        assert abs(Fraction(q) - E) <= Fraction(float(np.spacing(float(E))))


@pytest.mark.parametrize("w", [3, 6, 8])
def test_eq5_eq6_exact_rational(orc, w):
    """Eq.(5) on the full range equals J/(2^{2w} - 2^{w+1} - 1) * (1 - k^2), J = 2^w(x1-1) + x2,
    within one rounding of each of its two roundings; Eq.(6) agrees with it."""
    p = full(w)
    n = 1 << w
    Mp = n * n - 2 * n - 1
    kp = Fraction(1, n * n)
    for x1 in range(1, n - 1):
        for x2 in range(n):
            E = Fraction(n * (x1 - 1) + x2, Mp) * (1 - kp)
            q5 = orc.map_eq5(p, x1, x2)
            q6 = orc.map_eq6(w, x1, x2)
            tol = Fraction(float(np.spacing(float(E)))) if E > 0 else Fraction(0)
            assert abs(Fraction(q5) - E) <= tol and abs(Fraction(q6) - E) <= 2 * tol
    assert orc.map_eq5(p, 1, 0) == 0.0
    assert orc.map_eq5(p, n - 2, n - 1) == float(1 - kp)


# ----------------------------------------------------------------------------- NEXT-1/2 whole path

def test_alg1_z_formula_is_eq4():
    """Alg. 1's Z with min/max equals Eq.(4) with a0 = b0 = min, a = b = max (R2 note)."""
    import random
    rnd = random.Random(3)
    for w in (3, 8, 32):
        k = Fraction(1, 2**w)
        mn, mx = 0, 2**w - 1
        p = dict(w=w, a0=mn, a=mx, b0=mn, b=mx)
        for _ in range(200):
            r1, r2 = rnd.randrange(1, mx), rnd.randrange(0, mx + 1)
            z_alg1 = (r1 + k * r2 - (mn + k * mx)) / ((mx - mn) * (1 - k))
            assert z_alg1 == exact_eq4(p, r1, r2)


def test_alg1_consumption_matches_raw_draws(orc):
    """Alg. 1: x1 is redrawn alone until accepted, then one x2 is drawn."""
    p = W.config("cfg2", n_streams=4, n_per_stream=200, alg1=True)
    r = orc.generate(p, want_pidx=True, want_consumed=True)
    raw = orc.raw(p["seed"], 0, 4, int(r["consumed"].max()))
    for s in range(4):
        d, outs, idx = 0, [], []
        while len(outs) < 200:
            x1 = raw[s, d] >> 24
            if 0 < x1 < 255:
                x2 = raw[s, d + 1] >> 24
                outs.append(((int(x1) << 8) + int(x2) - 255) / 65025.0)
                idx.append(d)
                d += 2
            else:
                d += 1
        assert np.array_equal(r["out"][s], np.array(outs)) and list(r["pidx"][s]) == idx
        assert r["consumed"][s] == d


@pytest.mark.parametrize("kind", [5, 6])
def test_eq5_eq6_whole_path_uses_the_mapping(orc, kind):
    p = W.config("cfg2", n_streams=8, n_per_stream=100, map=kind)
    r = orc.generate(p, want_pidx=True)
    raw = orc.raw(p["seed"], 0, 8, 2 * (int(r["pidx"].max()) + 1))
    for s in range(8):
        x1 = raw[s, 2 * r["pidx"][s]] >> 24
        x2 = raw[s, 2 * r["pidx"][s] + 1] >> 24
        assert np.array_equal(r["out"][s], orc.map_kind(p, kind, x1, x2))
    # Eq.(5)/(6) include z' = 0 and stay below 1
    q, acc = orc.enumerate_pairs(W.BYTE8)
    x1, x2 = np.nonzero(acc)
    v = orc.map_kind(W.BYTE8, kind, x1, x2)
    assert v.min() == 0.0 and v.max() < 1.0 and np.unique(v).size == 65024


def test_open_interval_never_zero(orc):
    """1 - z' excludes 0; exact (Sterbenz) for z' >= 1/2."""
    q, acc = orc.enumerate_pairs(W.BYTE8)
    x1, x2 = np.nonzero(acc)
    for kind in (4, 5):
        z = orc.map_kind(W.BYTE8, kind, x1, x2)
        o = orc.map_kind(W.BYTE8, kind, x1, x2, open_interval=True)
        assert o.min() > 0.0 and o.max() <= 1.0
        big = z >= 0.5
        assert np.array_equal(o[big], 1.0 - z[big])
    assert orc.map_kind(W.BYTE8, 5, [1], [0], open_interval=True)[0] == 1.0


def test_eq5_w32_reaches_one_and_is_clamped(orc):
    """At w=32 (1 - k') rounds to 1, so Eq.(5)'s top pair needs the R11 clamp as well."""
    top = 2**32 - 1
    assert orc.map_eq5(W.FULL32, top - 1, top) == 1.0
    assert orc.map_kind(W.FULL32, 5, [top - 1], [top])[0] == float.fromhex("0x1.fffffffffffffp-1")


# ----------------------------------------------------------------------------- NEXT-2 MRG32k3a

M1, M2 = 2**32 - 209, 2**32 - 22853


def test_mrg32k3a_definition_first_outputs(orc):
    """L'Ecuyer (1999) MRG32k3a: x_n = (1403580 x_{n-2} - 810728 x_{n-3}) mod m1,
    y_n = (527612 y_{n-1} - 1370589 y_{n-3}) mod m2, u = (x_n - y_n) mod m1 (0 -> m1).
    From the all-12345 seed the first output is 545508589 (hand-checked: p1 = 592852*12345 mod m1
    = 3023790853, p2 = -842977*12345 mod m2 = 2478282264)."""
    seq = orc.mrg_sequence([12345] * 6, 200)
    assert seq[0] == 3023790853 - 2478282264 == 545508589
    x, y = [12345] * 3, [12345] * 3
    for u in seq:
        x.append((1403580 * x[-2] - 810728 * x[-3]) % M1)
        y.append((527612 * y[-1] - 1370589 * y[-3]) % M2)
        z = (x[-1] - y[-1]) % M1
        assert u == (z if z else M1) and 1 <= u <= M1


def test_mrg_alg1_consumption(orc):
    """Alg. 1 on reduced MRG32k3a values (R23).  Pins: (a) with a band that rejects
    nothing in these streams, Alg. 1 and pair-drop consume the same values in the same order, so
    the outputs coincide; (b) with a narrow band, the Alg. 1 stream is the reduced-value sequence
    cut as 'first in-band value, then the next value', read off the pair-drop-free raw sequence."""
    full = dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1, seed=21, n_streams=16,
                n_per_stream=300, mrg=True)
    pd = orc.generate(full, want_pidx=True)
    assert np.array_equal(pd["pidx"], np.tile(np.arange(300, dtype=np.uint32), (16, 1)))
    a1 = orc.generate(full, alg1=True)
    assert np.array_equal(a1["out"].view(np.int64), pd["out"].view(np.int64))
    # (b): w = 8 draws (x = top... reduced to 8 bits), band a0 < x1 < a with a - a0 = 40
    p = dict(w=8, a0=100, a=140, b0=0, b=255, seed=22, n_streams=1, n_per_stream=200, mrg=True)
    r = orc.generate(p, alg1=True, want_consumed=True)
    st = list(orc.mrg_stream_state(p["seed"], 0))
    m1 = 2**32 - 209
    T = (m1 // 256) * 256
    raw = [u - 1 for u in orc.mrg_sequence(st, int(r["consumed"][0]))]
    vals = [x & 255 for x in raw if x < T]            # R23: reduce to 8 bits by rejection
    x1s, x2s, k = [], [], 0
    while len(x1s) < 200:
        while not (100 < vals[k] < 140):              # Alg. 1: redraw R1 alone
            k += 1
        x1s.append(vals[k])
        x2s.append(vals[k + 1])
        k += 2
    assert k == len(vals)                             # every consumed value was used
    z = orc.map_kind(p, 4, np.array(x1s, np.uint32), np.array(x2s, np.uint32))
    assert np.array_equal(np.asarray(z).view(np.int64), r["out"].ravel().view(np.int64))


def test_mrg_stream_state_golden_vectors(orc):
    """R22 pinned by literal vectors: SplitMix64(seed 1) outputs #3s..#3s+2 split (lo, hi) into
    six words, the first three mod m1, the last three mod m2 (derivation in the golden's cite).
    A swapped word order, an off-by-one output index or a missing reduction fails here."""
    g = _gold("paper_examples.json")["mrg32k3a_stream_state_R22"]
    for s, st in g["streams"].items():
        assert orc.mrg_stream_state(g["seed"], int(s)) == tuple(st), f"stream {s}"
    # the words of streams 0/1 are SURVEY Appendix A's independently computed xorshift states
    a = _gold("survey_appendix_a.json")
    w = [int(h, 16) for h in a["stream0_state"]] + [int(h, 16) for h in a["stream1_state"]]
    assert list(g["streams"]["0"]) == w[:6]
    assert list(g["streams"]["1"])[:2] == w[6:8]


def test_mrg_reduce_to_width_literal_threshold(orc):
    """SPEC S:228-236's literal T = 63 * 2^26 = 4227858432 for w = 26 (R23).  States are hand-cut
    so the first draw is u = p1 exactly: with x-state (0, s1, *) and y-state (0, *, 0) the first
    step gives p1 = 1403580 * s1 mod m1 and p2 = 0, so u = p1.  u - 1 = T must be discarded and
    u - 1 = T - 1 kept as (T - 1) mod 2^26 = 2^26 - 1."""
    T = _gold("paper_examples.json")["mrg32k3a_reduce_to_width_T"]["T"]
    assert T == 4227858432
    inv = pow(1403580, -1, M1)

    def state_for_first_u(u):
        return [0, (u * inv) % M1, 5, 0, 7, 0]

    st = state_for_first_u(T + 1)                   # u - 1 = T: discarded
    assert orc.mrg_sequence(list(st), 1) == [T + 1]
    vals, draws = orc.mrg_reduced(st, 26, 1)
    assert draws >= 2                                # the first draw was skipped
    st = state_for_first_u(T)                        # u - 1 = T - 1: the largest kept value
    vals, draws = orc.mrg_reduced(st, 26, 1)
    assert (vals, draws) == ([2**26 - 1], 1)
    st = state_for_first_u(M1)                       # u = m1 (x = y), u - 1 = m1 - 1 > T
    vals, draws = orc.mrg_reduced(st, 26, 1)
    assert draws >= 2
    # and on a real stream: the discards of a long hand-cut sequence match the literal T
    s0 = list(orc.mrg_stream_state(1, 0))
    raw = orc.mrg_sequence(list(s0), 5000)
    kept = [(u - 1) & (2**26 - 1) for u in raw if u - 1 < T]
    vals, draws = orc.mrg_reduced(s0, 26, len(kept))
    assert draws == 5000 and vals == kept
    assert 5000 - len(kept) > 40                     # ~1/64 of the draws were discarded


def test_mrg_stream_states_in_range(orc):
    for s in range(300):
        st = orc.mrg_stream_state(1, s)
        assert all(0 <= v < M1 for v in st[:3]) and all(0 <= v < M2 for v in st[3:])
        assert any(st[:3]) and any(st[3:])


def test_mrg_reduced_draws_uniform_and_rejection_rate(orc):
    """R23: reduce-to-width keeps exactly T = floor(m1/2^w)*2^w of the m1 values."""
    p = dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1, seed=1, n_streams=64,
             n_per_stream=2000, mrg=True)
    r = orc.generate(p, want_consumed=True, want_pidx=True)
    pairs = int(r["pidx"][:, -1].sum() + 64)
    draws = int(r["consumed"].sum())
    T = (M1 // 2**26) * 2**26
    keep = T / M1
    # each pair needs 2 kept draws: draws ~ 2*pairs/keep
    expected = 2 * pairs / keep
    assert abs(draws - expected) < 6 * np.sqrt(expected * (1 - keep)) + 10
    v = r["out"].ravel()
    assert v.min() > 0 and v.max() < 1
    h = np.histogram(v, bins=64, range=(0, 1))[0]
    e = v.size / 64
    assert ((h - e) ** 2 / e).sum() < 64 + 8 * np.sqrt(2 * 64)   # chi2 sanity, 63 dof
