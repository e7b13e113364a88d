"""Randomised parity sweep: 64 seeded random parameter sets -- draw widths, accept bands (down to
the single-value band a - a0 = 2), x2 widths, Eq.(4)/(5)/(6), the open interval, Alg. 1
consumption, every store path, ragged shapes, stream offsets near 2^64 -- each through the C ABI
and compared bitwise with the oracle (and, for a third of them, the fused histogram / moments).
The generator of cases holds no method arithmetic (workloads-style parameter drawing only)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1401_8230_b200 import prngd as P  # noqa: E402

pytestmark = pytest.mark.gpu

STORES = ["auto", "row", "seg", "segc", "tma", "tile", "direct", "row1k"]
AVAILABLE = P.stores_available(STORES)


def _case(i):
    rng = np.random.default_rng(1000 + i)
    w = int(rng.integers(1, 33))
    wb = int(rng.integers(1, w + 1))               # x2 width <= w (b < 2^w, R5)
    b = (1 << wb) - 1
    wa = int(rng.integers(2 if w > 1 else 2, 33))  # bitlen(a) >= 2 so a - a0 >= 2 is possible
    top = (1 << wa) - 1
    a = int(rng.integers(max(2, 1 << (wa - 1)), top + 1))
    # accept band of at least 1/64 of the draw range (bounded rejection), or the minimum band
    if rng.random() < 0.15 and wa <= 8:
        a0 = a - 2                                 # single accepted x1 value (>= 1/256 accepted)
    else:
        lo = max(0, a - 1 - int(rng.integers(max(2, (1 << wa) // 64), (1 << wa) + 1)))
        a0 = int(rng.integers(lo, a - 1)) if a - 1 > lo else max(0, a - 2)
    p = dict(w=w, a0=a0, a=a, b0=0, b=b, seed=int(rng.integers(0, 2**63)),
             stream_begin=int(rng.choice([0, 12345, 2**62 + 7, 2**64 - 5000])),
             n_streams=int(rng.integers(1, 260)), n_per_stream=int(rng.integers(1, 700)))
    kind = 4
    if rng.random() < 0.25:
        kind = 5
    elif rng.random() < 0.2 and a0 == 0 and a == (1 << w) - 1 and b == a:
        kind = 6
    open_ = bool(rng.random() < 0.2)
    alg1 = bool(rng.random() < 0.2)
    store = STORES[int(rng.integers(0, len(STORES)))]
    if store not in AVAILABLE:  # an A/B path of the variant build: the library's AUTO choice
        store = "auto"
    flags = P.STORE_FLAGS[store] | P.MAP_FLAGS[kind] | (P.PRNGD_FLAG_OPEN if open_ else 0) | \
        (P.PRNGD_FLAG_ALG1 if alg1 else 0)
    return p, flags, kind, open_, alg1, bool(rng.random() < 0.35)


@pytest.mark.parametrize("i", range(64))
def test_random_parameter_sets_bitwise(orc, i):
    p, flags, kind, open_, alg1, consume = _case(i)
    if p["stream_begin"] + p["n_streams"] > 2**64:
        p["stream_begin"] = 2**64 - p["n_streams"]
    q = dict(p, flags=flags)
    g = P.Generator(**q)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    if consume:
        _, hist, pw, cnt = g.generate_consume(out)
    else:
        g.generate(out)
    torch.cuda.synchronize()
    ref = orc.generate(p, kind=kind, open_interval=open_, alg1=alg1, want_stats=consume)
    got = out.cpu().numpy().view(np.int64).ravel()
    exp = ref["out"].view(np.int64).ravel()
    bad = np.nonzero(got != exp)[0]
    assert bad.size == 0, f"case {i} {q}: {bad.size} mismatches, first {bad[:5]}"
    if consume:
        assert np.array_equal(hist.cpu().numpy(), ref["hist"]), f"case {i}: histogram"
        assert cnt.item() == ref["count"]
        assert np.allclose(pw.cpu().numpy(), ref["pow"], rtol=1e-12, atol=0)


def _mrg_case(i):
    rng = np.random.default_rng(5000 + i)
    w = int(rng.integers(1, 33))
    wb = int(rng.integers(1, min(w, 31) + 1))
    b = (1 << wb) - 1
    wa = int(rng.integers(2, 32))
    a = int(rng.integers(max(2, 1 << (wa - 1)), (1 << wa)))
    lo = max(0, a - 1 - int(rng.integers(max(2, (1 << wa) // 64), (1 << wa) + 1)))
    a0 = int(rng.integers(lo, a - 1)) if a - 1 > lo else max(0, a - 2)
    kind = 5 if rng.random() < 0.3 else 4
    p = dict(w=w, a0=a0, a=a, b0=0, b=b, seed=int(rng.integers(0, 2**63)), stream_begin=int(i * 977),
             n_streams=int(rng.integers(1, 200)), n_per_stream=2 * int(rng.integers(1, 300)),
             mrg=True)
    alg1 = bool(rng.random() < 0.35)  # Alg. 1 consumption on MRG32k3a
    p["alg1"] = alg1
    return p, P.PRNGD_FLAG_MRG32K3A | P.MAP_FLAGS[kind] | (P.PRNGD_FLAG_ALG1 if alg1 else 0), kind


@pytest.mark.parametrize("i", range(24))
def test_random_parameter_sets_mrg32k3a_bitwise(orc, i):
    p, flags, kind = _mrg_case(i)
    g = P.Generator(**dict(p, flags=flags))
    out = g.generate()
    torch.cuda.synchronize()
    ref = orc.generate(p, kind=kind)["out"]
    got = out.cpu().numpy().view(np.int64).ravel()
    bad = np.nonzero(got != ref.view(np.int64).ravel())[0]
    assert bad.size == 0, f"case {i} {p}: {bad.size} mismatches, first {bad[:5]}"
