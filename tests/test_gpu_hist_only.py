"""Histogram-only fused consumer (d_pow = NULL in the C ABI; include/prngd.h prngd_generate_consume):
BASELINE cfg4's "fused 2^16-bin histogram".  The full-batch paths skip the power sums; histogram,
count and outputs stay bit-identical to the oracle on every consumer layout (row segments, ROW
tiles, statistics only, the generic rejection-heavy path, MRG32k3a, exact-from-the-start carries),
and a later call with a power-sum accumulator on the same handle is unaffected."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1401_8230_b200 import prngd as P  # noqa: E402
from paper_1401_8230_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu


def _bits(t):
    return t.cpu().numpy().view(np.int64)


CASES = [
    ("full32-seg", dict(W.FULL32, n_streams=1000, n_per_stream=1024), 0),
    ("full32-row", dict(W.FULL32, n_streams=517, n_per_stream=2048), P.PRNGD_FLAG_STORE_ROW),
    ("asym-seg", dict(W.ASYM, n_streams=97, n_per_stream=4096), P.PRNGD_FLAG_STORE_SEG),
    ("w17-rejections", dict(w=17, a0=0, a=2**17 - 1, b0=0, b=2**17 - 1, n_streams=300,
                            n_per_stream=1024), 0),
    ("byte8-generic", dict(W.BYTE8, n_streams=200, n_per_stream=333), 0),
    ("ragged", dict(W.FULL32, n_streams=70, n_per_stream=129), 0),
    ("exact-hist", dict(W.FULL32, n_streams=256, n_per_stream=512), P.PRNGD_FLAG_EXACT_HIST),
    ("mrg32k3a", dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1, n_streams=257,
                      n_per_stream=300, mrg=True), P.PRNGD_FLAG_MRG32K3A),
]


@pytest.mark.parametrize("write", [True, False])
@pytest.mark.parametrize("name,par,flags", CASES, ids=[c[0] for c in CASES])
def test_hist_only_matches_oracle(orc, name, par, flags, write):
    p = dict(par, seed=5, stream_begin=4242, flags=flags)
    ref = orc.generate(p, want_out=write, want_stats=True)
    g = P.Generator(**p)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda") if write else None
    _, hist, pw, cnt = g.generate_consume(out, moments=False)
    torch.cuda.synchronize()
    assert pw is None
    assert cnt.item() == ref["count"]
    assert np.array_equal(hist.cpu().numpy(), ref["hist"])
    if write:
        assert np.array_equal(_bits(out), ref["out"].view(np.int64))
    # the same handle, now with power sums: nothing of the histogram-only call sticks
    _, hist2, pw2, cnt2 = g.generate_consume(None)
    torch.cuda.synchronize()
    assert cnt2.item() == ref["count"] and np.array_equal(hist2.cpu().numpy(), ref["hist"])
    assert np.allclose(pw2.cpu().numpy(), ref["pow"], rtol=1e-12, atol=0)


def test_hist_only_accumulates_and_raw_abi(orc):
    """Two histogram-only calls through the C-ABI names add into the same accumulators."""
    p = dict(W.FULL32, seed=9, stream_begin=0, n_streams=128, n_per_stream=1024)
    ref = orc.generate(p, want_out=False, want_stats=True)
    g = P.Generator(**p)
    hist = torch.zeros(65536, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        P.prngd_generate_consume(g.handle, None, hist, None, cnt)
    torch.cuda.synchronize()
    assert cnt.item() == 2 * ref["count"]
    assert np.array_equal(hist.cpu().numpy(), 2 * ref["hist"])
