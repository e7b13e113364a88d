"""Accepted-pair indices of the PRODUCTION kernels, not only of the debug hook (prngd_debug_pairs).

For a full-range width w <= 20 the closed form of Eq.(4) (pinned exhaustively in
tests/test_oracle_pins.py) gives q = RN(j / (2^w - 1)^2) with j = 2^w x1 + x2 - (2^w - 1) taking
each value once, and the doubles are far apart compared with their rounding, so every output
identifies its pair: j = rint(q (2^w - 1)^2), x1 = (j + 2^w - 1) >> w, x2 = (j + 2^w - 1) mod 2^w.
Reading the pair of every output back from what a production kernel wrote, and the raw draw
sequence from prngd_debug_raw (the same __device__ draw code), gives the pair index of each
output; it must be the index of the k-th accepted pair (pair-drop) and equal the
oracle's pair indices bit for bit.  Covered: the ROW kernel (speculative and exact paths), SEG,
the NEXT-3 jump kernel (17- and 33-pair rounds), and the fused consumer's row-segment and
ROW-tile layouts.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1401_8230_b200 import prngd as P  # noqa: E402

pytestmark = pytest.mark.gpu


def _pairs_of_outputs(out, w):
    m = (1 << w) - 1
    j = np.rint(out.astype(np.float64) * float(m * m)).astype(np.int64)
    v = j + m
    return v >> w, v & m


def _check_pair_indices(orc, p, out):
    w = p["w"]
    ns, nps = p["n_streams"], p["n_per_stream"]
    x1o, x2o = _pairs_of_outputs(out.cpu().numpy(), w)
    # pair index of every output = index of the k-th accepted pair of the raw draw sequence
    ref = orc.generate(p, want_out=True, want_pidx=True)
    need = int(ref["pidx"][:, -1].max()) + 1
    g = P.Generator(**p)
    raw = g.raw(2 * need).cpu().numpy().view(np.uint32).astype(np.int64)
    sh = 32 - w
    x1r, x2r = raw[:, 0::2] >> sh, raw[:, 1::2] >> sh
    acc = (x1r > p["a0"]) & (x1r < p["a"])
    for r in range(ns):
        idx = np.nonzero(acc[r])[0][:nps]
        assert idx.size == nps
        # what the production kernel wrote is exactly the accepted pairs, in order ...
        assert np.array_equal(x1o[r], x1r[r, idx]) and np.array_equal(x2o[r], x2r[r, idx]), r
        # ... and their indices are the oracle's
        assert np.array_equal(idx.astype(np.uint32), ref["pidx"][r]), r
    assert np.array_equal(out.cpu().numpy().view(np.int64), ref["out"].view(np.int64))


W17 = dict(w=17, a0=0, a=2**17 - 1, b0=0, b=2**17 - 1)   # rare rejection: speculative kernels
W12 = dict(w=12, a0=0, a=2**12 - 1, b0=0, b=2**12 - 1)   # 1 in 2048 pairs: exact kernels


@pytest.mark.parametrize("par,flags,shape", [
    (W17, P.PRNGD_FLAG_STORE_ROW, (4096, 1024)),   # gen_kernel ROW, speculation + replays
    (W12, P.PRNGD_FLAG_STORE_ROW, (1000, 520)),    # gen_kernel ROW, exact per-pair path
    (W17, P.PRNGD_FLAG_STORE_SEG, (2000, 1024)),   # gen_seg_kernel + seg_exact rewrites
    (W12, P.PRNGD_FLAG_JUMP, (600, 1024)),         # gen_jump_kernel, 33-pair rounds
    (W12, P.PRNGD_FLAG_JUMP, (600, 700)),          # gen_jump_kernel, 17-pair rounds
])
def test_production_kernel_pair_indices(orc, par, flags, shape):
    p = dict(par, seed=2024, stream_begin=99, n_streams=shape[0], n_per_stream=shape[1],
             flags=flags)
    g = P.Generator(**p)
    out = g.generate()
    torch.cuda.synchronize()
    _check_pair_indices(orc, p, out)


@pytest.mark.parametrize("flags", [P.PRNGD_FLAG_STORE_AUTO, P.PRNGD_FLAG_STORE_ROW])
def test_fused_consumer_pair_indices(orc, flags):
    """The outputs the fused consumer writes (row segments by default, ROW tiles when asked)."""
    p = dict(W17, seed=7, stream_begin=5, n_streams=3000, n_per_stream=2048, flags=flags)
    g = P.Generator(**p)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    g.generate_consume(out)
    torch.cuda.synchronize()
    _check_pair_indices(orc, p, out)
