"""Full-size parity at BASELINE.json's sizes, in the launch configuration bench.py times.

Every output of cfg3 (2^30) and cfg4 (2^32), and the cfg5 per-GPU histogram / count (2^31
outputs), against the CPU oracle run in parallel worker processes over stream ranges (the oracle
itself is unchanged and single-threaded; the pool only splits the streams)."""
import multiprocessing as mp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1401_8230_b200 import prngd as P  # noqa: E402
from paper_1401_8230_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu

CHUNK = 8192  # streams per oracle task


def _oracle_chunk(args):
    import oracle
    p, s0, ns, stats = args
    r = oracle.generate(p, stream_begin=s0, n_streams=ns, want_out=not stats, want_stats=stats)
    if stats:
        return s0, None, r["hist"], r["pow"], r["count"]
    return s0, r["out"], None, None, None


def _pool():
    n = max(1, min(32, len(os.sched_getaffinity(0))))
    return mp.get_context("fork").Pool(n)


def _chunks(p, stats):
    sb, ns = p["stream_begin"], p["n_streams"]
    return [(p, sb + s, min(CHUNK, ns - s), stats) for s in range(0, ns, CHUNK)]


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_every_output_bitwise(orc, name):
    p = W.CONFIGS[name]
    g = P.Generator(**p)
    out = g.generate()
    torch.cuda.synchronize()
    assert g.last_launches == 1
    bad = 0
    with _pool() as pool:
        for s0, ref, *_ in pool.imap_unordered(_oracle_chunk, _chunks(p, False)):
            r0 = s0 - p["stream_begin"]
            gpu = out[r0:r0 + ref.shape[0]].cpu().numpy()
            bad += int(np.count_nonzero(gpu.view(np.int64) != ref.view(np.int64)))
    assert bad == 0
    del out
    torch.cuda.empty_cache()


def test_cfg5_shard_statistics(orc):
    """cfg5 rank-3 shard (streams [3*2^20, 4*2^20)), fused write + histogram + moments."""
    p = dict(W.CONFIGS["cfg5"], stream_begin=3 * 2**20)
    g = P.Generator(**p)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    _, hist, pw, cnt = g.generate_consume(out)
    torch.cuda.synchronize()
    h = np.zeros(65536, dtype=np.int64)
    s = np.zeros(4)
    c = 0
    with _pool() as pool:
        for _, _, hh, pp, cc in pool.imap_unordered(_oracle_chunk, _chunks(p, True)):
            h += hh
            s += pp
            c += cc
    assert np.array_equal(hist.cpu().numpy(), h) and cnt.item() == c == 2**31
    assert np.allclose(pw.cpu().numpy(), s, rtol=1e-12, atol=0)
    del out
    torch.cuda.empty_cache()
