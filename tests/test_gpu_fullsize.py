"""Full-size parity at BASELINE.json's sizes, in the launch configuration bench.py times.

Every output of cfg3 (2^30) and cfg4 (2^32), the cfg5 per-GPU histogram / count (2^31
outputs), against the CPU oracle run in parallel worker processes over stream ranges (the oracle
itself is unchanged and single-threaded; the pool only splits the streams), and sampled rows of
the NEXT-1 / NEXT-2 bench workloads (eq5, eq6, open4, mrg26) at their full size."""
import multiprocessing as mp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1401_8230_b200 import prngd as P  # noqa: E402
from paper_1401_8230_b200 import workloads as W  # noqa: E402
import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

CHUNK = 8192  # streams per oracle task


def _pool():
    # forkserver: the workers fork from a clean server process (no CUDA context, no threads)
    # and import only the oracle (oracle.generate_chunk is picklable by reference)
    n = max(1, min(32, len(os.sched_getaffinity(0))))
    return mp.get_context("forkserver").Pool(n)


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
        for s0, ref, *_ in pool.imap_unordered(oracle.generate_chunk, _chunks(p, False)):
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
        for _, _, hh, pp, cc in pool.imap_unordered(oracle.generate_chunk, _chunks(p, True)):
            h += hh
            s += pp
            c += cc
    assert np.array_equal(hist.cpu().numpy(), h) and cnt.item() == c == 2**31
    assert np.allclose(pw.cpu().numpy(), s, rtol=1e-12, atol=0)
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["eq5", "eq6", "open4", "mrg26"])
def test_next_workloads_sampled_rows(orc, name):
    """The NEXT-1 / NEXT-2 bench workloads at full size (2^30 outputs, the flags bench.py sets):
    the first and last 64 rows and 4096 seeded random rows, each against the oracle."""
    p = dict(W.CONFIGS[name])
    flags = p.get("map_flags", 0) | (P.PRNGD_FLAG_MRG32K3A if p.get("mrg") else 0)
    g = P.Generator(**dict(p, flags=flags))
    out = g.generate()
    torch.cuda.synchronize()
    assert g.last_launches == 1
    ns = p["n_streams"]
    rng = np.random.default_rng(2024)
    rows = np.unique(np.concatenate([np.arange(64), np.arange(ns - 64, ns),
                                     rng.integers(0, ns, 4096)]))
    got = out[torch.from_numpy(rows).cuda()].cpu().numpy()
    bad = 0
    for i, r in enumerate(rows):
        ref = orc.generate(p, stream_begin=p["stream_begin"] + int(r), n_streams=1)["out"]
        bad += int(np.count_nonzero(got[i].view(np.int64) != ref.view(np.int64)))
    assert bad == 0
    del out
    torch.cuda.empty_cache()
