"""Multi-rank host logic on CPU: world_size-2 gloo process groups.

The per-rank generator is the CPU oracle here (test infrastructure); what is under test is the
product's sharding (paper_1401_8230_b200.dist) and the statistics all-reduce."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1401_8230_b200 import dist as D
from paper_1401_8230_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_local(q, consume, write):
    import oracle
    r = oracle.generate(q, want_out=write, want_stats=consume)
    out = torch.from_numpy(r["out"]) if write else None
    if not consume:
        return out, None, None, None
    return (out, torch.from_numpy(r["hist"]), torch.from_numpy(r["pow"]),
            torch.tensor([r["count"]], dtype=torch.int64))


def _worker(rank, world, port, p, mode, deterministic, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out, hist, pw, cnt, q = D.generate_sharded(p, mode=mode, consume=True, write=True,
                                                   deterministic=deterministic,
                                                   local=_oracle_local)
        q_out.put((rank, q, out.numpy(), hist.numpy(), pw.numpy(), int(cnt.item())))
    finally:
        dist.destroy_process_group()


def _run(p, mode, world=2, deterministic=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, mode, deterministic, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return res


def test_shard_ranges_partition():
    for n in (1, 7, 1024, 2**23 + 3):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_weak_shards_are_disjoint_consecutive():
    p = W.config("cfg5")
    qs = [D.shard_params(p, r, 8, D.WEAK) for r in range(8)]
    assert [q["stream_begin"] for q in qs] == [r * 2**20 for r in range(8)]
    assert all(q["n_streams"] == 2**20 for q in qs)


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_two_rank_strong_sharding_matches_whole(orc, name):
    p = W.config(name, n_streams=64, n_per_stream=128)
    res = _run(p, D.STRONG)
    whole = orc.generate(p, want_stats=True)
    out = np.concatenate([r[2] for r in res])
    assert np.array_equal(out.view(np.int64), whole["out"].view(np.int64))
    for r in res:   # every rank holds the global statistics after the all-reduce
        assert np.array_equal(r[3], whole["hist"]) and r[5] == whole["count"]
        assert np.allclose(r[4], whole["pow"], rtol=1e-12, atol=0)


def test_two_rank_weak_sharding_and_deterministic_moments(orc):
    p = W.config("cfg5", n_streams=32, n_per_stream=64)
    res = _run(p, D.WEAK, deterministic=True)
    glob = dict(p, n_streams=64)
    whole = orc.generate(glob, want_stats=True)
    assert np.array_equal(np.concatenate([r[2] for r in res]).view(np.int64),
                          whole["out"].view(np.int64))
    assert res[0][1]["stream_begin"] == 0 and res[1][1]["stream_begin"] == 32
    # deterministic mode: rank-ordered sum of the rank partials, identical on both ranks
    assert np.array_equal(res[0][4].view(np.int64), res[1][4].view(np.int64))
    parts = [orc.generate(D.shard_params(p, r, 2, D.WEAK), want_out=False, want_stats=True)["pow"]
             for r in range(2)]
    assert np.array_equal(res[0][4], parts[0] + parts[1])
    assert np.array_equal(res[0][3], whole["hist"])


def test_lost_rank_range_regenerates_identically(orc):
    """Failure recovery: a rank's stream range is a pure function of (params, range), so another
    rank can regenerate it bit for bit."""
    p = W.config("cfg1", n_streams=16, n_per_stream=64)
    q1 = D.shard_params(p, 1, 2, D.STRONG)
    a = orc.generate(q1)["out"]
    b = orc.generate(dict(q1))["out"]
    assert np.array_equal(a, b)
    whole = orc.generate(p)["out"]
    assert np.array_equal(whole[q1["stream_begin"]:q1["stream_begin"] + q1["n_streams"]], a)
