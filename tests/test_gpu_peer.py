"""Multi-process statistics reduction through peer memory (dist.PeerStats): rank 0's accumulator
is mapped into the other ranks with CUDA IPC and every rank's prngd_generate_consume adds its
shard's histogram / power sums / count into it with device atomics (the collective fused into the
library's finalize kernel).  Run here as 2-3 processes on ONE GPU (IPC works between processes on
one device); the kernels never wait on one another -- the ranks synchronise on the host (gloo
barriers) -- so sharing the GPU is safe.  Compared with the oracle over the whole stream range."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, calls, queue, poll=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1401_8230_b200 import dist as D
        from paper_1401_8230_b200 import prngd as P
        q = D.shard_params(p, rank, world, D.STRONG)
        g = P.Generator(**q)
        ps = D.PeerStats()
        # the bench's self-check of a shared buffer against the all-reduce: host-side completion
        # (the ranks share one GPU), or the reader polling the arrival counter (poll=True, the
        # separate-GPU path; host polling never blocks the other ranks' kernels)
        vok, why = D.verify_reduction(ps, device_wait=poll)
        assert vok, why
        ps.zero()
        torch.cuda.synchronize()
        dist.barrier()
        out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
        for _ in range(calls):  # the accumulator sums over calls as well as ranks
            ps.consume(g.handle, out, torch.cuda.current_stream())
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            # ranks share the GPU: host synchronisation, no device wait (which could starve the
            # other processes' kernels); the arrival counter must read world x calls
            hist, pw, cnt = ps.read()
            queue.put((hist.cpu().numpy(), pw.cpu().numpy(), int(cnt.item()),
                       out[:2].cpu().numpy(), ps.arrivals(), ps.expected(calls)))
        dist.barrier()
        if rank != 0:
            ps.close()
        dist.barrier()
        if rank == 0:
            ps.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,calls,name,poll", [(2, 1, "cfg1", False), (3, 2, "cfg2", False),
                                                   (2, 1, "cfg1", True)])
def test_peer_memory_statistics_reduction(orc, world, calls, name, poll):
    import torch.multiprocessing as mp
    from paper_1401_8230_b200 import workloads as W
    p = W.config(name, n_streams=3000, n_per_stream=520)
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, calls, queue, poll))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = queue.get(timeout=300)
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    hist, pw, cnt, head, arrived, expected = res
    assert arrived == expected == world * calls       # one release per call of every rank
    ref = orc.generate(p, want_stats=True)
    assert cnt == calls * ref["count"]
    assert np.array_equal(hist, calls * ref["hist"])
    assert np.allclose(pw, calls * ref["pow"], rtol=1e-12, atol=0)
    assert np.array_equal(head.view(np.int64), ref["out"][:2].view(np.int64))  # rank 0's rows


def test_multicast_statistics_single_process_or_clean_refusal(orc):
    """NEXT-4 on whatever this box offers: with the NVLS multicast object available even for one
    device, prngd_generate_consume_mc's in-switch reduction (multimem.red in the finalize
    kernel) must equal the oracle's statistics and bump the arrival counter; where the driver
    refuses the object (one-GPU leases), McStats raises RuntimeError naming the driver's reason
    and nothing is left allocated, so dist / bench fall back to peer memory."""
    from paper_1401_8230_b200 import dist as D
    from paper_1401_8230_b200 import prngd as P
    from paper_1401_8230_b200 import workloads as W
    torch.cuda.set_device(0)
    supported = P.prngd_mc_supported()
    try:
        ms = D.McStats()
    except RuntimeError as e:
        msg = str(e)
        assert "multicast" in msg and ("Multicast" in msg or "MULTICAST" in msg or "CUresult" in msg
                                       or "cuMulticast" in msg), msg
        return
    assert supported
    try:
        p = W.config("cfg1", n_streams=640, n_per_stream=520)
        g = P.Generator(**p)
        for _ in range(2):
            ms.consume(g.handle, None)
        ms.wait(2)
        hist, pw, cnt = ms.read()
        ref = orc.generate(p, want_stats=True)
        assert int(cnt.item()) == 2 * ref["count"]
        assert np.array_equal(hist.cpu().numpy(), 2 * ref["hist"])
        assert np.allclose(pw.cpu().numpy(), 2 * ref["pow"], rtol=1e-12, atol=0)
    finally:
        ms.close()


def test_verify_reduction_fails_cleanly_when_arrivals_never_land():
    """A shared buffer whose arrivals never reach the reader must fail the self-check after the
    deadline -- no device-side wait, no trap -- so the caller can still fall back to NCCL."""
    import time
    from paper_1401_8230_b200 import dist as D
    torch.cuda.set_device(0)

    class Lost:  # adds go nowhere; the counter stays 0
        owner = 0

        def zero(self, stream=None, counter=True):
            pass

        def consume(self, handle, out, stream=None):
            pass

        def expected(self, calls):
            return calls

        def arrivals(self):
            return 0

        def read(self):
            raise AssertionError("read before the arrivals landed")

    t0 = time.monotonic()
    ok, why = D.verify_reduction(Lost(), device_wait=True, timeout_s=0.3)
    assert not ok and "arrival counter" in why
    assert time.monotonic() - t0 < 30
    torch.cuda.synchronize()  # the context is still usable

