"""Host logic of dist.McStats (NEXT-4 setup) on CPU with world-size-2 gloo groups: every failure
mode of the multicast setup must raise on EVERY rank (no rank left waiting in a collective) and
release what was created; the success path must hand out the addresses and destroy on close.
The driver calls (paper_1401_8230_b200.prngd.prngd_mc_*) are replaced by recording fakes."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, scenario, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1401_8230_b200 import dist as D
        from paper_1401_8230_b200 import prngd as P
        log = []

        def fail_if(step):
            if scenario == (step, rank):
                raise P.PrngdError(2, f"simulated {step} failure")

        def supported():
            log.append("supported")
            return scenario != ("supported", rank)

        def create(nbytes, n):
            log.append(("create", n))
            fail_if("create")
            return 1000 + rank, 7

        def imp(pid, fd, nbytes):
            log.append(("import", fd))
            fail_if("import")
            return 2000 + rank

        def add(m):
            log.append(("add", m))
            fail_if("add")

        def bind(m):
            log.append(("bind", m))
            fail_if("bind")
            return 1 << 40, 1 << 41

        def destroy(m):
            log.append(("destroy", m))

        P.prngd_mc_supported, P.prngd_mc_create, P.prngd_mc_import = supported, create, imp
        P.prngd_mc_add_device, P.prngd_mc_bind_map, P.prngd_mc_destroy = add, bind, destroy
        P.prngd_mc_bytes = lambda m: 4 << 20
        try:
            ms = D.McStats()
            res = ("ok", ms.mc, ms.local, ms.arrive - ms.local, ms.expected(3))
            ms.close()
        except RuntimeError as e:
            res = ("raised", str(e))
        dist.barrier()  # every rank got here: nobody is stuck in a collective
        q.put((rank, res, log))
    finally:
        dist.destroy_process_group()


def _run(scenario, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, scenario, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict((r, (res, log)) for r, res, log in (q.get(timeout=120) for _ in range(world)))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_success_path_hands_out_addresses_and_destroys():
    out = _run(None)
    for r in (0, 1):
        res, log = out[r]
        assert res[0] == "ok" and res[1] == 1 << 40 and res[2] == 1 << 41
        assert res[3] == 65541 * 8 and res[4] == 6
        assert log[-1] == ("destroy", 1000 if r == 0 else 2001)
    assert ("create", 2) in out[0][1] and not any(e[0] == "create" for e in out[1][1] if isinstance(e, tuple))
    assert ("import", 7) in out[1][1]


@pytest.mark.parametrize("scenario", [("supported", 1), ("create", 0), ("import", 1),
                                      ("add", 0), ("bind", 1)])
def test_every_failure_raises_on_every_rank(scenario):
    out = _run(scenario)
    step, bad = scenario
    for r in (0, 1):
        res, log = out[r]
        assert res[0] == "raised", (r, res)
        made = [e for e in log if isinstance(e, tuple) and e[0] in ("create", "import")]
        destroyed = [e for e in log if isinstance(e, tuple) and e[0] == "destroy"]
        if step in ("import", "add", "bind"):
            # whatever a rank created or imported it released again
            ok_made = [e for e in made if not (step == "import" and r == bad and e[0] == "import")]
            assert len(destroyed) == len(ok_made), (r, log)
