"""Multi-GPU sharding of the PRNGD path.

Streams are independent and counter-addressed (R6), so the path shards by disjoint
stream-id ranges with NO communication on the generation path: rank r of R generates global
streams [stream_begin_r, stream_begin_r + n_r) into its own HBM; its outputs are the contiguous
slice [stream_begin_r * n_per_stream, ...) of the logical global array.  The only exchange is
the all-reduce of the fused consumer's statistics (65536-bin int64 histogram, 4 FP64 power sums,
int64 count).  Two ways:

* PeerStats (default for the fused consumer): rank 0's accumulator is mapped into every rank with
  CUDA IPC (peer memory over NVLink); each rank's prngd_generate_consume adds its partial sums into
  it with device atomics inside its own finalize kernel -- the collective is fused into the
  library's kernels, no separate launch (NEXT-4 over peer memory; NVLS multicast is unavailable
  in this environment).
* allreduce_stats: torch.distributed all-reduce after the kernel (NCCL over NVLink on B200, gloo
  in the CPU tests) -- the baseline and the fallback.
"""
from __future__ import annotations

from typing import Callable

WEAK, STRONG = "weak", "strong"


def shard_range(n_global: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of rank r's streams when N global streams are split over R ranks."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world {world}")
    return rank * n_global // world, (rank + 1) * n_global // world


def shard_params(p: dict, rank: int, world: int, mode: str = STRONG) -> dict:
    """Parameters of rank r's shard.

    STRONG: p["n_streams"] is the global stream count, split over the ranks.
    WEAK:   p["n_streams"] is the per-rank count; rank r starts at stream_begin + r * n_streams.
    """
    q = dict(p)
    base = p.get("stream_begin", 0)
    if mode == STRONG:
        lo, hi = shard_range(p["n_streams"], rank, world)
        q["stream_begin"], q["n_streams"] = base + lo, hi - lo
    elif mode == WEAK:
        q["stream_begin"] = base + rank * p["n_streams"]
    else:
        raise ValueError(mode)
    return q


def allreduce_stats(hist, pw, count, group=None, deterministic: bool = False):
    """Sum the consumer statistics over ranks, in place.  hist and count are int64 (exact in
    any order); the FP64 power sums are order-dependent, so `deterministic=True` all-gathers the
    per-rank partials and adds them in rank order (bit-identical for any NCCL algorithm)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return hist, pw, count
    with _nvtx("prngd_allreduce_stats"):
        dist.all_reduce(hist, group=group)
        dist.all_reduce(count, group=group)
        if deterministic:
            parts = [torch.empty_like(pw) for _ in range(dist.get_world_size(group))]
            dist.all_gather(parts, pw, group=group)
            acc = torch.zeros_like(pw)
            for t in parts:
                acc += t
            pw.copy_(acc)
        else:
            dist.all_reduce(pw, group=group)
    return hist, pw, count


def _nvtx(name: str):
    """An NVTX range on CUDA builds (for nsys), else nothing."""
    import contextlib

    import torch
    if torch.cuda.is_available():
        return torch.cuda.nvtx.range(name)
    return contextlib.nullcontext()


class PeerStats:
    """Rank `owner`'s statistics accumulator (65536 int64 bins, 1 int64 count, 4 FP64 power
    sums, 1 uint64 arrival counter) mapped into every rank of `group` through CUDA IPC, so
    prngd_generate_consume_ex on any rank adds into it directly (system-scope atomics in the
    library's finalize kernel) and then bumps the arrival counter with a system-scope release.

    Completion protocol: after n calls in total (all ranks), the counter reads n.  The owner
    enqueues ps.wait(n) (a device-side acquire wait, for ranks on DIFFERENT GPUs) before reading
    on the same stream, and sees every add of those n calls.  Ranks sharing one GPU (the one-GPU
    tests) synchronise on the host instead (cuda sync + barrier), which needs no device wait.

    Usage: ps = PeerStats(group); ps.zero(); barrier; every rank: ps.consume(h, out, stream);
    owner: ps.wait(ps.expected(calls_per_rank)); ps.read().  Needs peer access between the
    ranks' GPUs (NVLink / NVSwitch) or ranks on one GPU; raises otherwise (callers fall back to
    allreduce_stats)."""

    NBINS = 65536
    NBYTES = (65536 + 1 + 4 + 1) * 8

    def __init__(self, group=None, owner: int = 0):
        import torch.distributed as dist
        from . import prngd as P
        self.P = P
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.owner = owner
        self.base = None
        err = None
        handle = None
        if self.rank == owner:
            try:
                self.base = P.prngd_peer_alloc(self.NBYTES)
                handle = P.prngd_ipc_export(self.base)
            except Exception as e:  # reported to every rank below
                err = str(e)
        objs = [(handle, err)]
        if dist.is_initialized():
            dist.broadcast_object_list(objs, src=owner, group=group)
        handle, err = objs[0]
        if err is not None:
            raise RuntimeError(f"peer accumulator unavailable: {err}")
        if self.rank != owner:
            self.base = P.prngd_ipc_open(handle)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.hist = self.base
        self.count = self.base + self.NBINS * 8
        self.pow = self.base + (self.NBINS + 1) * 8
        self.arrive = self.base + (self.NBINS + 5) * 8

    def zero(self, stream=None, counter: bool = True):
        """Owner only: zero the statistics (and the arrival counter unless counter=False),
        stream-ordered."""
        if self.rank == self.owner:
            n = self.NBYTES if counter else self.NBYTES - 8
            self.P.prngd_zero(self.base, n, stream)

    def consume(self, handle: int, out, stream=None):
        """This rank's prngd_generate_consume_ex into the shared accumulator (+1 arrival)."""
        self.P.prngd_generate_consume_ex(handle, out, self.hist, self.pow, self.count,
                                         self.arrive, stream)

    def expected(self, calls_per_rank: int) -> int:
        """Arrival count once every rank has made `calls_per_rank` calls."""
        return self.world * calls_per_rank

    def wait(self, target: int, stream=None, timeout_ns: int = 0):
        """Owner: enqueue a device-side wait until the arrival counter reaches `target`
        (system-scope acquire); work enqueued after it on `stream` sees those calls' adds."""
        self.P.prngd_wait_arrivals(self.arrive, target, timeout_ns, stream)

    def arrivals(self) -> int:
        """Current value of the arrival counter (synchronous read)."""
        import torch
        buf = torch.empty(1, dtype=torch.int64, device="cuda")
        self.P.prngd_copy(buf, self.arrive, 8, None)
        torch.cuda.current_stream().synchronize()
        return int(buf.item())

    def read(self):
        """Owner only: (hist int64[65536], pow float64[4], count int64[1]) torch copies."""
        import torch
        buf = torch.empty(self.NBYTES // 8, dtype=torch.int64, device="cuda")
        self.P.prngd_copy(buf, self.base, self.NBYTES, None)
        torch.cuda.current_stream().synchronize()
        return (buf[:self.NBINS], buf[self.NBINS + 1:self.NBINS + 5].view(torch.float64),
                buf[self.NBINS:self.NBINS + 1])

    def close(self):
        if self.base is None:
            return
        if self.rank == self.owner:
            self.P.prngd_peer_free(self.base)
        else:
            self.P.prngd_ipc_close(self.base)
        self.base = None


def _agree(ok: bool, group=None) -> bool:
    """True iff `ok` on every rank of `group` (all-reduce MIN of a flag)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return ok
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return bool(t.item())


class McStats:
    """NEXT-4: the statistics buffer as an NVLS multicast object spanning the ranks' GPUs (one
    process per GPU).  prngd_generate_consume_mc on any rank adds its statistics with
    multimem.red through the multicast address, so the NVSwitch reduces them into EVERY rank's
    local copy (an all-reduce inside the finalize kernel) and bumps every copy's arrival counter
    with a release.  After R ranks x n calls each rank's wait(R*n) + read() returns the global
    statistics.  Raises RuntimeError on every rank (consistently) when the driver / fabric cannot
    create the object (one-GPU leases, no NVSwitch); callers fall back to PeerStats / NCCL."""

    def __init__(self, group=None, owner: int = 0):
        import os

        import torch.distributed as dist
        from . import prngd as P
        self.P, self.group, self.owner = P, group, owner
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.m = None
        err = None
        try:
            if not P.prngd_mc_supported():
                raise RuntimeError("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0")
        except Exception as e:
            err = str(e)
        if not _agree(err is None, group):
            raise RuntimeError(f"multicast unavailable: {err or 'on another rank'}")
        info = [None]
        if self.rank == owner:
            try:
                self.m, fd = P.prngd_mc_create(P.STATS_BYTES, self.world)
                info = [(os.getpid(), fd, P.prngd_mc_bytes(self.m), None)]
            except Exception as e:
                info = [(None, None, None, str(e))]
        if dist.is_initialized():
            dist.broadcast_object_list(info, src=owner, group=group)
        pid, fd, nbytes, err = info[0]
        if err is not None:
            raise RuntimeError(f"multicast object unavailable: {err}")
        err = None
        try:
            if self.rank != owner:
                self.m = P.prngd_mc_import(pid, fd, nbytes)
            P.prngd_mc_add_device(self.m)
        except Exception as e:
            err = str(e)
        if not _agree(err is None, group):
            self.close(barrier=False)
            raise RuntimeError(f"multicast setup failed: {err or 'on another rank'}")
        try:  # every device is in the team before any rank binds memory
            self.mc, self.local = P.prngd_mc_bind_map(self.m)
        except Exception as e:
            err = str(e)
        if not _agree(err is None, group):
            self.close(barrier=False)
            raise RuntimeError(f"multicast bind failed: {err or 'on another rank'}")
        self.hist = self.local
        self.count = self.local + P.STATS_COUNT_OFFSET
        self.pow = self.local + P.STATS_POW_OFFSET
        self.arrive = self.local + P.STATS_ARRIVE_OFFSET

    def consume(self, handle: int, out, stream=None):
        """This rank's prngd_generate_consume_mc (in-switch reduction into every copy)."""
        self.P.prngd_generate_consume_mc(handle, out, self.mc, stream)

    def expected(self, calls_per_rank: int) -> int:
        return self.world * calls_per_rank

    def wait(self, target: int, stream=None, timeout_ns: int = 0):
        """Device-side acquire wait on this rank's local arrival counter."""
        self.P.prngd_wait_arrivals(self.arrive, target, timeout_ns, stream)

    def arrivals(self) -> int:
        """Current value of this rank's local arrival counter (synchronous read)."""
        import torch
        buf = torch.empty(1, dtype=torch.int64, device="cuda")
        self.P.prngd_copy(buf, self.arrive, 8, None)
        torch.cuda.current_stream().synchronize()
        return int(buf.item())

    def zero(self, stream=None, counter: bool = True):
        """Zero THIS rank's local copy (every rank zeroes its own, then a barrier)."""
        n = self.P.STATS_BYTES if counter else self.P.STATS_ARRIVE_OFFSET
        self.P.prngd_zero(self.local, n, stream)

    def read(self):
        import torch
        buf = torch.empty(self.P.STATS_BYTES // 8, dtype=torch.int64, device="cuda")
        self.P.prngd_copy(buf, self.local, self.P.STATS_BYTES, None)
        torch.cuda.current_stream().synchronize()
        n = 65536
        return buf[:n], buf[n + 1:n + 5].view(torch.float64), buf[n:n + 1]

    def close(self, barrier: bool = True):
        import torch.distributed as dist
        if self.m is None:
            return
        if barrier and dist.is_initialized():
            dist.barrier(group=self.group)
        self.P.prngd_mc_destroy(self.m)
        self.m = None


def verify_reduction(ps, group=None, device_wait: bool = True,
                     timeout_s: float = 20.0) -> tuple[bool, str]:
    """Self-check of a shared statistics buffer (PeerStats or McStats) before it is trusted: every
    rank reduces a small known workload through it and the result is compared, bin for bin, with
    the NCCL all-reduce of the same workload's local statistics.  Returns (ok on every rank,
    detail); leaves the buffer zeroed.  device_wait=False synchronises every rank on the host
    (ranks sharing one GPU); otherwise the reader polls the arrival counter until it reaches the
    ranks' count, for at most timeout_s (a buffer whose arrivals never land fails the check)."""
    import time

    import torch
    import torch.distributed as dist
    from . import prngd as P
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    st = torch.cuda.current_stream()
    p = dict(w=32, a0=0, a=2**32 - 1, b0=0, b=2**32 - 1, seed=0x5EED, stream_begin=64 * rank,
             n_streams=64, n_per_stream=256)
    g = P.Generator(**p)
    try:
        _, h, pw, c = g.generate_consume(None)
        allreduce_stats(h, pw, c, group=group)
        ps.zero(st)
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier(group=group)
        ps.consume(g.handle, None, st)
        reader = isinstance(ps, McStats) or rank == getattr(ps, "owner", 0)
        if not device_wait:
            torch.cuda.synchronize()
            if dist.is_initialized():
                dist.barrier(group=group)
        ok, detail = True, "ok"
        if reader:
            if device_wait:
                # poll the arrival counter from the host with a deadline instead of the device
                # wait (whose timeout traps and would leave this process unable to fall back)
                deadline = time.monotonic() + timeout_s
                while ps.arrivals() < ps.expected(1):
                    if time.monotonic() > deadline:
                        ok, detail = False, (f"arrival counter below {ps.expected(1)} after "
                                             f"{timeout_s:g} s")
                        break
                    time.sleep(0.001)
            if ok:
                gh, gp, gc = ps.read()
                if int(gc.item()) != int(c.item()) or not torch.equal(gh, h):
                    ok, detail = False, (f"count {int(gc.item())} vs {int(c.item())} or "
                                         "histogram differs")
                elif not torch.allclose(gp, pw, rtol=1e-12, atol=0):
                    ok, detail = False, "power sums differ"
        torch.cuda.synchronize()
        ok = _agree(ok, group)
        ps.zero(st)
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier(group=group)
        return ok, detail if ok else (detail if detail != "ok" else "failed on another rank")
    finally:
        g.close()


def generate_sharded(p: dict, mode: str = STRONG, consume: bool = False, write: bool = True,
                     group=None, deterministic: bool = False,
                     local: Callable | None = None):
    """Run this rank's shard and (if `consume`) all-reduce the statistics.

    Returns (local_outputs_or_None, hist, pw, count, shard_params).  `local` replaces the
    per-rank generator (the CPU tests pass the oracle; the product path is the CUDA library)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    q = shard_params(p, rank, world, mode)
    if local is not None:
        out, hist, pw, count = local(q, consume, write)
    else:
        from . import prngd as P
        g = P.Generator(**q)
        out = torch.empty(g.shape, dtype=torch.float64, device="cuda") if write else None
        if consume:
            out, hist, pw, count = g.generate_consume(out)
        else:
            g.generate(out)
            hist = pw = count = None
    if consume:
        allreduce_stats(hist, pw, count, group=group, deterministic=deterministic)
    return out, hist, pw, count, q
