#!/usr/bin/env python
"""Benchmark of the PRNGD hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3|cfg5|cfg4|...]
                    [--impl ours|reference]

A step is one pass of the hot path over one batch: S1-S6 (generate n_streams x n_per_stream
doubles into HBM) for the write workloads, plus S7 (fused histogram + moments) and the NCCL
all-reduce of the histogram/moments for cfg5.  Default workload = cfg3 (BASELINE configs[2],
"Single-GPU bulk": 2^20 streams x 1024 = 2^30 doubles = 8 GiB per GPU per step).  With N > 1
every rank generates its own 2^20-stream range (stream_begin = rank * 2^20): weak scaling, no
communication on the generation path.

--impl reference times the CPU oracle (oracle/, plain C, one thread) on a bounded sample of the
same workload; it is the only other place this file executes oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1401_8230_b200 import workloads as W  # noqa: E402

METRIC = "Gdoubles/s generated (1/2/4/8 B200) and % of HBM-write roofline"
FALLBACK_HBM = 6650.0  # GB/s, /opt/skills/guides/B200_PROFILING.md fallback
KERNELS = {0: "gen_kernel", 1: "gen_seg_kernel", 2: "gen_jump_kernel", 3: "gen_mrg_kernel",
           4: "gen_segc_kernel", 5: "gen_jump_narrow_kernel"}
STORES = {0: "TMA", 1: "TILE", 2: "STG8", 3: "DIRECT", 4: "ROW", 5: "ROW1K", 6: "SEG", 7: "SEGC"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--warm-l2", action="store_true",
                    help="experiments only: no L2 flush between the steps of small workloads "
                         "(the line says so in config.l2); never a bench value")
    ap.add_argument("--sustained-s", type=float, default=1.5,
                    help="length of the sustained-throughput window (0: skip)")
    ap.add_argument("--hist-only", action="store_true",
                    help="consume workloads on one GPU: histogram + count only (d_pow = NULL; "
                         "BASELINE cfg4's 'fused 2^16-bin histogram'), no power sums")
    ap.add_argument("--consume", action="store_true",
                    help="add the fused consumer (S7) to a write workload (cfg5 always has it)")
    ap.add_argument("--no-write", action="store_true",
                    help="consume workloads: fused histogram/moments only, outputs not stored")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flags", type=int, default=0, help="extra prngd flags")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank its own per-GPU shard (default); strong: one global "
                         "stream space split over the ranks")
    ap.add_argument("--reduce", default="auto", choices=["auto", "nvls", "p2p", "nccl"],
                    help="N > 1 statistics exchange: NVLS multicast reductions in the finalize "
                         "kernel (NEXT-4), peer-memory atomics in the kernel, or NCCL; auto = "
                         "the first of nvls, p2p, nccl that works on every rank")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay each step from a CUDA graph (auto: steps under 0.2 ms, N=1)")
    ap.add_argument("--streams", type=int, default=0,
                    help="override streams per GPU (experiments; the config names it)")
    ap.add_argument("--store", default="auto",
                    choices=["auto", "seg", "segc", "row", "row1k", "tma", "tile", "direct"],
                    help="store path A/B (include/prngd.h PRNGD_FLAG_STORE_*)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload_params(name: str, rank: int, world: int, scaling: str = "weak") -> dict:
    from paper_1401_8230_b200 import dist as D
    if scaling == "strong":
        # a fixed global stream space split over the ranks (cfg5's 2^23 global
        # streams; at N = 1 that is 2^34 outputs, so use it with --no-write)
        p = W.config(name)
        if name == "cfg5":
            p["n_streams"] = 1 << 23
        return D.shard_params(p, rank, world, D.STRONG)
    # per-GPU shard of the global stream space: rank r owns [r*n, (r+1)*n) (weak scaling)
    return D.shard_params(W.config(name), rank, world, D.WEAK)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def traffic_per_launch():
    """dram read+write bytes per launch of the generate kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.power, self.reasons, self.ok = [], [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    @staticmethod
    def max_mhz_static():
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(0)
            return pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return None

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["nvml unavailable"]}
        rs = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        out = {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
               "reasons": rs, "samples": len(self.samples)}
        if self.power:
            out["power_w_median"] = statistics.median(self.power)
            out["power_w_max"] = max(self.power)
        return out


def cpu_baseline(p: dict, target_s: float = 12.0) -> dict:
    """The oracle as it stands, one host thread, on the first streams of the workload."""
    import oracle
    oracle.build()
    ns = 1024
    t0 = time.perf_counter()
    oracle.generate(p, stream_begin=p["stream_begin"], n_streams=ns, want_out=False,
                    want_stats=p.get("_consume", False))
    dt = time.perf_counter() - t0
    ns = max(1024, min(p["n_streams"], int(ns * target_s / max(dt, 1e-3)) // 1024 * 1024))
    t0 = time.perf_counter()
    oracle.generate(p, stream_begin=p["stream_begin"], n_streams=ns, want_out=True,
                    want_stats=p.get("_consume", False))
    dt = time.perf_counter() - t0
    n = ns * p["n_per_stream"]
    res = {"value": n / dt / 1e9, "unit": "Gdoubles/s", "cores": 1, "kind": "oracle",
           "sample": f"first {ns} of {p['n_streams']} streams x {p['n_per_stream']} "
                     f"({n} doubles, {dt:.1f} s, outputs written to host RAM)"}
    # The same unmodified oracle over stream-range shards on every host core:
    # one thread per core, each calling the C oracle (ctypes releases the GIL) on its own slice.
    try:
        import threading
        cores = max(1, len(os.sched_getaffinity(0)))
        # half the 1-core sample in total (bounded host memory), split over the cores
        per = max(256, ns // (2 * cores) // 256 * 256)
        per = min(per, max(1, p["n_streams"] // cores))
        outs = [None] * cores

        def work(i):
            outs[i] = oracle.generate(p, stream_begin=p["stream_begin"] + i * per, n_streams=per,
                                      want_out=True, want_stats=p.get("_consume", False))
        th = [threading.Thread(target=work, args=(i,)) for i in range(cores)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        dtn = time.perf_counter() - t0
        nn = cores * per * p["n_per_stream"]
        res["n_core"] = {"value": nn / dtn / 1e9, "unit": "Gdoubles/s", "cores": cores,
                         "sample": f"{cores} threads x {per} streams x {p['n_per_stream']} "
                                   f"({nn} doubles, {dtn:.1f} s)"}
    except Exception as e:  # a reported baseline only
        res["n_core"] = {"value": None, "note": f"unavailable: {e}"}
    return res


def device_facts(torch) -> dict:
    """SURVEY Appendix B facts confirmed on the box the bench ran on."""
    try:
        pr = torch.cuda.get_device_properties(torch.cuda.current_device())
        d = {"name": pr.name, "sm_count": pr.multi_processor_count,
             "cc": f"{pr.major}.{pr.minor}", "hbm_gib": round(pr.total_memory / 2**30, 1)}
        for k in ("L2_cache_size", "shared_memory_per_multiprocessor",
                  "shared_memory_per_block_optin", "regs_per_multiprocessor",
                  "max_threads_per_multi_processor"):
            if hasattr(pr, k):
                d[k] = getattr(pr, k)
        return d
    except Exception as e:  # informational only
        return {"error": str(e)}


def write_ceiling(out, stream, torch) -> dict:
    import ctypes
    try:
        from paper_1401_8230_b200 import build as B
        L = ctypes.CDLL(B.build_tools())
    except Exception as e:  # measurement aid only
        return {"write_ceiling_gbs": None, "write_ceiling_note": f"unavailable: {e}"}
    L.wc_store.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                           ctypes.c_void_p]
    n = out.numel()
    res = {}
    names = {0: "contig_stg16", 1: "contig_stg32", 2: "rowtile_pattern_stg16", 3: "contig_bulk16k"}
    for mode, name in names.items():
        for k in range(3):
            L.wc_store(out.data_ptr(), n, mode, k, stream.cuda_stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for k in range(20):
            L.wc_store(out.data_ptr(), n, mode, 100 + k, stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        res[name] = 20 * 8 * n / (a.elapsed_time(b) * 1e-3) / 1e9
    contig = {k: v for k, v in res.items() if k.startswith("contig")}
    return {"write_ceiling_gbs": max(contig.values()), "write_ceiling_detail": res}


def small_step_floor(out, stream, torch, scratch, scratch_rd, steps: int = 50) -> dict:
    """A plain store of the step's bytes (tools/write_ceiling.cu, contiguous 32-byte stores),
    timed exactly like an L2-flushed bench step: the flush (write + read of 256 MiB), then
    events around the store launch alone.  The floor a small step cannot beat."""
    import ctypes
    import statistics as stt
    try:
        from paper_1401_8230_b200 import build as B
        L = ctypes.CDLL(B.build_tools())
    except Exception as e:  # measurement aid only
        return {"store_step_us": None, "note": f"unavailable: {e}"}
    L.wc_store.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                           ctypes.c_void_p]
    n = out.numel()
    for k in range(3):
        L.wc_store(out.data_ptr(), n, 1, k, stream.cuda_stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    for k in range(steps):
        scratch.fill_(float(k))
        scratch_rd.sum()
        ev[k][0].record(stream)
        L.wc_store(out.data_ptr(), n, 1, 100 + k, stream.cuda_stream)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    per = [a.elapsed_time(b) * 1e3 for a, b in ev]
    return {"store_step_us": stt.mean(per), "store_step_us_median": stt.median(per),
            "store_gd_s": n / (stt.mean(per) * 1e-6) / 1e9,
            "note": "plain contiguous 32-byte store kernel of the same bytes, same flush + "
                    "per-step-event protocol (tools/write_ceiling.cu); frac = its step time / "
                    "this step's"}


def shared_config(args, p: dict, world: int) -> dict:
    """The workload keys both arms report (this implementation's line adds its launch details,
    the reference arm its CPU sample), so the driver's ratio compares like with like."""
    consume = args.workload == "cfg5" or args.consume
    return {"workload": f"{args.workload}: {W.DESCRIPTIONS.get(args.workload, args.workload)}",
            "streams_per_gpu": p["n_streams"], "n_per_stream": p["n_per_stream"],
            "seed": p["seed"], "bytes_written_per_step_per_gpu": 8 * p["n_streams"] * p["n_per_stream"],
            "parallelism": f"stream-range shards x{world}",
            "method_flags": args.flags | p.get("map_flags", 0),
            "base_generator": "MRG32k3a" if p.get("mrg") else "xorshift128",
            "write_outputs": not (consume and args.no_write),
            **({"statistics": "histogram + count" if getattr(args, "hist_only", False)
                else "histogram + count + 4 power sums"} if consume else {})}


def run_reference(args, rank, world):
    """Reference arm = the CPU oracle (this tier has no upstream code)."""
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    p = workload_params(args.workload, 0, 1, args.scaling)
    cons = args.workload == "cfg5" or args.consume
    ns = 4096  # bounded sample per step: 4096 streams x n_per_stream
    nout = ns * p["n_per_stream"]
    for _ in range(args.warmup):
        oracle.generate(p, stream_begin=0, n_streams=ns, want_out=True, want_stats=cons)
    t0 = time.perf_counter()
    for k in range(args.steps):
        oracle.generate(p, stream_begin=k * ns, n_streams=ns, want_out=True, want_stats=cons)
    dt = time.perf_counter() - t0
    v = nout * args.steps / dt / 1e9
    sample = f"{ns} streams x {p['n_per_stream']} per step ({args.workload} shape)"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Gdoubles/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(shared_config(args, p, world), sample=sample),
            "cpu_baseline": {"value": v, "unit": "Gdoubles/s", "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "Gdoubles/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_1401_8230_b200 import dist as D
    from paper_1401_8230_b200 import prngd as P

    if not torch.cuda.is_available():
        print(json.dumps({"error": "no CUDA device"}))
        return 1
    # Test hooks for exercising the N > 1 code path on a one-GPU box (timings meaningless):
    # PRNGD_BENCH_SAME_GPU=1 puts every rank on cuda:0, PRNGD_BENCH_BACKEND=gloo avoids NCCL's
    # one-rank-per-GPU rule.  The driver's multi-GPU runs use neither.
    same_gpu = os.environ.get("PRNGD_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("PRNGD_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    p = workload_params(args.workload, rank, world, args.scaling)
    if args.streams:
        p["stream_begin"] = rank * args.streams
        p["n_streams"] = args.streams
    p["flags"] = args.flags | P.STORE_FLAGS[args.store] | p.get("map_flags", 0)
    if p.get("mrg"):
        p["flags"] |= P.PRNGD_FLAG_MRG32K3A
    consume = args.workload == "cfg5" or args.consume
    g = P.Generator(**p)
    nout = p["n_streams"] * p["n_per_stream"]
    out = torch.empty((p["n_streams"], p["n_per_stream"]), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    if consume:
        # one buffer for the three accumulators, so a step clears them with one fill
        acc = torch.zeros(65536 + 4 + 1, dtype=torch.int64, device="cuda")
        hist = acc[:65536]
        pw = acc[65536:65540].view(torch.float64)
        cnt = acc[65540:]
    # The statistics exchange (N > 1): by default rank 0's accumulator is mapped into every rank
    # (CUDA IPC, peer memory over NVLink) and each rank's finalize kernel adds into it with device
    # atomics -- fused into the library's own launches; NCCL all-reduce is the fallback.
    peer, reduce_mode = None, None
    mc_err = None
    if consume and world > 1 and args.reduce in ("auto", "nvls"):
        # NEXT-4: in-switch reduction through an NVLS multicast object (every rank's copy gets
        # the all-reduced statistics inside the finalize kernels); raises consistently on every
        # rank when the fabric cannot provide it
        try:
            peer = D.McStats()
            ok, why = D.verify_reduction(peer, device_wait=not same_gpu)
            if not ok:
                peer.close()
                raise RuntimeError(f"self-check against NCCL failed: {why}")
            reduce_mode = "nvls (verified against NCCL on a small workload)"
        except Exception as e:
            peer, mc_err = None, str(e)
    if consume and world > 1 and peer is None:
        reduce_mode = "nccl" + (f" (multicast unavailable: {mc_err})" if mc_err else "")
        if args.reduce in ("auto", "p2p"):
            err = None
            try:
                peer = D.PeerStats()
                peer.zero(stream)
                torch.cuda.synchronize()
                if os.environ.get("PRNGD_BENCH_FAIL_PEER_RANK") == str(rank):  # test hook
                    raise RuntimeError("simulated peer-mapping failure")
            except Exception as e:  # e.g. no peer access to rank 0's GPU
                err, peer = str(e), None
            # every rank must take the same path: p2p only if it worked everywhere
            ok = torch.tensor([0 if err else 1], dtype=torch.int32, device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() == 1:
                vok, why = D.verify_reduction(peer, device_wait=not same_gpu)
                if vok:
                    reduce_mode = "p2p (verified against NCCL on a small workload)"
                else:
                    err = f"self-check against NCCL failed: {why}"
            if ok.item() != 1 or err:
                if peer is not None:
                    torch.cuda.synchronize()
                    if rank != 0:
                        peer.close()
                    dist.barrier()
                    if rank == 0:
                        peer.close()
                    peer = None
                else:
                    dist.barrier()
                reduce_mode = "nccl (peer memory unavailable" + (f": {err})" if err else " on a rank)")
            dist.barrier()
            if reduce_mode.startswith("p2p") and mc_err:
                reduce_mode += f"; multicast unavailable: {mc_err}"

    def step(st=stream):
        if consume and peer is not None:
            # accumulates over steps into rank 0's peer-mapped buffer (no per-step collective);
            # each call also bumps the accumulator's arrival counter (completion protocol)
            peer.consume(g.handle, None if args.no_write else out, st)
        elif consume:
            acc.zero_()
            P.prngd_generate_consume(g.handle, None if args.no_write else out, hist,
                                     None if args.hist_only else pw, cnt, st)
            if world > 1:  # the path's only exchange: NCCL all-reduce of the statistics
                D.allreduce_stats(hist, pw, cnt)
        else:
            P.prngd_generate(g.handle, out, st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = g.last_launches

    # Small configurations are launch-bound from Python (cfg1: a 7 us kernel behind ~6 us of
    # host work per call): replay the step from a CUDA graph there (same kernels, same launches).
    wa, wb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wa.record(stream)
    for _ in range(3):
        step()
    wb.record(stream)
    torch.cuda.synchronize()
    # Outputs smaller than twice the 126 MB L2 would stay cache-resident between steps: those
    # workloads write a 256 MiB scratch buffer between timed steps (an L2 flush) and are timed
    # by per-step events around the step alone.
    l2_flush = 8 * nout < (256 << 20) and not args.warm_l2
    # (written, then a second buffer read, so the flush's own dirty lines are written back
    # before the timed step rather than during it)
    scratch = torch.empty(32 << 20, dtype=torch.float64, device="cuda") if l2_flush else None
    scratch_rd = torch.zeros(32 << 20, dtype=torch.float64, device="cuda") if l2_flush else None
    use_graph = args.graph == "on" or (args.graph == "auto" and world == 1 and not l2_flush and
                                        wa.elapsed_time(wb) / 3 < 0.2)
    graph = None
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                step(torch.cuda.current_stream())
        stream.wait_stream(side)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()

    # -------------------------------------------------- timed region (device events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        if graph is not None:
            for k in range(args.steps):
                graph.replay()
        elif l2_flush:
            for k in range(args.steps):
                scratch.fill_(float(k))
                scratch_rd.sum()
                ev[k][0].record(stream)
                step()
                ev[k][1].record(stream)
        else:
            for k in range(args.steps):
                ev[k][0].record(stream)
                step()
                ev[k][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = t0.elapsed_time(t1)
    per = ([total_ms / args.steps] * args.steps if graph is not None
           else [a.elapsed_time(b) for a, b in ev])
    step_stats = {"step_ms_median": statistics.median(per), "step_ms_best": min(per),
                  "value_at_median": world * nout / (statistics.median(per) * 1e-3) / 1e9,
                  "value_at_best": world * nout / (min(per) * 1e-3) / 1e9,
                  "note": "this rank's per-step events (x N ranks)"}
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = t.item()
    ms = total_ms / args.steps
    if l2_flush:  # the timed region is the steps alone, not the flushes between them
        ms = statistics.mean(per)
        if world > 1:
            tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = tt.item()
    total_out = world * nout
    if world > 1:  # strong sharding gives ranks slightly different counts
        tt = torch.tensor([nout], dtype=torch.int64, device="cuda")
        dist.all_reduce(tt)
        total_out = int(tt.item())
    value = total_out / (ms * 1e-3) / 1e9

    # -------------------------------------------------- sustained window (power-capped regime)
    # The driver's short run (e.g. 20 steps = 26 ms of cfg3) sees burst clocks; the same step
    # repeated back to back for >= --sustained-s seconds shows the steady state under the
    # board's power cap, with its own clock / power sample.
    sustained = None
    if args.sustained_s > 0 and not l2_flush:
        n_sus = max(args.steps, int(args.sustained_s * 1e3 / max(ms, 1e-3)) + 1)
        if world > 1:
            tn = torch.tensor([n_sus], dtype=torch.int64, device="cuda")
            dist.all_reduce(tn, op=dist.ReduceOp.MAX)
            n_sus = int(tn.item())
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(torch.cuda.current_device()) as clk_s:
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(n_sus):
                if graph is not None:
                    graph.replay()
                else:
                    step()
            s1.record(stream)
            torch.cuda.synchronize()
        ts = torch.tensor([s0.elapsed_time(s1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        ms_s = ts.item() / n_sus
        sustained = {"value": total_out / (ms_s * 1e-3) / 1e9, "unit": "Gdoubles/s",
                     "steps": n_sus, "seconds": ts.item() / 1e3, "ms_per_step": ms_s,
                     "clocks": clk_s.summary(),
                     "note": "same step back to back for >= --sustained-s s (device events, max "
                             "over ranks); the headline value is the driver's short run"}

    # -------------------------------------------------- roofline of the dominant kernel
    # For write workloads the step is exactly one generate launch; its average duration is
    # the mean of the per-step event pairs on the launching stream.
    peak, peak_src = peaks()
    kern_ms = statistics.mean(per) if not consume else None
    bytes_launch = 8 * nout
    tr = traffic_per_launch()
    traffic, traffic_src = None, None
    path_name = STORES.get(g.info["store"])
    kind = "consume" if consume else "generate"
    for ent in (tr or {}).get("entries", []):
        if (ent.get("workload") == args.workload and ent.get("kind", "generate") == kind and
                args.store == "auto" and not args.no_write):
            traffic, traffic_src = ent.get("dram_bytes_per_launch"), ent.get("source")
    if consume:
        # dominant kernel = fused generate+consume; its own duration needs the launch list.
        kern_ms = statistics.mean(per)
    achieved = bytes_launch / (kern_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": peak_src,
            "kernel": ("consume_kernel+finalize" if consume else
                       KERNELS[g.info["kernel"]] if g.info["kernel"] in (2, 5) else  # no store path
                       KERNELS[g.info["kernel"]] + f" (store path {STORES[g.info['store']]})"),
            "algorithmic_bytes_per_launch": bytes_launch, "kernel_ms": kern_ms,
            "frac_of_8TBs_nominal": achieved / 8000.0}
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    clk_ghz = (ClockSampler.max_mhz_static() or 1965) / 1e3
    if consume and not args.no_write and not p.get("mrg"):
        # The fused write + statistics kernel is not HBM-bound (S7): its
        # instruction-issue share, from the algorithmic count per output -- generator 18
        # (2 xorshift128 draws x 6, band test 1, Eq.(4) 5), statistics 10 (power sums 5; bin by
        # one round-toward-zero DADD, word mask, field increment 2, packed add), store 1.5 (STS,
        # LDS, STG per 2 outputs): 29.5 -- against 4 schedulers x 32 lanes x SMs x max SM clock.
        ins = 29.5
        roof["issue"] = {"algorithmic_instructions_per_output": ins,
                         "achieved": ins * nout / (kern_ms * 1e-3) / 1e9,
                         "peak": 4 * 32.0 * sms * clk_ghz, "unit": "Ginstr/s",
                         "frac": ins * nout / (kern_ms * 1e-3) / 1e9 / (4 * 32.0 * sms * clk_ghz),
                         "note": "issue/latency-bound: 34.0 issued per output at 67% issue, "
                                 "ALU pipe 57%, 16 warps per SM (row-segment consumer, "
                                 "profiles/r02s_summary.txt)"}
    if consume and args.no_write and not p.get("mrg"):
        # Nothing is written: one shared-memory histogram add per output.  Peak = the measured
        # rate of the same packed adds (no return value) at the kernel's 16 warps per SM
        # (tools/smem_hist_rate.py, profiles/r01b_smem_hist_rate.json); DESIGN.md section 8.
        ach = nout / (kern_ms * 1e-3) / 1e9
        try:
            with open(os.path.join(ROOT, "profiles", "r01b_smem_hist_rate.json")) as f:
                pk = float(json.load(f)["G_adds_per_s"]["red_w16"])
            src = "measured: tools/smem_hist_rate.py red.shared packed adds, 16 warps/SM"
        except Exception:
            pk = 2.0 * sms * clk_ghz
            src = "derived: 2 ATOMS lanes/clk/SM x SMs x max SM clock (B300_MICROARCH.md)"
        roof = {"bound": "smem_atomics", "achieved": ach, "peak": pk, "unit": "Gadd/s",
                "frac": ach / pk, "traffic": None, "kernel": "consume_kernel+finalize",
                "peak_source": src, "algorithmic_adds_per_launch": nout, "kernel_ms": kern_ms,
                "note": "issue-bound below this peak (DESIGN.md section 8)"}
    elif p.get("mrg"):
        # MRG32k3a (NEXT-2): instruction-issue bound.  Algorithmic
        # instructions per output (mrg26 runs the per-batch band test): per MRG32k3a draw 21
        # (two binary64 components x 5: product, fused product-difference, round-down shift
        # pair, remainder; combination 6 with the floor reduction's values in [0, m]: two exact
        # conversions, component 2's m2 -> 0 min, subtract-and-wrap 3; R23 test + mask 2; ring
        # append 3: address, predicated store, counter), 2.03 draws per output (26-bit
        # reduce-to-width rejects 1/64), plus 11 per output (Eq.(4) 6, ring read 2, band test 2,
        # store 1): 21 x 2.03 + 11 = 54 (60 with round 2's balanced representatives, whose
        # combination needed two sign fixes of 2 more).  The fused consumer (consume_mrg_kernel)
        # adds the statistics' 10 (power sums 5, bin 5) and drops the store (1) when nothing is
        # written.
        # Peak: 4 schedulers x 32 lanes per clock per SM x SMs x max SM clock.
        ops = 54.0 + (10.0 if consume else 0.0) - (1.0 if consume and args.no_write else 0.0)
        ach = ops * nout / (kern_ms * 1e-3) / 1e9
        pk = 4 * 32.0 * sms * clk_ghz
        roof = {"bound": "alu", "achieved": ach, "peak": pk, "unit": "Ginstr/s", "frac": ach / pk,
                "traffic": None,
                "kernel": "consume_mrg_kernel+finalize" if consume else "gen_mrg_kernel",
                "peak_source": "derived: 4 warp-instructions/clk/SM (one per scheduler) x 32 "
                               "lanes x SMs x max SM clock",
                "algorithmic_instructions_per_output": ops,
                "fp64_ops_per_output": 24.3, "kernel_ms": kern_ms,
                "hbm_write_gbs": achieved}

    if sustained is not None and roof["bound"] == "hbm":
        sustained["achieved_gbs"] = bytes_launch * world / (sustained["ms_per_step"] * 1e-3) / 1e9 / world
        sustained["roofline_frac"] = sustained["achieved_gbs"] / peak
        sustained["frac_of_8TBs_nominal"] = sustained["achieved_gbs"] / 8000.0

    # -------------------------------------------------- pure-store ceiling on the same buffer
    # (B13, tools/write_ceiling.cu: incompressible values, 16/32-byte coalesced stores)
    if not consume and not l2_flush:
        roof.update(write_ceiling(out, stream, torch))
        if roof.get("write_ceiling_gbs"):
            roof["frac_of_write_ceiling"] = achieved / roof["write_ceiling_gbs"]
    elif not consume:
        # small outputs (L2-resident, flushed between steps): the step is launch-bound, so the
        # reference is a plain 32-byte store kernel of the same bytes timed by the same protocol
        fl = small_step_floor(out, stream, torch, scratch, scratch_rd)
        if fl.get("store_step_us"):
            fl["frac"] = fl["store_step_us"] / (ms * 1e3)  # our step vs the store-only step
        roof["small_step_floor"] = fl

    # -------------------------------------------------- end to end through the C ABI, host buffer
    e2e = None
    if args.e2e_steps > 0 and not consume:
        # prngd_generate_host into pinned host memory: the whole per-rank workload when the host
        # has the memory to pin it for every local rank (3x headroom), else a 2^17-stream
        # sample (the call is PCIe-bound, so the rate does not depend on the sample size)
        ns_e = p["n_streams"]
        try:
            with open("/proc/meminfo") as f:
                avail = int(next(l for l in f if l.startswith("MemAvailable")).split()[1]) * 1024
        except Exception:
            avail = 0
        local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        if 3 * local_ranks * 8 * nout > avail:
            ns_e = min(p["n_streams"], 1 << 17)
        ge = P.Generator(**dict(p, n_streams=ns_e))
        ne = ns_e * p["n_per_stream"]
        host = torch.empty((ns_e, p["n_per_stream"]), dtype=torch.float64, pin_memory=True)
        P.prngd_generate_host(ge.handle, host, stream)  # warm-up (allocates staging)
        if world > 1:
            dist.barrier()
        te = time.perf_counter()
        for _ in range(args.e2e_steps):
            P.prngd_generate_host(ge.handle, host, stream)
        torch.cuda.synchronize()
        de = torch.tensor([time.perf_counter() - te], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(de, op=dist.ReduceOp.MAX)
        e2e = {"value": world * ne * args.e2e_steps / de.item() / 1e9, "unit": "Gdoubles/s",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8 * ne,
               "full_workload": ns_e == p["n_streams"],
               "note": f"prngd_generate_host: chunked generate + pinned D2H, overlapped; inputs "
                       f"are the parameter struct only; {ns_e} streams x {p['n_per_stream']} "
                       f"per rank per step"}
        del host
        ge.close()
    elif args.e2e_steps > 0 and consume:
        # The consumer's result is its statistics: every step generates (and writes, unless
        # --no-write) on the device, reduces, and reads the histogram + power sums + count back
        # into pinned host memory (the step's "metric").
        hh = torch.empty(65536, dtype=torch.int64, pin_memory=True)
        hp = torch.empty(4, dtype=torch.float64, pin_memory=True)
        hc = torch.empty(1, dtype=torch.int64, pin_memory=True)
        if peer is not None:
            # per-step results from the shared accumulator: start from zero, then every step
            # rank 0 waits (device-side acquire on the arrival counter) for all ranks' calls,
            # reads, and zeroes the statistics before the barrier releases the next step
            torch.cuda.synchronize()
            dist.barrier()
            peer.zero(stream)
            torch.cuda.synchronize()
            dist.barrier()
        else:
            step()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e2e_counts = []
        te = time.perf_counter()
        for k in range(args.e2e_steps):
            step()
            if peer is not None:
                if same_gpu:  # ranks share one GPU (test hook): host-side completion instead
                    torch.cuda.synchronize()
                    dist.barrier()
                if rank == 0:
                    if not same_gpu:
                        peer.wait(peer.expected(k + 1), stream)
                    P.prngd_copy(hh, peer.hist, 65536 * 8, stream)
                    P.prngd_copy(hp, peer.pow, 32, stream)
                    P.prngd_copy(hc, peer.count, 8, stream)
                    peer.zero(stream, counter=False)
                torch.cuda.synchronize()
                dist.barrier()
            else:
                hh.copy_(hist, non_blocking=True)
                hp.copy_(pw, non_blocking=True)
                hc.copy_(cnt, non_blocking=True)
                torch.cuda.synchronize()
            e2e_counts.append(int(hc[0]))
        de = torch.tensor([time.perf_counter() - te], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(de, op=dist.ReduceOp.MAX)
        e2e = {"value": world * nout * args.e2e_steps / de.item() / 1e9, "unit": "Gdoubles/s",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 65536 * 8 + 32 + 8,
               "counts_per_step_ok": all(c == world * nout for c in e2e_counts) if rank == 0
                                     else None,
               "note": "prngd_generate_consume per step + D2H of the statistics (histogram, power "
                       "sums, count) into pinned host memory, synchronised every step"
                       + ("; N > 1: rank 0 waits on the accumulator's arrival counter, reads and "
                          "zeroes it, then a barrier" if peer is not None else "")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        q = dict(p)
        q["_consume"] = consume
        cpu = cpu_baseline(q)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gdoubles/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": dict(shared_config(args, p, world), **{
                       "l2": ("EXPERIMENT: warm L2, no flush between steps (--warm-l2)"
                              if args.warm_l2 and 8 * nout < (256 << 20) else
                              "outputs fit in the 126 MB L2: a 256 MiB buffer is written and "
                              "another read between timed steps (L2 flush, write-back drained); "
                              "per-step events time the step"
                              if l2_flush else
                              "inputs none; 8 B/output written, >126 MB L2 per step (no flush)"),
                       "flags": p["flags"], "store": args.store,
                       "cuda_graph": graph is not None,
                       "stats_reduce": reduce_mode}),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "device": device_facts(torch),
            "gpu_launches": launches_per_step * args.steps,
            "per_step": step_stats,
            "sustained": sustained,
            "pct_hbm_write_roofline": 100.0 * achieved / peak if roof["bound"] == "hbm" else None,
        }
        print(json.dumps(line), flush=True)
    if isinstance(peer, D.McStats):
        torch.cuda.synchronize()
        peer.close()  # barrier, then every rank releases its mappings
    elif peer is not None:  # the owner frees only after every other rank unmapped
        torch.cuda.synchronize()
        dist.barrier()
        if rank != 0:
            peer.close()
        dist.barrier()
        peer.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
