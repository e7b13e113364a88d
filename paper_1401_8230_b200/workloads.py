"""Seeded synthetic workloads shared by the tests, bench.py and smoke().

This module holds NO arithmetic of the method: only parameter sets (BASELINE.json configs) and
seeded numpy generators of raw (x1, x2) draw values for the mapping tests.  It is the one module
both the oracle side and the CUDA side may use.
"""
from __future__ import annotations

import numpy as np

FULL32 = dict(w=32, a0=0, a=2**32 - 1, b0=0, b=2**32 - 1)
BYTE8 = dict(w=8, a0=0, a=255, b0=0, b=255)
ASYM = dict(w=32, a0=1, a=2**32 - 1, b0=0, b=2**31 - 1)

SEED = 1                       # BASELINE.json configs[0] "splitmix64(seed=1, stream)"
SEED2 = 0x0123456789ABCDEF     # repeat parity seed

# BASELINE.json configs[0..4] (cfg1..cfg5).  n_streams / n_per_stream are per GPU; cfg5 is the
# per-rank shard of 2^23 global streams (stream_begin = rank * 2^20).
CONFIGS = {
    "cfg1": dict(FULL32, seed=SEED, stream_begin=0, n_streams=1024, n_per_stream=1024),
    "cfg2": dict(BYTE8, seed=SEED, stream_begin=0, n_streams=4096, n_per_stream=1024),
    "cfg3": dict(FULL32, seed=SEED, stream_begin=0, n_streams=2**20, n_per_stream=1024),
    "cfg4": dict(ASYM, seed=SEED, stream_begin=0, n_streams=2**20, n_per_stream=4096),
    "cfg5": dict(FULL32, seed=SEED, stream_begin=0, n_streams=2**20, n_per_stream=2048),
    # NEXT-2 (not a BASELINE config): cfg3's shape on the MRG32k3a base generator, 26-bit draws
    # NEXT-1 (not BASELINE configs): cfg3's shape with the other mappings.  `map` / `open` are
    # the oracle's parameters, `map_flags` the same choice as include/prngd.h flag bits.
    "eq5": dict(FULL32, seed=SEED, stream_begin=0, n_streams=2**20, n_per_stream=1024, map=5,
                map_flags=1 << 6),
    "eq6": dict(FULL32, seed=SEED, stream_begin=0, n_streams=2**20, n_per_stream=1024, map=6,
                map_flags=2 << 6),
    "open4": dict(FULL32, seed=SEED, stream_begin=0, n_streams=2**20, n_per_stream=1024,
                  open=True, map_flags=0x100),
    "mrg26": dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1, seed=SEED, stream_begin=0,
                  n_streams=2**20, n_per_stream=1024, mrg=True),
}

DESCRIPTIONS = {
    "cfg1": "w=32 full range, 1024 streams x 1024 (oracle-scale parity)",
    "cfg2": "w=8 top byte, 4096 streams x 1024 (rejection stress)",
    "cfg3": "w=32 full range, 2^20 streams x 1024 = 2^30 doubles (8 GiB) single-GPU bulk",
    "cfg4": "x1 in [1,2^32-1], x2 in [0,2^31-1], k=2^-32, 2^20 x 4096, write + histogram",
    "cfg5": "w=32 full range, 2^23 global streams, 2^20 x 2048 per GPU, write + hist + moments",
    "mrg26": "NEXT-2: MRG32k3a base generator, w=26 full range, 2^20 streams x 1024",
    "eq5": "NEXT-1: Eq.(5) discrete-grid normalisation, cfg3 shape",
    "eq6": "NEXT-1: Eq.(6) unit-interval form, cfg3 shape",
    "open4": "NEXT-1: open interval 1 - z' of Eq.(4), cfg3 shape",
}


def config(name: str, **over) -> dict:
    p = dict(CONFIGS[name])
    p.update(over)
    return p


def shard(p: dict, rank: int, world: int) -> dict:
    """Stream-range shard of rank r of R over p's N = n_streams global streams:
    [floor(rN/R), floor((r+1)N/R))."""
    n = p["n_streams"]
    lo, hi = rank * n // world, (rank + 1) * n // world
    q = dict(p)
    q["stream_begin"] = p.get("stream_begin", 0) + lo
    q["n_streams"] = hi - lo
    return q


def random_pairs(seed: int, n: int, bits1: int, bits2: int):
    """n uniformly random (x1, x2) draw values of the given widths (numpy PCG64)."""
    g = np.random.Generator(np.random.PCG64(seed))
    x1 = g.integers(0, 1 << bits1, size=n, dtype=np.uint64).astype(np.uint32)
    x2 = g.integers(0, 1 << bits2, size=n, dtype=np.uint64).astype(np.uint32)
    return x1, x2


def edge_pairs(bits1: int, bits2: int, span: int = 16):
    """Pairs at the corners of the draw square: x1, x2 within `span` of 0 and of the maximum,
    plus x1 at every power of two +-3 (binade edges).  All combinations, deduplicated."""
    m1, m2 = (1 << bits1) - 1, (1 << bits2) - 1
    xs1 = set(range(0, min(span, m1 + 1))) | set(range(max(0, m1 - span + 1), m1 + 1))
    for e in range(bits1):
        for d in (-3, -2, -1, 0, 1, 2, 3):
            v = (1 << e) + d
            if 0 <= v <= m1:
                xs1.add(v)
    xs2 = set(range(0, min(span, m2 + 1))) | set(range(max(0, m2 - span + 1), m2 + 1))
    xs2 |= {m2 >> 1, (m2 >> 1) + 1}
    a1 = np.array(sorted(xs1), dtype=np.uint64)
    a2 = np.array(sorted(xs2), dtype=np.uint64)
    g1, g2 = np.meshgrid(a1, a2, indexing="ij")
    return g1.ravel().astype(np.uint32), g2.ravel().astype(np.uint32)
