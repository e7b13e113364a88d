"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE north_star): bit-exact raw draws and pair indices, 0 ulp for the doubles (compared
as int64 bit patterns), identical histograms/counts; FP64 power sums at relative 1e-12 (R16).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1401_8230_b200 import prngd as P  # noqa: E402
from paper_1401_8230_b200 import workloads as W  # noqa: E402

# store paths of the loaded library (the A/B ones exist only in the variant build)
STORES_AVAILABLE = [P.STORE_FLAGS[n] for n in P.stores_available(list(P.STORE_FLAGS))]

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    P.lib()  # fail loudly if the native library is missing
    yield


def bits(a):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def gen(p, **over):
    q = dict(p)
    q.update(over)
    g = P.Generator(**q)
    out = g.generate()
    torch.cuda.synchronize()
    assert g.last_launches == 1
    return g, out


def assert_same(gpu_out, ref):
    gb, rb = bits(gpu_out).ravel(), bits(ref).ravel()
    bad = np.nonzero(gb != rb)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}: " \
        f"{bits(gpu_out).ravel()[bad[:3]]} vs {rb[bad[:3]]}"


# ------------------------------------------------------------------ full-config parity

@pytest.mark.parametrize("flags", STORES_AVAILABLE + [P.PRNGD_FLAG_IEEE_DIV])
def test_cfg1_bitwise(orc, flags):
    p = W.CONFIGS["cfg1"]
    _, out = gen(p, flags=flags)
    assert_same(out, orc.generate(p)["out"])


@pytest.mark.parametrize("seed", [W.SEED, W.SEED2])
def test_cfg2_bitwise_rejection_path(orc, seed):
    p = W.config("cfg2", seed=seed)
    _, out = gen(p)
    assert_same(out, orc.generate(p)["out"])


@pytest.mark.parametrize("name,over", [
    ("cfg1", {}),                                           # SEG (few streams, rare rejection)
    ("cfg2", {}),                                           # NEXT-3 narrow jump kernel
    ("cfg3", dict(n_streams=4096)),                         # ROW, bulk shape (a slice)
    ("cfg4", dict(n_streams=2048)),                         # ROW, MODE 3 (asymmetric ranges)
    ("mrg26", dict(n_streams=2048)),                        # NEXT-2 MRG32k3a
])
def test_second_seed_repeat_run(orc, name, over):
    """SURVEY 8(d)'s repeat parity run with the second seed 0x0123456789ABCDEF, on the kernel
    each BASELINE shape takes by default (AUTO), plus the fused statistics on the same inputs."""
    p = W.config(name, seed=W.SEED2, **over)
    if p.get("mrg"):
        p["flags"] = p.get("flags", 0) | P.PRNGD_FLAG_MRG32K3A
    _, out = gen(p)
    ref = orc.generate(p, want_stats=True)
    assert_same(out, ref["out"])
    g = P.Generator(**p)
    buf = torch.empty_like(out)
    _, hist, pw, cnt = g.generate_consume(buf)
    torch.cuda.synchronize()
    assert_same(buf, ref["out"])
    assert np.array_equal(hist.cpu().numpy(), ref["hist"]) and cnt.item() == ref["count"]
    assert np.allclose(pw.cpu().numpy(), ref["pow"], rtol=1e-12, atol=0)


def test_cfg2_pair_indices_and_consumed(orc):
    p = W.CONFIGS["cfg2"]
    g = P.Generator(**p)
    pidx, cons = g.pairs()
    torch.cuda.synchronize()
    r = orc.generate(p, want_out=False, want_pidx=True, want_consumed=True)
    assert np.array_equal(pidx.cpu().numpy().view(np.uint32), r["pidx"])
    assert np.array_equal(cons.cpu().numpy().view(np.uint64), r["consumed"])


def test_raw_draws_bit_exact(orc):
    p = W.CONFIGS["cfg1"]
    g = P.Generator(**p)
    raw = g.raw(64)
    torch.cuda.synchronize()
    assert np.array_equal(raw.cpu().numpy().view(np.uint32), orc.raw(p["seed"], 0, 1024, 64))


def test_cfg4_asymmetric_sampled_streams(orc):
    """cfg4 at full size (2^20 x 4096, 32 GiB) in the production launch; 48 streams spread over
    the range compared bitwise with the oracle, and properties over all 2^32 outputs."""
    p = W.CONFIGS["cfg4"]
    _, out = gen(p)
    rows = np.linspace(0, p["n_streams"] - 1, 48).astype(np.int64)
    for r in rows[:8].tolist() + rows[8:].tolist():
        ref = orc.generate(p, stream_begin=int(r), n_streams=1)["out"]
        assert_same(out[r], ref[0])
    assert bool((out > 0).all()) and bool((out < 1).all())
    mx = out.max().item()
    assert mx == float.fromhex("0x1.ffffffff00000p-1") or mx < 1.0
    del out
    torch.cuda.empty_cache()


def test_cfg3_full_size_sampled(orc):
    """cfg3 exactly as bench.py launches it: 2^30 doubles; sampled streams bitwise, and global
    properties (range, no 1.0, no 0) over every output."""
    p = W.CONFIGS["cfg3"]
    _, out = gen(p)
    rows = np.linspace(0, p["n_streams"] - 1, 64).astype(np.int64)
    ref = np.stack([orc.generate(p, stream_begin=int(r), n_streams=1)["out"][0] for r in rows])
    assert_same(out[torch.from_numpy(rows).cuda()], ref)
    assert bool((out > 0).all()) and bool((out < 1).all())
    del out
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ ragged / edge shapes

@pytest.mark.parametrize("ns,nps", [(1, 1), (1, 2), (31, 17), (33, 16), (1000, 1000),
                                    (77, 999), (64, 3), (5, 4096 + 6)])
@pytest.mark.parametrize("base", ["cfg1", "cfg2"])
def test_ragged_shapes(orc, ns, nps, base):
    p = W.config(base, n_streams=ns, n_per_stream=nps, stream_begin=12345)
    _, out = gen(p)
    assert_same(out, orc.generate(p)["out"])


@pytest.mark.parametrize("flags", STORES_AVAILABLE)
@pytest.mark.parametrize("offset", [1, 2, 3])
def test_misaligned_output_pointer(orc, flags, offset):
    """8-, 16- and 24-byte offsets: each store path falls back to the next legal one."""
    p = W.config("cfg1", n_streams=96, n_per_stream=64, flags=flags)
    g = P.Generator(**p)
    buf = torch.full((96 * 64 + offset,), -1.0, dtype=torch.float64, device="cuda")
    P.prngd_generate(g.handle, buf[offset:])
    torch.cuda.synchronize()
    assert bool((buf[:offset] == -1.0).all())
    assert_same(buf[offset:], orc.generate(p)["out"])


@pytest.mark.parametrize("flags", STORES_AVAILABLE)
@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_store_paths_bitwise(orc, flags, name):
    p = W.config(name, n_streams=200, n_per_stream=100, flags=flags)
    _, out = gen(p)
    assert_same(out, orc.generate(p)["out"])


def test_no_out_of_bounds_writes(orc):
    p = W.config("cfg1", n_streams=40, n_per_stream=30)
    g = P.Generator(**p)
    buf = torch.full((40 * 30 + 512,), -7.0, dtype=torch.float64, device="cuda")
    g.generate(buf[:40 * 30].view(40, 30))
    torch.cuda.synchronize()
    assert bool((buf[40 * 30:] == -7.0).all())


def test_general_ranges(orc):
    for par in [dict(w=20, a0=5, a=2**20 - 3, b0=0, b=2**20 - 1),
                dict(w=32, a0=1000, a=2**31 + 7, b0=0, b=2**16 - 1),
                dict(w=12, a0=0, a=100, b0=0, b=63),
                dict(w=1, a0=0, a=2, b0=0, b=1)]:
        p = dict(par, seed=9, n_streams=100, n_per_stream=130)
        _, out = gen(p)
        assert_same(out, orc.generate(p)["out"])


def test_sharding_equals_whole(orc):
    p = W.config("cfg1", n_streams=256, n_per_stream=96)
    _, whole = gen(p)
    parts = [gen(W.shard(p, r, 4))[1] for r in range(4)]
    assert_same(torch.cat(parts), whole.cpu().numpy())


def test_determinism():
    p = W.config("cfg1", n_streams=512)
    _, a = gen(p)
    _, b = gen(p)
    assert torch.equal(a.view(torch.int64), b.view(torch.int64))


def test_generate_host_matches_device(orc):
    p = W.config("cfg1", n_streams=3000, n_per_stream=512)
    g, dev = gen(p)
    host = g.generate_host()
    assert g.last_launches >= 1
    assert_same(host, dev.cpu().numpy())


def test_generate_host_jump_kernel_chunks(orc):
    """prngd_generate_host takes the kernel prngd_get_info reports (here the NEXT-3 jump kernel,
    33-pair rounds) for each staging chunk (2720 rows of 96 KiB per 256 MiB chunk: 2 chunks)."""
    p = W.config("cfg2", n_streams=4000, n_per_stream=12288)
    g = P.Generator(**p)
    assert g.info["kernel"] == 5  # w = 8: the narrow jump kernel
    host = g.generate_host().numpy()
    dev = g.generate()
    torch.cuda.synchronize()
    assert np.array_equal(host.view(np.int64), dev.cpu().numpy().view(np.int64))
    for r in (0, 1, 2719, 2720, 3999):
        ref = orc.generate(p, stream_begin=r, n_streams=1)["out"]
        assert np.array_equal(host[r].view(np.int64), ref.ravel().view(np.int64))


# ------------------------------------------------------------------ the mapping alone

def test_map_exhaustive_w8(orc):
    p = W.BYTE8
    g = P.Generator(**p, seed=1, n_streams=1, n_per_stream=2)
    x1, x2 = np.meshgrid(np.arange(256, dtype=np.uint32), np.arange(256, dtype=np.uint32),
                         indexing="ij")
    z = g.map(torch.from_numpy(x1.ravel()).cuda(), torch.from_numpy(x2.ravel()).cuda())
    torch.cuda.synchronize()
    q, _ = orc.enumerate_pairs(p)
    assert_same(z, q.ravel())


def test_map_exhaustive_w16_closed_form():
    """All 2^32 pairs at w=16 against the closed form RN(j/(2^16-1)^2) computed by torch's IEEE
    tensor/tensor division on the GPU (independent of the library's division; a Python-scalar
    divisor would make torch multiply by a rounded reciprocal instead)."""
    p = dict(w=16, a0=0, a=65535, b0=0, b=65535)
    g = P.Generator(**p, seed=1, n_streams=1, n_per_stream=2)
    M = float(65535 ** 2)
    x2 = torch.arange(65536, dtype=torch.int64, device="cuda")
    for lo in range(1, 65535, 4096):
        x1 = torch.arange(lo, min(lo + 4096, 65535), dtype=torch.int64, device="cuda")
        X1, X2 = torch.meshgrid(x1, x2, indexing="ij")
        z = g.map(X1.reshape(-1).to(torch.int32), X2.reshape(-1).to(torch.int32))
        j = (X1 * 65536 + X2 - 65535).reshape(-1).to(torch.float64)
        assert torch.equal(z.view(torch.int64), (j / torch.full_like(j, M)).view(torch.int64))


def test_map_w32_edges_and_random(orc):
    p = W.FULL32
    g = P.Generator(**p, seed=1, n_streams=1, n_per_stream=2)
    e1, e2 = W.edge_pairs(32, 32, span=24)
    r1, r2 = W.random_pairs(11, 1 << 20, 32, 32)
    x1 = np.concatenate([e1, r1, np.full(4096, 2**32 - 2, np.uint32)])
    x2 = np.concatenate([e2, r2, (np.arange(4096, dtype=np.uint64) + 2**32 - 4096).astype(np.uint32)])
    z = g.map(torch.from_numpy(x1.view(np.int32)).cuda(), torch.from_numpy(x2.view(np.int32)).cuda())
    torch.cuda.synchronize()
    assert_same(z, orc.map_pairs(p, x1, x2))
    assert bool((z < 1.0).all())


@pytest.mark.parametrize("par", [W.FULL32, W.ASYM, W.BYTE8,
                                 dict(w=27, a0=0, a=2**27 - 1, b0=0, b=2**27 - 1),
                                 dict(w=32, a0=1000, a=2**31 + 7, b0=0, b=2**16 - 1)])
def test_fast_division_equals_ieee(par):
    """R10 on the GPU: reciprocal + 2 FMA quotient == __ddiv_rn on 2^34 sampled numerators."""
    g = P.Generator(**par, seed=1, n_streams=1, n_per_stream=2)
    mism = torch.zeros(1, dtype=torch.int64, device="cuda")
    P.prngd_debug_div_check(g.handle, 1 << 34, 0xC0FFEE, mism)
    torch.cuda.synchronize()
    assert mism.item() == 0


# ------------------------------------------------------------------ fused consumer (S7)

@pytest.mark.parametrize("flags", STORES_AVAILABLE)
@pytest.mark.parametrize("write", [False, True])
@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_consume_matches_oracle(orc, name, write, flags):
    if flags and not write:
        pytest.skip("store flags only matter when outputs are written")
    p = W.config(name, flags=flags)
    g = P.Generator(**p)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda") if write else None
    _, hist, pw, cnt = g.generate_consume(out)
    torch.cuda.synchronize()
    assert g.last_launches == 3  # optimistic consume, exact pass (idle here), finalize
    r = orc.generate(p, want_out=write, want_stats=True)
    assert np.array_equal(hist.cpu().numpy(), r["hist"])
    assert cnt.item() == r["count"] == p["n_streams"] * p["n_per_stream"]
    assert np.allclose(pw.cpu().numpy(), r["pow"], rtol=1e-12, atol=0)
    if write:
        assert_same(out, r["out"])


def test_consume_accumulates_across_shards(orc):
    p = W.config("cfg4", n_streams=4096, n_per_stream=256)
    hist = torch.zeros(65536, dtype=torch.int64, device="cuda")
    pw = torch.zeros(4, dtype=torch.float64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for r in range(3):
        P.Generator(**W.shard(p, r, 3)).generate_consume(None, hist, pw, cnt)
    torch.cuda.synchronize()
    ref = orc.generate(p, want_out=False, want_stats=True)
    assert np.array_equal(hist.cpu().numpy(), ref["hist"]) and cnt.item() == ref["count"]
    assert np.allclose(pw.cpu().numpy(), ref["pow"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("exact", [False, True])
def test_consume_packed_counter_carries(exact):
    """w=1, [0;2] x [0;1]: every output is 1/3 or 2/3, so two bins (one low, one high field of a
    packed word) receive ~2^27 counts -- thousands of 16-bit carries per CTA.  The histogram must
    equal the counts of the written outputs (torch bincount, independent of the consumer).
    Default flags: the optimistic adds wrap, the CTA check raises the overflow flag and the exact
    pass recomputes the histogram; EXACT_HIST: carry tracking from the start."""
    p = dict(w=1, a0=0, a=2, b0=0, b=1, seed=5, n_streams=4096, n_per_stream=65536,
             flags=P.PRNGD_FLAG_EXACT_HIST if exact else 0)
    g = P.Generator(**p)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    _, hist, pw, cnt = g.generate_consume(out)
    torch.cuda.synchronize()
    b = torch.floor(out.view(-1) * 65536.0).to(torch.int64)
    ref = torch.bincount(b, minlength=65536)
    assert torch.equal(hist, ref)
    assert cnt.item() == 4096 * 65536
    nz = torch.nonzero(ref).view(-1).tolist()
    assert nz == [21845, 43690]
    assert ref.max().item() > 2 * 148 * 65536  # carries certainly happened
    assert g.last_launches == (2 if exact else 3)
    # a second call on the same handle: the overflow flag was reset by the first call's finalize
    _, hist2, _, _ = g.generate_consume(out)
    torch.cuda.synchronize()
    assert torch.equal(hist2, ref)


def test_consume_exact_hist_flag_matches_oracle(orc):
    p = W.config("cfg2", flags=P.PRNGD_FLAG_EXACT_HIST)
    g = P.Generator(**p)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    _, hist, pw, cnt = g.generate_consume(out)
    torch.cuda.synchronize()
    assert g.last_launches == 2
    r = orc.generate(p, want_stats=True)
    assert np.array_equal(hist.cpu().numpy(), r["hist"]) and cnt.item() == r["count"]
    assert np.allclose(pw.cpu().numpy(), r["pow"], rtol=1e-12, atol=0)
    assert_same(out, r["out"])


def test_cfg4_histogram_full_size_consistent():
    """cfg4 write + histogram in one fused call at full size: histogram == bincount of the
    outputs it wrote, count == 2^32."""
    p = W.CONFIGS["cfg4"]
    g = P.Generator(**p)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    _, hist, pw, cnt = g.generate_consume(out)
    torch.cuda.synchronize()
    ref = torch.zeros(65536, dtype=torch.int64, device="cuda")
    flat = out.view(-1)
    for lo in range(0, flat.numel(), 1 << 28):
        ref += torch.bincount(torch.floor(flat[lo:lo + (1 << 28)] * 65536.0).to(torch.int64),
                              minlength=65536)
    assert torch.equal(hist, ref)
    assert cnt.item() == 2**32
    del out, flat
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ NEXT-1 / NEXT-2 variants

VARIANTS = [(k, o) for k in (4, 5, 6) for o in (False, True)]


@pytest.mark.parametrize("kind,open_", VARIANTS)
@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_mappings_bitwise(orc, name, kind, open_):
    """Eq.(5)/(6) and the open interval 1 - z' through the whole path."""
    flags = P.MAP_FLAGS[kind] | (P.PRNGD_FLAG_OPEN if open_ else 0)
    p = W.config(name, n_streams=512, n_per_stream=256)
    _, out = gen(p, flags=flags)
    ref = orc.generate(p, kind=kind, open_interval=open_)["out"]
    assert_same(out, ref)
    if open_:
        assert bool((out > 0).all()) and bool((out <= 1).all())
    else:
        assert bool((out >= 0).all()) and bool((out < 1).all())


@pytest.mark.parametrize("kind,open_", [v for v in VARIANTS if v != (4, False)])
@pytest.mark.parametrize("name,ns,nps", [("cfg3", 300, 517), ("cfg2", 97, 1030), ("w27", 64, 640)])
def test_mappings_static_row_kernel(orc, name, ns, nps, kind, open_):
    """Compile-time mapping kernels (MODE >= 16) of the bulk ROW path: Eq.(5)/(6)
    and the open interval, several tiles and a ragged tail, bitwise."""
    flags = P.MAP_FLAGS[kind] | (P.PRNGD_FLAG_OPEN if open_ else 0) | P.STORE_FLAGS["row"]
    if name == "w27":  # w >= 27: the R11 clamp is live; narrower accept band
        if kind == 6:
            pytest.skip("Eq.(6) needs the full range (P:150-153)")
        p = dict(w=27, a0=5, a=2**27 - 3, b0=0, b=2**27 - 1, seed=77, stream_begin=2**40 + 3,
                 n_streams=ns, n_per_stream=nps)
    else:
        p = W.config(name, n_streams=ns, n_per_stream=nps, stream_begin=2**40 + 3)
    _, out = gen(p, flags=flags)
    assert_same(out, orc.generate(p, kind=kind, open_interval=open_)["out"])


@pytest.mark.parametrize("kind,open_", VARIANTS)
def test_mappings_exhaustive_w8(orc, kind, open_):
    flags = P.MAP_FLAGS[kind] | (P.PRNGD_FLAG_OPEN if open_ else 0)
    g = P.Generator(**W.BYTE8, seed=1, n_streams=1, n_per_stream=2, flags=flags)
    x1, x2 = np.meshgrid(np.arange(1, 255, dtype=np.uint32), np.arange(256, dtype=np.uint32),
                         indexing="ij")
    z = g.map(torch.from_numpy(x1.ravel()).cuda(), torch.from_numpy(x2.ravel()).cuda())
    torch.cuda.synchronize()
    assert_same(z, orc.map_kind(W.BYTE8, kind, x1.ravel(), x2.ravel(), open_interval=open_))


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_alg1_consumption_bitwise(orc, name):
    p = W.config(name, n_streams=512, n_per_stream=256, flags=P.PRNGD_FLAG_ALG1)
    g, out = gen(p)
    ref = orc.generate(p, alg1=True, want_pidx=True, want_consumed=True)
    assert_same(out, ref["out"])
    pidx, cons = g.pairs()
    torch.cuda.synchronize()
    assert np.array_equal(pidx.cpu().numpy().view(np.uint32), ref["pidx"])
    assert np.array_equal(cons.cpu().numpy().view(np.uint64), ref["consumed"])


@pytest.mark.parametrize("kind", [5, 4])
def test_open_interval_histogram_top_bin(orc, kind):
    """R18: with 1 - z' the value 1.0 (from z' = 0 in Eq.(5)) lands in bin 65535."""
    flags = P.MAP_FLAGS[kind] | P.PRNGD_FLAG_OPEN
    p = W.config("cfg2", n_streams=1024, n_per_stream=512, flags=flags)
    g = P.Generator(**p)
    _, hist, pw, cnt = g.generate_consume()
    torch.cuda.synchronize()
    ref = orc.generate(p, kind=kind, open_interval=True, want_out=False, want_stats=True)
    assert np.array_equal(hist.cpu().numpy(), ref["hist"]) and cnt.item() == ref["count"]
    assert np.allclose(pw.cpu().numpy(), ref["pow"], rtol=1e-12, atol=0)


# ------------------------------------------------------------------ NEXT-3 jump-ahead kernel

@pytest.mark.parametrize("jump", [P.PRNGD_FLAG_JUMP, P.PRNGD_FLAG_NO_JUMP])
@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_jump_and_sequential_kernels_bitwise(orc, name, jump):
    p = W.config(name, flags=jump)
    _, out = gen(p)
    assert_same(out, orc.generate(p)["out"])


@pytest.mark.parametrize("ns,nps", [(1, 1), (3, 5), (33, 1000), (5, 2049), (100, 4096 + 7)])
@pytest.mark.parametrize("base", ["cfg1", "cfg2", "cfg4"])
def test_jump_ragged(orc, base, ns, nps):
    p = W.config(base, n_streams=ns, n_per_stream=nps, stream_begin=777, flags=P.PRNGD_FLAG_JUMP)
    _, out = gen(p)
    assert_same(out, orc.generate(p)["out"])


@pytest.mark.parametrize("kind,open_", [(5, False), (6, True), (4, True)])
def test_jump_with_mappings(orc, kind, open_):
    flags = P.PRNGD_FLAG_JUMP | P.MAP_FLAGS[kind] | (P.PRNGD_FLAG_OPEN if open_ else 0)
    p = W.config("cfg2", n_streams=64, n_per_stream=3000, flags=flags)
    _, out = gen(p)
    assert_same(out, orc.generate(p, kind=kind, open_interval=open_)["out"])


def test_jump_general_ranges(orc):
    for par in [dict(w=12, a0=0, a=100, b0=0, b=63), dict(w=1, a0=0, a=2, b0=0, b=1),
                dict(w=32, a0=1000, a=2**31 + 7, b0=0, b=2**16 - 1)]:
        p = dict(par, seed=9, n_streams=37, n_per_stream=2500, flags=P.PRNGD_FLAG_JUMP)
        _, out = gen(p)
        assert_same(out, orc.generate(p)["out"])


@pytest.mark.parametrize("par", [dict(w=8, a0=0, a=255, b0=0, b=255),
                                 dict(w=8, a0=17, a=200, b0=0, b=255),
                                 dict(w=8, a0=0, a=128, b0=0, b=255),
                                 dict(w=16, a0=0, a=65535, b0=0, b=65535),
                                 dict(w=16, a0=999, a=40000, b0=0, b=65535)])
@pytest.mark.parametrize("nps", [700, 1500, 701, 1025])
def test_jump_narrow_modes(orc, par, nps):
    """w = 8 / 16 with both draws at full width (sh1 = sh2 = 32 - w) take the narrow jump
    kernel (pair values compacted, Eq.(4) in the copy-out), 17- and 33-pair rounds; narrow
    bands make rejection frequent; odd rows start rounds at odd elements (the one-output head
    and tail of the paired copy-out)."""
    p = dict(par, seed=5, n_streams=45, n_per_stream=nps, stream_begin=3, flags=P.PRNGD_FLAG_JUMP)
    _, out = gen(p)
    assert_same(out, orc.generate(p)["out"])


# ------------------------------------------------------------------ NEXT-2 MRG32k3a base generator

@pytest.mark.parametrize("par", [dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1),
                                 dict(w=31, a0=0, a=2**31 - 1, b0=0, b=2**31 - 1),
                                 dict(w=16, a0=3, a=40000, b0=0, b=2**12 - 1),
                                 dict(w=32, a0=0, a=2**31 - 1, b0=0, b=2**31 - 1)])
@pytest.mark.parametrize("kind", [4, 5])
def test_mrg32k3a_bitwise(orc, par, kind):
    p = dict(par, seed=11, n_streams=300, n_per_stream=130,
             flags=P.PRNGD_FLAG_MRG32K3A | P.MAP_FLAGS[kind], mrg=True)
    _, out = gen(p)
    assert_same(out, orc.generate(p, kind=kind)["out"])


def test_mrg32k3a_generate_host(orc):
    """prngd_generate_host on the MRG32k3a kernel: several staging chunks (streams of 96 KiB)."""
    p = dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1, seed=5, n_streams=5000,
             n_per_stream=12288, flags=P.PRNGD_FLAG_MRG32K3A, mrg=True)
    g = P.Generator(**p)
    host = g.generate_host().numpy()
    dev = g.generate()
    torch.cuda.synchronize()
    assert np.array_equal(host.view(np.int64), dev.cpu().numpy().view(np.int64))
    rows = [0, 1, 2719, 2720, 4999]  # 256 MiB chunks: 2720 rows (whole warp tasks)
    for r in rows:
        ref = orc.generate(p, stream_begin=r, n_streams=1)["out"]
        assert np.array_equal(host[r].view(np.int64), ref.ravel().view(np.int64))


def _mrg_stats_match(g, p, out=None):
    """Histogram and count against the oracle's; the power sums (R16, relative 1e-12) against
    pairwise (numpy) sums of the oracle's outputs, taken over 2048-stream pieces: at 10^7-10^8
    outputs the oracle's own sequential sums drift by ~1e-12 relative themselves."""
    _, hist, pw, cnt = g.generate_consume(out)
    torch.cuda.synchronize()
    h = np.zeros(65536, dtype=np.int64)
    c = 0
    parts = []
    for s0 in range(0, p["n_streams"], 2048):
        ns = min(2048, p["n_streams"] - s0)
        r = orc_mod().generate(p, stream_begin=p.get("stream_begin", 0) + s0, n_streams=ns,
                               want_out=True, want_stats=True)
        h += r["hist"]
        c += r["count"]
        z = r["out"].ravel()
        z2 = z * z
        parts.append([z.sum(), z2.sum(), (z2 * z).sum(), (z2 * z2).sum()])
        if out is not None:
            got = out[s0:s0 + ns].cpu().numpy()
            assert np.array_equal(got.view(np.int64), r["out"].view(np.int64))
    assert np.array_equal(hist.cpu().numpy(), h)
    assert cnt.item() == c == p["n_streams"] * p["n_per_stream"]
    assert np.allclose(pw.cpu().numpy(), np.array(parts).sum(axis=0), rtol=1e-12, atol=0)


def orc_mod():
    import oracle
    return oracle


@pytest.mark.parametrize("alg1", [False, True])
@pytest.mark.parametrize("par", [dict(w=14, a0=0, a=2**14 - 1, b0=0, b=2**14 - 1),
                                 dict(w=17, a0=3, a=2**17 - 2, b0=0, b=2**9 - 1)])
def test_mrg32k3a_batch_band_test(orc, par, alg1):
    """Per-batch band test (SPECB: fewer than 1 in 4096 x1 out of band): 1/8192 .. 1/26000 of the
    x1 fall outside, so ~2-6% of the warp batches take the ring compaction and refill."""
    p = dict(par, seed=17, n_streams=400, n_per_stream=2050, alg1=alg1, mrg=True,
             flags=P.PRNGD_FLAG_MRG32K3A | (P.PRNGD_FLAG_ALG1 if alg1 else 0))
    _, out = gen(p)
    assert_same(out, orc.generate(p)["out"])


def test_mrg32k3a_alg1_bitwise(orc):
    """Alg. 1 consumption on MRG32k3a: a narrow band (most x1 redrawn) and a wide one."""
    for par in (dict(w=16, a0=3000, a=3400, b0=0, b=2**16 - 1),
                dict(w=26, a0=5, a=2**26 - 3, b0=0, b=2**20 - 1)):
        p = dict(par, seed=13, n_streams=333, n_per_stream=258, alg1=True, mrg=True,
                 flags=P.PRNGD_FLAG_MRG32K3A | P.PRNGD_FLAG_ALG1)
        _, out = gen(p)
        assert_same(out, orc.generate(p)["out"])
        g = P.Generator(**p)
        _mrg_stats_match(g, p)


@pytest.mark.parametrize("alg1", [False, True])
@pytest.mark.parametrize("seed,stream,draw,comp", [(1, 7790325, 1190, 1), (1, 16147924, 918, 2),
                                                   (1, 19033657, 1147, 2), (1, 33099832, 1992, 1)])
def test_mrg32k3a_floor_edge(seed, stream, draw, comp, alg1):
    """PRNGD_MRG_FLOOR's one edge: a component value that is exactly 0 with the sign of p for
    which the GPU's floor is one low, so the kernel carries r = m (= 0 mod m) into the next
    draws and the combination (tests/test_mrg_floor_reduction.py pins that these streams hit
    it, from the oracle).  Outputs and fused statistics bit for bit against the oracle, with the
    event inside the rows (draw <= 1992 ~ output 980 of 1100)."""
    flags = P.PRNGD_FLAG_MRG32K3A | (P.PRNGD_FLAG_ALG1 if alg1 else 0)
    p = dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1, seed=seed, stream_begin=stream - 3,
             n_streams=7, n_per_stream=1100, flags=flags, mrg=True, alg1=alg1)
    _, out = gen(p)
    ref = orc_mod().generate(p)["out"]
    assert_same(out, ref)
    g = P.Generator(**p)
    _mrg_stats_match(g, p, out=torch.empty_like(out))


@pytest.mark.parametrize("kind", [4, 5])
def test_mrg32k3a_generate_consume(kind):
    """S7 fused into the MRG32k3a generator (consume_mrg_kernel): outputs written through the
    in-ring staging, histogram / moments / count; ragged rows and a ragged last batch."""
    p = dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1, seed=9, n_streams=700, n_per_stream=1030,
             flags=P.PRNGD_FLAG_MRG32K3A | P.MAP_FLAGS[kind], mrg=True, map=kind)
    g = P.Generator(**p)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    _mrg_stats_match(g, p, out)
    assert g.last_launches == 3  # fused pass, exact pass (returns at once), finalize


@pytest.mark.parametrize("shape,offset", [((45, 77), 1), ((3, 64), 0), ((5000, 18), 0),
                                          ((33, 1), 0)])
def test_mrg32k3a_fused_consume_shapes(orc, shape, offset):
    """The fused MRG32k3a consumer on odd row lengths, an 8-byte-offset output (scalar stores
    instead of the staged tile), fewer tasks than SMs, one-output rows, with a stream offset."""
    ns, nps = shape
    p = dict(w=26, a0=7, a=2**26 - 9, b0=0, b=2**20 - 1, seed=23, stream_begin=123457,
             n_streams=ns, n_per_stream=nps, flags=P.PRNGD_FLAG_MRG32K3A, mrg=True)
    g = P.Generator(**p)
    buf = torch.full((ns * nps + 8,), -3.0, dtype=torch.float64, device="cuda")
    out = buf[offset:offset + ns * nps].view(ns, nps)
    _mrg_stats_match(g, p, out)
    assert bool((buf[:offset] == -3.0).all()) and bool((buf[offset + ns * nps:] == -3.0).all())


def test_mrg32k3a_consume_open_interval_top_bin():
    """R18 on the memory histogram: Eq.(5) with 1 - z' reaches 1.0, which lands in bin 65535."""
    p = dict(w=8, a0=0, a=255, b0=0, b=255, seed=31, n_streams=4096, n_per_stream=258, mrg=True,
             map=5, open=True,
             flags=P.PRNGD_FLAG_MRG32K3A | P.MAP_FLAGS[5] | P.PRNGD_FLAG_OPEN)
    g = P.Generator(**p)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    _mrg_stats_match(g, p, out)
    assert bool((out == 1.0).any())


def test_mrg32k3a_consume_only_long_rows():
    """Consume-only (no output buffer) on long rows: the fused kernel keeps nothing but the
    statistics, whatever the size (no staging chunks)."""
    p = dict(w=26, a0=5, a=2**26 - 3, b0=0, b=2**20 - 1, seed=3, n_streams=11500,
             n_per_stream=12288, flags=P.PRNGD_FLAG_MRG32K3A, mrg=True)
    g = P.Generator(**p)
    _mrg_stats_match(g, p)
    assert g.last_launches == 3


def test_mrg32k3a_consume_counter_wrap():
    """8 distinct values over 2^26.3 outputs: every CTA's 16-bit fields wrap, the exact pass
    (the fused kernel again, with carry-tracking adds) must take over."""
    p = dict(w=2, a0=0, a=3, b0=0, b=3, seed=4, n_streams=8192, n_per_stream=10240,
             flags=P.PRNGD_FLAG_MRG32K3A, mrg=True)
    g = P.Generator(**p)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    _mrg_stats_match(g, p, out)
    del out
    torch.cuda.empty_cache()


def test_mrg32k3a_unsupported_calls():
    p = dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1, seed=1, n_streams=32, n_per_stream=64,
             flags=P.PRNGD_FLAG_MRG32K3A)
    g = P.Generator(**p)
    with pytest.raises(P.PrngdError):
        g.raw(4)


# ------------------------------------------------------------------ guard bands (no sanitizer here)

GUARD = 4096  # doubles of sentinel before and after the output


def _guarded(shape):
    n = shape[0] * shape[1]
    buf = torch.full((n + 2 * GUARD,), -3.25, dtype=torch.float64, device="cuda")
    return buf, buf[GUARD:GUARD + n].view(shape)


def _guards_intact(buf, n):
    return bool((buf[:GUARD] == -3.25).all()) and bool((buf[GUARD + n:] == -3.25).all())


@pytest.mark.parametrize("flags", STORES_AVAILABLE +
                         [P.PRNGD_FLAG_JUMP, P.PRNGD_FLAG_MAP_EQ6 | P.PRNGD_FLAG_OPEN])
@pytest.mark.parametrize("ns,nps", [(45, 70), (31, 1030), (1, 6)])
def test_guard_bands_generate(orc, flags, ns, nps):
    p = W.config("cfg1", n_streams=ns, n_per_stream=nps, flags=flags)
    g = P.Generator(**p)
    buf, out = _guarded(g.shape)
    g.generate(out)
    torch.cuda.synchronize()
    assert _guards_intact(buf, ns * nps)
    kind = 6 if flags & P.PRNGD_FLAG_MAP_EQ6 else 4
    assert_same(out, orc.generate(p, kind=kind, open_interval=bool(flags & P.PRNGD_FLAG_OPEN))["out"])


@pytest.mark.parametrize("offset", [0, 1])
@pytest.mark.parametrize("ns,nps", [(45, 70), (31, 1030), (1, 6), (5, 1025)])
def test_guard_bands_narrow_jump(orc, ns, nps, offset):
    """gen_jump_narrow_kernel (w = 8): sentinels on both sides, and with offset 1 an output that
    is 8- but not 16-byte aligned, so rounds start on odd elements (head / tail outputs)."""
    p = W.config("cfg2", n_streams=ns, n_per_stream=nps, flags=P.PRNGD_FLAG_JUMP)
    g = P.Generator(**p)
    assert g.info["kernel"] == 5
    n = ns * nps
    buf = torch.full((n + 2 * GUARD + 1,), -3.25, dtype=torch.float64, device="cuda")
    out = buf[GUARD + offset:GUARD + offset + n].view(ns, nps)
    g.generate(out)
    torch.cuda.synchronize()
    assert bool((buf[:GUARD + offset] == -3.25).all())
    assert bool((buf[GUARD + offset + n:] == -3.25).all())
    assert_same(out, orc.generate(p)["out"])


@pytest.mark.parametrize("flags", [P.STORE_FLAGS[n] for n in P.stores_available(
    ["row", "tma", "tile", "direct"])])
def test_guard_bands_consume(orc, flags):
    p = W.config("cfg2", n_streams=77, n_per_stream=130, flags=flags)
    g = P.Generator(**p)
    buf, out = _guarded(g.shape)
    hbuf = torch.full((65536 + 2 * GUARD,), -7, dtype=torch.int64, device="cuda")
    hist = hbuf[GUARD:GUARD + 65536]
    hist.zero_()
    g.generate_consume(out, hist)
    torch.cuda.synchronize()
    assert _guards_intact(buf, 77 * 130)
    assert bool((hbuf[:GUARD] == -7).all()) and bool((hbuf[GUARD + 65536:] == -7).all())
    ref = orc.generate(p, want_stats=True)
    assert np.array_equal(hist.cpu().numpy(), ref["hist"])
    assert_same(out, ref["out"])


def test_guard_bands_mrg(orc):
    p = dict(w=26, a0=0, a=2**26 - 1, b0=0, b=2**26 - 1, seed=2, n_streams=45, n_per_stream=70,
             flags=P.PRNGD_FLAG_MRG32K3A, mrg=True)
    g = P.Generator(**p)
    buf, out = _guarded(g.shape)
    g.generate(out)
    torch.cuda.synchronize()
    assert _guards_intact(buf, 45 * 70)
    assert_same(out, orc.generate(p)["out"])


@pytest.mark.parametrize("par", [dict(w=32, a0=2**12, a=2**32 - 1, b0=0, b=2**20 - 1),
                                 dict(w=32, a0=0, a=2**32 - 1, b0=0, b=2**31 - 1),
                                 dict(w=32, a0=5, a=2**32 - 3, b0=0, b=2**32 - 1)])
def test_w32_runtime_band_kernel(orc, par):
    """Kernel MODE 3 (w = 32, 32-bit x1 draws, runtime x2 width and accept band: cfg4's family)
    through the ROW generator and the fused consumer, with rare rejections (p ~ 1e-6) included."""
    p = dict(par, seed=21, stream_begin=5, n_streams=4096, n_per_stream=1024,
             flags=P.PRNGD_FLAG_STORE_ROW)
    _, out = gen(p)
    r = orc.generate(p, want_stats=True, want_consumed=True)
    assert_same(out, r["out"])
    g = P.Generator(**p)
    out2 = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    _, hist, pw, cnt = g.generate_consume(out2)
    torch.cuda.synchronize()
    assert_same(out2, r["out"])
    assert np.array_equal(hist.cpu().numpy(), r["hist"]) and cnt.item() == r["count"]
    assert np.allclose(pw.cpu().numpy(), r["pow"], rtol=1e-12, atol=0)
