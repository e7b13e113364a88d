"""GPU parity of the jump-ahead store paths:

* SEG (gen_seg_kernel): n_per_stream / 128 lanes share a row, lane j starts at pair 128 j of its
  stream by GF(2) jump-ahead, and a warp vote sends any warp that met a rejected x1 (or
  x1 = a - 1, the R11 clamp row) to the exact rewrite (seg_exact);
* SEGC (gen_segc_kernel): a CTA of 8 warps owns 32 rows, warp j column block j (pairs
  j * nps / 8 ...), flagged rows rewritten exactly after the task barrier (segc_exact).

The rejection cases use widths where rejection is rare enough for the speculative path
(prngd_info.speculative) yet frequent at test sizes: w = 17 (p_rej = 2^-16 per pair) and
w = 20 (2^-19), so many warps take the exact rewrite, including rows with several rejections
and rejections in the last segment (the tail continues past pair n_per_stream).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1401_8230_b200 import prngd as P  # noqa: E402
from paper_1401_8230_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu

SEG_KERNEL = 1
SEGC_KERNEL = 4


@pytest.fixture(scope="module", autouse=True)
def gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    P.lib()
    yield


def bits(a):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


# SEGC is an A/B path of the variant build (-DPRNGD_AB_STORES=1); the product library has SEG
PATHS = P.stores_available(["seg", "segc"])


def assert_same(gpu_out, ref):
    gb, rb = bits(gpu_out).ravel(), bits(ref).ravel()
    bad = np.nonzero(gb != rb)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}"


def full(w):
    return dict(w=w, a0=0, a=2**w - 1, b0=0, b=2**w - 1)


def run(p, path="seg"):
    flag = P.PRNGD_FLAG_STORE_SEG if path == "seg" else P.PRNGD_FLAG_STORE_SEGC
    p["flags"] = p.get("flags", 0) | flag  # else AUTO may pick another kernel
    g = P.Generator(**p)
    assert g.info["kernel"] == (SEG_KERNEL if path == "seg" else SEGC_KERNEL), g.info
    out = g.generate()
    torch.cuda.synchronize()
    return g, out


def eligible(path, nps):
    return (nps % 128 == 0 and nps // 128 in (1, 2, 4, 8, 16, 32)) if path == "seg" \
        else nps % 512 == 0


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("nps", [128, 256, 512, 1024, 1536, 2048, 4096, 8192])
@pytest.mark.parametrize("ns", [1, 37, 1000])
def test_seg_full32_shapes(orc, nps, ns, path):
    if not eligible(path, nps):
        pytest.skip("shape not eligible for this path")
    p = dict(W.FULL32, seed=W.SEED, stream_begin=4242, n_streams=ns, n_per_stream=nps)
    _, out = run(p, path)
    assert_same(out, orc.generate(p)["out"])


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("w", [17, 20])
@pytest.mark.parametrize("nps", [128, 1024, 4096])
def test_seg_rejections_exact_rewrite(orc, w, nps, path):
    if not eligible(path, nps):
        pytest.skip("shape not eligible for this path")
    ns = (1 << 22) // nps + 3      # ~4 M pairs: w = 17 -> ~128 rejections, w = 20 -> ~16
    p = dict(full(w), seed=W.SEED2, stream_begin=99, n_streams=ns, n_per_stream=nps)
    g, out = run(p, path)
    assert g.info["speculative"] == 1
    ref = orc.generate(p, want_consumed=True)
    extra = ref["consumed"].astype(np.int64) - nps
    assert (extra > 0).sum() >= 3, "the case must exercise the exact rewrite"
    assert_same(out, ref["out"])


@pytest.mark.parametrize("path", PATHS)
def test_seg_rejection_in_last_segment(orc, path):
    """Find rows (w = 17, nps = 512) whose rejections fall in the last segment / block (the
    tail draws past pair n_per_stream come from the row's last lane) and check them bitwise."""
    nps, ns = 512, 8192
    p = dict(full(17), seed=5, stream_begin=0, n_streams=ns, n_per_stream=nps)
    g, out = run(p, path)
    ref = orc.generate(p, want_pidx=True, want_consumed=True)
    pidx = ref["pidx"].reshape(ns, nps).astype(np.int64)
    last = 384 if path == "seg" else 448   # first pair of the last segment (SEG) / block (SEGC)
    late = np.nonzero((pidx[:, last - 1] == last - 1) & (ref["consumed"] > nps))[0]
    assert late.size > 0
    assert_same(out, ref["out"])


@pytest.mark.parametrize("par", [W.ASYM, dict(w=32, a0=2**12, a=2**32 - 1, b0=0, b=2**32 - 1),
                                 dict(w=24, a0=0, a=2**24 - 1, b0=0, b=2**16 - 1)])
@pytest.mark.parametrize("path", PATHS)
def test_seg_general_ranges(orc, par, path):
    p = dict(par, seed=3, stream_begin=1 << 33, n_streams=3000, n_per_stream=2048)
    _, out = run(p, path)
    assert_same(out, orc.generate(p)["out"])


@pytest.mark.parametrize("kind,open_", [(5, False), (6, False), (4, True), (6, True)])
@pytest.mark.parametrize("path", PATHS)
def test_seg_mappings(orc, kind, open_, path):
    flags = P.MAP_FLAGS[kind] | (P.PRNGD_FLAG_OPEN if open_ else 0)
    p = dict(full(20), seed=11, stream_begin=0, n_streams=2000, n_per_stream=1024, flags=flags)
    _, out = run(p, path)
    assert_same(out, orc.generate(p, kind=kind, open_interval=open_)["out"])


@pytest.mark.parametrize("path", PATHS)
def test_seg_ieee_division(orc, path):
    p = dict(full(20), seed=12, stream_begin=0, n_streams=2000, n_per_stream=1024,
             flags=P.PRNGD_FLAG_IEEE_DIV)
    _, out = run(p, path)
    assert_same(out, orc.generate(p)["out"])


@pytest.mark.parametrize("path", PATHS)
def test_seg_clamp_row_w27(orc, path):
    """w = 27: x1 = a - 1 (the only row the R11 clamp can reach, routed to the exact rewrite)
    appears with probability 2^-27 per pair, rejection 2^-26.  Over these 2^28 pairs seed 2 has
    five x1 = a - 1 outputs (asserted through the oracle's own map).  Compared bitwise in full."""
    w = 27
    p = dict(full(w), seed=2, stream_begin=0, n_streams=1 << 18, n_per_stream=1024)
    g, out = run(p, path)
    assert g.info["clamp"] == 1
    ref = orc.generate(p)["out"]
    thr = orc.map_pairs(p, np.array([2**w - 2], dtype=np.uint32), np.array([0], dtype=np.uint32))
    assert int((ref >= thr[0]).sum()) >= 3
    assert_same(out, ref)


@pytest.mark.parametrize("path,nps", [(q, n) for q, n in (("seg", 256), ("segc", 512))
                                      if q in PATHS])
def test_seg_guard_bands(orc, path, nps):
    GUARD = 4096
    flag = P.PRNGD_FLAG_STORE_SEG if path == "seg" else P.PRNGD_FLAG_STORE_SEGC
    p = dict(full(17), seed=8, stream_begin=0, n_streams=203, n_per_stream=nps, flags=flag)
    g = P.Generator(**p)
    assert g.info["kernel"] == (SEG_KERNEL if path == "seg" else SEGC_KERNEL)
    n = 203 * nps
    buf = torch.full((n + 2 * GUARD,), -3.25, dtype=torch.float64, device="cuda")
    g.generate(buf[GUARD:GUARD + n].view(203, nps))
    torch.cuda.synchronize()
    assert bool((buf[:GUARD] == -3.25).all()) and bool((buf[GUARD + n:] == -3.25).all())
    assert_same(buf[GUARD:GUARD + n], orc.generate(p)["out"])


@pytest.mark.parametrize("nps,kernel", [(1000, 0), (8192, 0), (96, 0)])
def test_seg_ineligible_shapes_fall_back(orc, nps, kernel):
    p = dict(W.FULL32, seed=2, stream_begin=0, n_streams=20000, n_per_stream=nps)
    g = P.Generator(**p)
    assert g.info["kernel"] == kernel
    out = g.generate()
    torch.cuda.synchronize()
    rows = [0, 1, 9999, 19999]
    ref = np.stack([orc.generate(p, stream_begin=r, n_streams=1)["out"][0] for r in rows])
    assert_same(out[rows], ref)


@pytest.mark.parametrize("path", PATHS)
def test_seg_generate_host_matches_device(orc, path):
    p = dict(full(17), seed=4, stream_begin=0, n_streams=70000, n_per_stream=1024)
    g, out = run(p, path)
    host = torch.empty(g.shape, dtype=torch.float64, pin_memory=True)
    P.prngd_generate_host(g.handle, host, torch.cuda.current_stream())
    assert_same(host, out)


def test_seg_multi_task_ctas_with_prefetched_jumps(orc):
    """Bulk SEG launches give each one-warp CTA 4 consecutive tasks and prefetch the next task's
    jump during the current one (n_tasks >= 148 * 12 * 16).  nps = 256 (S = 2, 16 rows per task),
    w = 20 (rejections -> exact rewrites inside multi-task CTAs), ragged last CTA; bitwise."""
    ns = 148 * 12 * 16 * 16 + 37
    p = dict(full(20), seed=13, stream_begin=5, n_streams=ns, n_per_stream=256)
    _, out = run(p)
    ref = orc.generate(p, want_consumed=True)
    assert (ref["consumed"] > 256).sum() > 50
    assert_same(out, ref["out"])


# ------------------------------------------------------------------ fused consumer, row segments

def _consume(p, flags):
    g = P.Generator(**dict(p, flags=flags))
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    _, hist, pw, cnt = g.generate_consume(out)
    torch.cuda.synchronize()
    return out, hist.cpu().numpy(), pw.cpu().numpy(), int(cnt.item())


@pytest.mark.parametrize("par", [W.FULL32,
                                 dict(w=17, a0=0, a=2**17 - 1, b0=0, b=2**17 - 1),
                                 dict(w=32, a0=2**16, a=2**32 - 1, b0=0, b=2**31 - 1),
                                 dict(w=27, a0=0, a=2**27 - 1, b0=0, b=2**27 - 1)])
@pytest.mark.parametrize("nps,ns", [(128, 70), (1024, 1000), (2048, 517), (4096, 97)])
def test_consume_row_segments(orc, par, nps, ns):
    """The fused consumer with 1 KiB row segments (run_task_seg_consume; AUTO and explicit SEG)
    and with ROW tiles: outputs, histogram, count bitwise and power sums (relative 1e-12) equal
    the oracle's.  w = 17 and the 2^-16 band on 32-bit draws reject often enough that many warps
    take the exact finish (remaining pairs counted exactly, the row's tail past pair nps, the
    outputs rewritten at their shifted positions); w = 27 has the R11 clamp row."""
    p = dict(par, seed=77, stream_begin=31337, n_streams=ns, n_per_stream=nps)
    ref = orc.generate(p, want_stats=True)
    for flags in (P.PRNGD_FLAG_STORE_AUTO, P.PRNGD_FLAG_STORE_SEG, P.PRNGD_FLAG_STORE_ROW):
        out, hist, pw, cnt = _consume(p, flags)
        assert_same(out, ref["out"])
        assert cnt == ref["count"] and np.array_equal(hist, ref["hist"]), flags
        assert np.allclose(pw, ref["pow"], rtol=1e-12, atol=0), flags


def test_consume_row_segments_misaligned_falls_back(orc):
    """An 8-byte-offset output cannot take the 16-byte row-segment flush: the consumer falls back
    to 8-byte stores with the same bits and statistics."""
    p = dict(W.FULL32, seed=5, stream_begin=0, n_streams=300, n_per_stream=1024)
    ref = orc.generate(p, want_stats=True)
    g = P.Generator(**p)
    buf = torch.full((300 * 1024 + 2,), -1.0, dtype=torch.float64, device="cuda")
    out = buf[1:1 + 300 * 1024].view(300, 1024)
    _, hist, pw, cnt = g.generate_consume(out)
    torch.cuda.synchronize()
    assert_same(out, ref["out"])
    assert np.array_equal(hist.cpu().numpy(), ref["hist"]) and int(cnt.item()) == ref["count"]
    assert float(buf[0]) == -1.0 and float(buf[-1]) == -1.0


@pytest.mark.parametrize("nps", [256, 512])
def test_consume_row_segments_high_stream_ids(orc, nps):
    """Row-segment consumer near the top of the 64-bit stream-id space (counter addressing)."""
    p = dict(W.FULL32, seed=0x0123456789ABCDEF, stream_begin=2**64 - 1000, n_streams=1000,
             n_per_stream=nps)
    ref = orc.generate(p, want_stats=True)
    out, hist, pw, cnt = _consume(p, P.PRNGD_FLAG_STORE_AUTO)
    assert_same(out, ref["out"])
    assert cnt == ref["count"] and np.array_equal(hist, ref["hist"])
    assert np.allclose(pw, ref["pow"], rtol=1e-12, atol=0)
