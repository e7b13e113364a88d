"""prngd_get_info's kernel id names the kernel a generate call actually launches (bench.py labels
its roofline with it): the CUDA kernel names are read back with torch.profiler (CUPTI) around
one generate call of each BASELINE shape's default (AUTO) plan and of the forced plans."""
import pytest

torch = pytest.importorskip("torch")

from paper_1401_8230_b200 import prngd as P  # noqa: E402
from paper_1401_8230_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu

NAMES = {0: "gen_kernel", 1: "gen_seg_kernel", 2: "gen_jump_kernel", 3: "gen_mrg_kernel",
         5: "gen_jump_narrow_kernel"}


def _launched(g, out):
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g.generate(out)
        torch.cuda.synchronize()
    return [e.name for e in prof.events() if "prngd::" in e.name]


@pytest.mark.parametrize("name,over,kernel", [
    ("cfg1", {}, 1),                                     # few streams: SEG
    ("cfg2", {}, 5),
    ("cfg3", dict(n_streams=32768), 0),             # >= 16384 streams: bulk ROW
    ("cfg4", dict(n_streams=32768), 0),
    ("mrg26", dict(n_streams=4096, flags=P.PRNGD_FLAG_MRG32K3A), 3),
    ("cfg1", dict(flags=P.PRNGD_FLAG_JUMP), 2),               # w = 32: the generic jump kernel
    ("cfg2", dict(n_per_stream=700, flags=P.PRNGD_FLAG_JUMP), 5),
])
def test_reported_kernel_is_launched(name, over, kernel):
    g = P.Generator(**W.config(name, **over))
    assert g.info["kernel"] == kernel, g.info
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    g.generate(out)  # warm-up (tables, attributes)
    names = _launched(g, out)
    assert len(names) == 1, names
    base = names[0].split("<")[0].split("(")[0].replace("void ", "").replace("prngd::", "").strip()
    assert base == NAMES[kernel], (names, g.info)
