"""-m gpu run-to-run reproducibility (R34): the same call twice on the same
inputs.  Integer results -- group keys, rows, K, per-world counts, int64 sums -- and MIN/MAX are
byte-identical on every path (exact arithmetic in any order; extremes are order-free).  f64 world
sums are accumulated with atomics from CTAs / warps in scheduling order, so they may differ in the
last bits between runs: they must agree to far inside R16 (1e-12 relative here), and so must the
releases computed from them.  NULL flags depend only on K and the Philox stream: identical."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import run_gpu

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_15023_b200 as pac  # noqa: E402

G_CAP = {"C1": 1, "C2": 8, "C3": 1 << 20, "C4": 1024, "C5": 100}


@pytest.mark.parametrize("cfg,n", [("C1", 1_000_000), ("C2", 3_000_000), ("C3", 2_000_000), ("C4", 4_000_000),
                                   ("C5", 4_000_000)])
def test_run_twice(cfg, n):
    w = dg.WORKLOADS[cfg]
    cols = w.host_columns(0, n)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    outs = []
    for _ in range(2):
        t, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=77, G_cap=G_CAP[cfg])
        s = pac.Session(4242, w.budget)
        rel, isn, flags, _ = pac.finalize(s, t, 0)
        outs.append((t.to_host(), rel.cpu().numpy(), isn.cpu().numpy(), flags.cpu().numpy()))
    (a, ra, na, fa), (b, rb, nb, fb) = outs
    for f in ("keys", "rows", "K"):
        assert a[f].tobytes() == b[f].tobytes(), f
    if a["count"] is not None:
        assert a["count"].tobytes() == b["count"].tobytes()
    for k, x, y in zip(a["kinds"], a["world"], b["world"]):
        if x is None:
            continue
        if k in (dg.AGG_SUM_I64, dg.AGG_MIN_F64, dg.AGG_MAX_F64):
            assert x.tobytes() == y.tobytes(), k
        else:
            np.testing.assert_allclose(x, y, rtol=1e-12, atol=0)
    G = a["G"]
    np.testing.assert_array_equal(na[:G], nb[:G])
    np.testing.assert_array_equal(fa[:G], fb[:G])
    ok = na[:G] == 0
    np.testing.assert_allclose(ra[:G][ok], rb[:G][ok], rtol=1e-9)


def test_mask_is_deterministic():
    keys = torch.arange(-5_000_000, 5_000_000, dtype=torch.int64, device="cuda") * 7919
    a = pac.mask(keys, 123)
    b = pac.mask(keys, 123)
    assert torch.equal(a, b)
