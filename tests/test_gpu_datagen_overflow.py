"""-m gpu: (1) the device-side generator that bench.py times produces the same columns as the
host generator the parity tests feed the oracle (bit-exact for integers and uniform doubles,
<= 16 ulp for Box-Muller normals, whose log / cos come from host libm vs CUDA libdevice), at the start, in the middle and at the end of each BASELINE
config; (2) int64 overflow detection (R33): every exact overflow the oracle finds is flagged by
the GPU (PAC_E_OVERFLOW), and inputs inside the bound max|v| x rows < 2^63 are flagged by
neither."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import run_gpu

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_15023_b200 as pac  # noqa: E402


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5"])
def test_device_columns_equal_host_columns(cfg):
    w = dg.WORKLOADS[cfg]
    n = 200_003
    for row0 in (0, w.n_rows // 2 - 77, w.n_rows - n):
        h = w.host_columns(row0, n)
        d = dg.device_columns(w, row0, n)
        np.testing.assert_array_equal(d["pu"].cpu().numpy(), h["pu"])
        for a, b in zip(d["keys"], h["keys"]):
            np.testing.assert_array_equal(a.cpu().numpy(), b)
        for spec, a, b in zip(w.values, d["values"], h["values"]):
            a = a.cpu().numpy()
            if spec.kind == dg.KIND_NORMAL_F64:
                # mu + sigma * sqrt(-2 ln u1) cos(2 pi u2): host libm vs CUDA libdevice, a few ulp
                np.testing.assert_array_max_ulp(a, b, maxulp=16)
            else:
                np.testing.assert_array_equal(a, b)


def _flagged(t):
    return int(t.status.item()) == pac._lib.PAC_E_OVERFLOW


def test_exact_overflow_is_always_flagged(orc):
    ones = np.full(16, 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
    cases = [np.full(16, 2**60, dtype=np.int64),                           # 2^64: overflows
             np.array([2**62] * 2 + [-(2**62)] * 14, dtype=np.int64),       # -2^65 + 2^63: overflows
             np.array([2**63 - 1, 1] + [0] * 14, dtype=np.int64)]           # 2^63: overflows
    for iv in cases:
        g = np.zeros(len(iv), dtype=np.int32)
        aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv)]
        ref = orc.agg(ones[:len(iv)], [g], aggs)
        assert ref["overflow"]
        t, _ = run_gpu(aggs, [g], masks=ones[:len(iv)], G_cap=4)
        assert _flagged(t)


def test_no_flag_inside_the_bound(orc):
    rng = np.random.default_rng(1)
    n = 300_000
    iv = rng.integers(-(2**40), 2**40, n).astype(np.int64)   # max|v| x rows ~ 3e17 < 2^63
    g = rng.integers(0, 5, n).astype(np.int32)
    pu = rng.integers(0, 1000, n).astype(np.int64)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv)]
    ref = orc.agg(orc.pac_hash(pu, 3), [g], aggs)
    t, _ = run_gpu(aggs, [g], pu=pu, salt=3, G_cap=8)
    assert not ref["overflow"] and not _flagged(t)
