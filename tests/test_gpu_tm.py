"""-m gpu parity of k_agg_tiles_tm -- the tile kernel whose CTA accumulator table lives in Tensor
Memory (chosen for 33..~200 local slots) -- against the oracle: the C5 shape at its own capacity
(100 groups), every aggregate kind together, ragged sizes across 2048-row tiles, explicit
masks, and the A/B switch to the shared-memory kernel (PAC_NO_TM)."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import assert_tables_equal, run_gpu, workload_aggs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.mark.parametrize("n", [1_000_003, 2048 * 148 + 77])
def test_c5_shape_tmem_table(orc, n):
    w = dg.WORKLOADS["C5"]
    cols = w.host_columns(0, n)
    aggs = workload_aggs(w, cols)
    salt = 0x243F6A8885A308D3
    t, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=salt, G_cap=100)
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(cols["pu"], salt), cols["keys"], aggs))


@pytest.mark.parametrize("n", [0, 1, 2047, 2048, 2049, 70_001])
def test_all_kinds_ragged(orc, n):
    rng = np.random.default_rng(n + 5)
    pu = rng.integers(0, 3000, n).astype(np.int64)
    keys = [rng.integers(-30, 30, n).astype(np.int16)]
    iv = rng.integers(-10**9, 10**9, n).astype(np.int64)
    fv = rng.normal(0, 10, n)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv), (dg.AGG_AVG_F64, fv), (dg.AGG_MIN_F64, fv),
            (dg.AGG_MAX_F64, fv)]
    t, _ = run_gpu(aggs, keys, pu=pu, salt=11, G_cap=64)
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 11), keys, aggs))


def test_explicit_masks_and_ab_switch(orc, monkeypatch):
    rng = np.random.default_rng(9)
    n = 300_000
    masks = orc.pac_hash(rng.integers(0, 9000, n).astype(np.int64), 4)
    masks[::17] = 0
    masks[1::5] &= np.uint64(0x0000FFFF0000FFFF)
    keys = [rng.integers(0, 120, n).astype(np.int32)]
    iv = rng.integers(1, 10**6, n).astype(np.int64)
    aggs = [(dg.AGG_SUM_I64, iv), (dg.AGG_COUNT, None)]
    t, _ = run_gpu(aggs, keys, masks=masks, G_cap=128)
    got = t.to_host()
    assert_tables_equal(got, orc.agg(masks, keys, aggs))
    monkeypatch.setenv("PAC_NO_TM", "1")
    t2, _ = run_gpu(aggs, keys, masks=masks, G_cap=128)
    assert_tables_equal(t2.to_host(), got)
