"""-m gpu parity of the small-table path (G_cap <= 8: the compile-time-layout instance of
k_agg_tiles, 8 local slots) against the CPU oracle, element by element on the same seeded
inputs: BASELINE configs C1/C2 at sizes that span many CTAs and a ragged tail, plus the edge
cases -- straggler queues, partial runs, int64 values beyond the int32 tables, non-finite f64
values, MIN/MAX next to COUNT, explicit (reduced / zero) masks, capacity overflow, and the A/B
switch to the runtime-layout instance (PAC_NO_FIXED)."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import assert_tables_equal, run_gpu, workload_aggs

pytestmark = pytest.mark.gpu


torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

SALT = 0x243F6A8885A308D3


@pytest.mark.parametrize("cfg,n,G_cap", [("C1", 100_003, 1), ("C1", 1_000_000, 1), ("C2", 200_017, 8),
                                         ("C2", 2_000_000, 8), ("C2", 300_001, 6)])
def test_workloads_low_cardinality(orc, cfg, n, G_cap):
    w = dg.WORKLOADS[cfg]
    cols = w.host_columns(0, n)
    aggs = workload_aggs(w, cols)
    t, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=SALT, G_cap=G_cap)
    ref = orc.agg(orc.pac_hash(cols["pu"], SALT), cols["keys"], aggs)
    assert_tables_equal(t.to_host(), ref)


@pytest.mark.parametrize("n", [0, 1, 2, 31, 32, 33, 47, 48, 63, 64, 65, 1000, 8191, 8193, 77_777])
def test_ragged_sizes_all_aggregates(orc, n):
    rng = np.random.default_rng(100 + n)
    pu = rng.integers(0, 700, n).astype(np.int64)
    keys = [rng.integers(-2, 3, n).astype(np.int16)]
    iv = rng.integers(-10**6, 10**6, n).astype(np.int64)
    fv = rng.normal(5, 2, n)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv), (dg.AGG_AVG_F64, fv), (dg.AGG_SUM_F64, fv),
            (dg.AGG_MIN_F64, fv), (dg.AGG_MAX_F64, fv)]
    t, _ = run_gpu(aggs, keys, pu=pu, salt=17, G_cap=8)
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 17), keys, aggs))


def test_big_int64_and_nonfinite_values(orc):
    # |v| >= 2^26 in some runs (int64 tables) and +-inf / nan in some (select-built f64 tables)
    rng = np.random.default_rng(5)
    n = 150_000
    pu = rng.integers(0, 3000, n).astype(np.int64)
    keys = [rng.integers(0, 4, n).astype(np.int8)]
    iv = rng.integers(-1000, 1000, n).astype(np.int64)
    iv[rng.integers(0, n, 40)] = rng.integers(-(2**40), 2**40, 40)
    fv = rng.random(n)
    fv[rng.integers(0, n, 5)] = np.inf
    fv[rng.integers(0, n, 3)] = -np.inf
    aggs = [(dg.AGG_SUM_I64, iv), (dg.AGG_COUNT, None), (dg.AGG_SUM_F64, fv)]
    t, _ = run_gpu(aggs, keys, pu=pu, salt=3, G_cap=4)
    got, ref = t.to_host(), orc.agg(orc.pac_hash(pu, 3), keys, aggs)
    # R30: the non-finite class of every world sum is exact (NaN / +inf / -inf positions
    # equal), finite worlds agree to 1e-9
    assert_tables_equal(got, ref)
    assert (~np.isfinite(ref["world"][2])).any() and np.isfinite(ref["world"][2]).any()


def test_explicit_masks_with_zeros(orc):
    rng = np.random.default_rng(9)
    n = 50_000
    masks = orc.pac_hash(rng.integers(0, 400, n).astype(np.int64), 21)
    masks[::5] &= np.uint64(0x0F0F0F0F0F0F0F0F)
    masks[::9] = 0
    keys = [rng.integers(0, 7, n).astype(np.int32)]
    iv = rng.integers(1, 100, n).astype(np.int64)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv)]
    t, _ = run_gpu(aggs, keys, masks=masks, G_cap=7)
    assert_tables_equal(t.to_host(), orc.agg(masks, keys, aggs))


def test_capacity_exceeded_reported():
    import paper_2603_15023_b200 as pac
    from gpu_helpers import to_dev
    n = 20_000
    keys = [to_dev(np.arange(n, dtype=np.int64) % 12)]
    pu = to_dev(np.arange(n, dtype=np.int64))
    ag = pac.Aggregator([pac.COUNT], 8)
    t = ag([None], keys, pu_key=pu, salt=1)
    with pytest.raises(pac.PacError) as e:
        t.check()
    assert e.value.rc == 2


def test_fixed_and_runtime_layouts_agree(orc, monkeypatch):
    w = dg.WORKLOADS["C2"]
    cols = w.host_columns(0, 400_000)
    aggs = workload_aggs(w, cols)
    t1, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=SALT, G_cap=8)
    a = t1.to_host()
    monkeypatch.setenv("PAC_NO_FIXED", "1")
    t2, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=SALT, G_cap=8)
    assert_tables_equal(a, t2.to_host())
