"""-m gpu parity of non-finite f64 values (R30: IEEE sums; R31: MIN/MAX under
DuckDB's total order, NaN largest) on every aggregation path: the shared-memory tile kernel
(compile-time and runtime layouts), the TMEM-table kernel, the HBM tier with direct atomics,
the deferred HBM tier (records folded after the pass) and the pruned MIN/MAX kernel.  The
non-finite class of every world value is compared exactly (assert_tables_equal: NaN == NaN,
+-inf positions equal), presence K exactly -- including worlds that hold only +inf under MIN
or only -inf under MAX (present, not empty)."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import assert_tables_equal, run_gpu

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)


def _values(rng, n, frac=0.004):
    v = rng.normal(10.0, 5.0, n)
    for x in (np.nan, np.inf, -np.inf):
        v[rng.choice(n, max(1, int(frac * n)), replace=False)] = x
    v[rng.choice(n, 7, replace=False)] = -np.nan  # negative-sign NaN: the same value (R31)
    return v


def _with_special_groups(pu, g, v, base_key):
    # groups holding only NaN, only +inf, only -inf rows (a few PUs each)
    extra_g, extra_v = [], []
    for i, x in enumerate((np.nan, np.inf, -np.inf)):
        extra_g += [base_key + i] * 40
        extra_v += [x] * 40
    extra_pu = np.arange(len(extra_g), dtype=np.int64) % 9 + 10**9
    return (np.concatenate([pu, extra_pu]).astype(np.int64), np.concatenate([g, extra_g]).astype(g.dtype),
            np.concatenate([v, extra_v]))


def _case(seed, n, n_groups, dtype=np.int32):
    rng = np.random.default_rng(seed)
    pu = rng.integers(0, 5000, n).astype(np.int64)
    g = rng.integers(0, n_groups, n).astype(dtype)
    v = _values(rng, n)
    pu, g, v = _with_special_groups(pu, g, v, n_groups)
    iv = rng.integers(-1000, 1000, len(v)).astype(np.int64)
    return pu, [g], v, iv


ALL = lambda v, iv: [(dg.AGG_COUNT, None), (dg.AGG_SUM_F64, v), (dg.AGG_AVG_F64, v), (dg.AGG_MIN_F64, v),
                     (dg.AGG_MAX_F64, v), (dg.AGG_SUM_I64, iv)]


@pytest.mark.parametrize("n_groups,G_cap,fixed", [(5, 8, True), (5, 8, False), (20, 32, True)])
def test_tile_kernel_smem_table(orc, monkeypatch, n_groups, G_cap, fixed):
    if not fixed:
        monkeypatch.setenv("PAC_NO_FIXED", "1")
    pu, keys, v, iv = _case(1, 120_001, n_groups)
    aggs = ALL(v, iv)
    t, _ = run_gpu(aggs, keys, pu=pu, salt=5, G_cap=G_cap)
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 5), keys, aggs))


def test_tmem_table_kernel(orc, monkeypatch):
    monkeypatch.setenv("PAC_DEBUG", "1")
    pu, keys, v, iv = _case(2, 400_003, 97)
    aggs = ALL(v, iv)
    t, _ = run_gpu(aggs, keys, pu=pu, salt=6, G_cap=100)
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 6), keys, aggs))


@pytest.mark.parametrize("spill_rows", [0, None])
def test_hbm_tier_atomics_and_deferred_records(orc, spill_rows):
    # 20 000 groups: most rows miss a CTA-local slot (direct atomics with spill_rows = 0, the
    # deferred tier otherwise)
    pu, keys, v, iv = _case(3, 300_007, 20_000)
    aggs = ALL(v, iv)
    t, _ = run_gpu(aggs, keys, pu=pu, salt=7, G_cap=1 << 15, spill_rows=spill_rows)
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 7), keys, aggs))


@pytest.mark.parametrize("kinds", [(dg.AGG_MIN_F64,), (dg.AGG_MAX_F64,), (dg.AGG_MIN_F64, dg.AGG_MAX_F64)])
@pytest.mark.parametrize("n_groups", [50, 3000])
def test_pruned_minmax_kernel(orc, kinds, n_groups):
    # MIN/MAX-only: k_agg_minmax; presence must come from the rows (worlds holding only +inf
    # under MIN / only -inf under MAX are present)
    pu, keys, v, _ = _case(4, 500_009, n_groups)
    aggs = [(k, v) for k in kinds]
    t, _ = run_gpu(aggs, keys, pu=pu, salt=8, G_cap=4096)
    got, ref = t.to_host(), orc.agg(orc.pac_hash(pu, 8), keys, aggs)
    assert_tables_equal(got, ref)
    # the special groups are present in 32+ worlds although their values equal the sentinels
    for i in range(3):
        gi = int(np.searchsorted(ref["keys"], np.uint64((n_groups + i) ^ 0x80000000)))
        assert bin(int(got["K"][gi])).count("1") >= 32


def test_explicit_masks_nonfinite_sum_classes(orc):
    # closed forms with all-ones masks: every world sums the whole group
    n = 6000
    rng = np.random.default_rng(5)
    g = (np.arange(n) % 6).astype(np.int8)
    v = rng.random(n)
    v[g == 1] = np.where(rng.random((g == 1).sum()) < 0.01, np.inf, v[g == 1])
    v[np.flatnonzero(g == 2)[:2]] = [np.inf, -np.inf]
    v[np.flatnonzero(g == 3)[5]] = np.nan
    v[np.flatnonzero(g == 4)[7]] = -np.inf
    masks = np.full(n, 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_F64, v), (dg.AGG_MIN_F64, v), (dg.AGG_MAX_F64, v)]
    t, _ = run_gpu(aggs, [g], masks=masks, G_cap=8)
    got = t.to_host()
    assert_tables_equal(got, orc.agg(masks, [g], aggs))
    s = got["world"][1]
    assert np.all(np.isfinite(s[0])) and np.all(s[1] == np.inf) and np.all(np.isnan(s[2]))
    assert np.all(np.isnan(s[3])) and np.all(s[4] == -np.inf)
    assert np.all(np.isnan(got["world"][3][3]))  # MAX of a group with a NaN is NaN (R31)
    assert np.all(np.isfinite(got["world"][2][3]))  # ... its MIN ignores it
