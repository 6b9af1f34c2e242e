"""Sort-first aggregation (sortagg.cu: radix passes on the packed key, then a streaming 64-world
fold; the default for high-cardinality COUNT / SUM / AVG tables with keys of <= 4 bytes, e.g.
BASELINE C3): element-by-element parity with the oracle -- Zipf and uniform keys, hashed pu keys
and explicit masks with zero rows (R21), one to three key columns with constant and varying bytes,
groups spanning many 2048-row chunks, singleton groups, every value-column combination, non-finite
f64 values (R30), ragged sizes, CAPACITY -- and equality with the deferred-tier path."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import assert_tables_equal, run_gpu

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_15023_b200 as pac  # noqa: E402


def _run(aggs, keys, **kw):
    pac.profile_enable(True)
    try:
        t, _ = run_gpu(aggs, keys, **kw)
        torch.cuda.synchronize()
        return t, pac.profile_last_kernel()
    finally:
        pac.profile_enable(False)


def _zipf(rng, n, groups, s=1.1):
    return np.minimum(rng.zipf(s, n), groups) - 1


@pytest.mark.parametrize("n", [1, 31, 2049, 300_017, 1_000_003])
def test_c3_shape_scrambled_int32_keys(orc, n):
    rng = np.random.default_rng(n)
    pu = rng.integers(0, max(2, n // 3), n).astype(np.int64)
    g = (_zipf(rng, n, 100_000).astype(np.int64) * 2654435761 % (2**32) - 2**31).astype(np.int32)
    v = rng.integers(1, 1_000_000, n).astype(np.int64)
    aggs = [(dg.AGG_SUM_I64, v), (dg.AGG_COUNT, None)]
    t, kern = _run(aggs, [g], pu=pu, salt=77, G_cap=1 << 17)
    assert kern.startswith("k_srt"), kern
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 77), [g], aggs))


@pytest.mark.parametrize("ni,nf", [(0, 0), (0, 1), (1, 1), (2, 0), (2, 2), (1, 2)])
def test_value_column_combinations(orc, ni, nf):
    rng = np.random.default_rng(10 * ni + nf)
    n = 400_009
    pu = rng.integers(0, 2**40, n).astype(np.int64)
    g = rng.integers(0, 20_000, n).astype(np.int32)
    aggs = [(dg.AGG_COUNT, None)]
    for c in range(ni):  # one column beyond the int32 subset tables (|v| >= 2^26)
        hi = 10_000_000 if c == 0 else 2**40
        aggs.append((dg.AGG_SUM_I64, rng.integers(-hi, hi, n).astype(np.int64)))
    for c in range(nf):
        aggs.append((dg.AGG_AVG_F64 if c == 0 else dg.AGG_SUM_F64, rng.uniform(-1, 1, n) * 10.0 ** c))
    t, kern = _run(aggs, [g], pu=pu, salt=3, G_cap=1 << 15)
    assert kern.startswith("k_srt"), kern
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 3), [g], aggs))


def test_explicit_masks_zero_rows_dropped(orc):
    rng = np.random.default_rng(5)
    n = 500_003
    masks = rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64).astype(np.uint64)
    masks[::7] = 0  # R21: in no world -- no group, not counted
    g = rng.integers(0, 50_000, n).astype(np.int32)
    only_zero = g == 12_345
    masks[only_zero] = 0  # a key whose every row is dropped must not exist
    v = rng.integers(0, 1000, n).astype(np.int64)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, v)]
    t, kern = _run(aggs, [g], masks=masks, G_cap=1 << 16)
    assert kern.startswith("k_srt"), kern
    got = t.to_host()
    assert 12_345 ^ 0x80000000 not in set(got["keys"].tolist())
    assert_tables_equal(got, orc.agg(masks, [g], aggs))


def test_three_key_columns_and_constant_bytes(orc):
    rng = np.random.default_rng(6)
    n = 600_001
    pu = rng.integers(0, 10**6, n).astype(np.int64)
    k1 = rng.integers(-3, 3, n).astype(np.int8)      # varying top byte
    k2 = np.full(n, 7, np.int8)                       # constant byte: its pass is skipped
    k3 = rng.integers(-30_000, 30_000, n).astype(np.int16)
    f = rng.uniform(0, 1, n)
    aggs = [(dg.AGG_AVG_F64, f), (dg.AGG_COUNT, None)]
    t, kern = _run(aggs, [k1, k2, k3], pu=pu, salt=9, G_cap=1 << 19)
    assert kern.startswith("k_srt"), kern
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 9), [k1, k2, k3], aggs))


def test_one_huge_group_and_singletons(orc):
    # one key holds half the rows (spans hundreds of chunks: boundary atomics), the rest singletons
    rng = np.random.default_rng(7)
    n = 1_000_000
    g = np.where(rng.random(n) < 0.5, 42, rng.permutation(n)).astype(np.int32)
    pu = rng.integers(0, 2**62, n).astype(np.int64)
    v = rng.integers(-5_000_000, 5_000_000, n).astype(np.int64)
    f = rng.standard_normal(n)
    aggs = [(dg.AGG_SUM_I64, v), (dg.AGG_COUNT, None), (dg.AGG_SUM_F64, f)]
    t, kern = _run(aggs, [g], pu=pu, salt=11, G_cap=1 << 20)
    assert kern.startswith("k_srt"), kern
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 11), [g], aggs))


def test_all_rows_one_key(orc):
    n = 70_001
    g = np.full(n, -5, np.int16)
    pu = np.arange(n, dtype=np.int64)
    v = np.arange(n, dtype=np.int64)
    aggs = [(dg.AGG_SUM_I64, v), (dg.AGG_COUNT, None)]
    t, kern = _run(aggs, [g], pu=pu, salt=1, G_cap=8192)
    assert kern.startswith("k_srt"), kern
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 1), [g], aggs))


def test_nonfinite_f64_classes(orc):
    rng = np.random.default_rng(8)
    n = 300_000
    g = rng.integers(0, 10_000, n).astype(np.int32)
    pu = rng.integers(0, 2**50, n).astype(np.int64)
    f = rng.uniform(0, 1, n)
    f[rng.integers(0, n, 40)] = np.nan
    f[rng.integers(0, n, 40)] = np.inf
    f[rng.integers(0, n, 40)] = -np.inf
    aggs = [(dg.AGG_SUM_F64, f), (dg.AGG_COUNT, None)]
    t, kern = _run(aggs, [g], pu=pu, salt=2, G_cap=1 << 14)
    assert kern.startswith("k_srt"), kern
    got, ref = t.to_host(), orc.agg(orc.pac_hash(pu, 2), [g], aggs)
    for k in ("keys", "rows", "K", "count"):
        np.testing.assert_array_equal(got[k], ref[k])
    a, b = got["world"][0], ref["world"][0]
    np.testing.assert_array_equal(np.isnan(a), np.isnan(b))   # R30: the class is order-free
    np.testing.assert_array_equal(np.isposinf(a), np.isposinf(b))
    np.testing.assert_array_equal(np.isneginf(a), np.isneginf(b))
    ok = np.isfinite(b)
    np.testing.assert_allclose(a[ok], b[ok], rtol=1e-9, atol=1e-300)


def test_capacity_reported():
    rng = np.random.default_rng(9)
    n = 200_000
    g = rng.integers(0, 50_000, n).astype(np.int32)
    aggs = [(dg.AGG_COUNT, None)]
    t, kern = _run(aggs, [g], pu=np.arange(n, dtype=np.int64), salt=1, G_cap=4096)
    assert kern.startswith("k_srt"), kern
    assert int(t.status.item()) == pac._lib.PAC_E_CAPACITY
    assert int(t.num_groups.item()) > 4096


def test_equals_deferred_tier_on_c3_rows(monkeypatch):
    w = dg.WORKLOADS["C3"]
    cols = w.host_columns(0, 2_000_000)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    a, kern = _run(aggs, cols["keys"], pu=cols["pu"], salt=123, G_cap=1 << 21)
    assert kern.startswith("k_srt"), kern
    monkeypatch.setenv("PAC_NO_SORT", "1")
    b, kern_b = _run(aggs, cols["keys"], pu=cols["pu"], salt=123, G_cap=1 << 21)
    assert not kern_b.startswith("k_srt"), kern_b
    assert_tables_equal(a.to_host(), b.to_host())


def test_run_twice_identical_integers():
    w = dg.WORKLOADS["C3"]
    cols = w.host_columns(0, 1_000_000)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    a, _ = _run(aggs, cols["keys"], pu=cols["pu"], salt=5, G_cap=1 << 20)
    b, _ = _run(aggs, cols["keys"], pu=cols["pu"], salt=5, G_cap=1 << 20)
    a, b = a.to_host(), b.to_host()
    for k in ("keys", "rows", "K", "count"):
        np.testing.assert_array_equal(a[k], b[k])
    np.testing.assert_array_equal(a["world"][0], b["world"][0])
