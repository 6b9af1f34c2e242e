"""Partition-first aggregation (part.cu + k_agg_tiles_tm over units; opt-in with PAC_PART=1) for
tables with many more groups than a CTA holds: parity with the oracle for the aggregate kinds the
TMEM table takes (int64 SUM + COUNT as BASELINE C3, f64 AVG, MIN next to COUNT), hashed pu keys and explicit masks
with zero rows, one to three key columns, equality with the first-touch + deferred-tier path
(the default), and CAPACITY."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import assert_tables_equal, run_gpu

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_15023_b200 as pac  # noqa: E402


@pytest.fixture(autouse=True)
def _partition_on(monkeypatch):
    monkeypatch.setenv("PAC_PART", "1")


def _zipf_keys(rng, n, groups, s=1.1):
    return (np.minimum(rng.zipf(s, n), groups) - 1).astype(np.int64)


def _run(aggs, keys, **kw):
    pac.profile_enable(True)
    try:
        t, ag = run_gpu(aggs, keys, **kw)
        torch.cuda.synchronize()
        return t, pac.profile_last_kernel()
    finally:
        pac.profile_enable(False)


def test_partition_c3_shape_matches_oracle(orc):
    rng = np.random.default_rng(31)
    n = 1_500_007
    pu = rng.integers(0, 300_000, n).astype(np.int64)
    g = (_zipf_keys(rng, n, 200_000) * 2654435761 % (2**31)).astype(np.int32)
    v = rng.integers(1, 1_000_000, n).astype(np.int64)
    aggs = [(dg.AGG_SUM_I64, v), (dg.AGG_COUNT, None)]
    t, kern = _run(aggs, [g], pu=pu, salt=77, G_cap=1 << 18)
    assert "partition" in kern, kern
    got = t.to_host()
    assert got["G"] > 50_000
    assert_tables_equal(got, orc.agg(orc.pac_hash(pu, 77), [g], aggs))


def test_partition_masks_min_and_count_int64_key(orc):
    rng = np.random.default_rng(32)
    n = 1_200_001
    masks = rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64).astype(np.uint64)
    masks[::11] = 0  # R21: rows in no world are dropped
    g = rng.integers(-(2**62), 2**62, 60_000)[rng.integers(0, 60_000, n)].astype(np.int64)
    m = rng.standard_normal(n) * 100
    m[::997] = np.inf
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_MIN_F64, m)]
    t, kern = _run(aggs, [g], masks=masks, G_cap=1 << 17)
    assert "partition" in kern, kern
    assert_tables_equal(t.to_host(), orc.agg(masks, [g], aggs))


def test_partition_avg_two_key_columns(orc):
    rng = np.random.default_rng(33)
    n = 1_100_000
    pu = rng.integers(0, 2**40, n).astype(np.int64)
    k1 = rng.integers(-300, 300, n).astype(np.int16)
    k2 = rng.integers(0, 200, n).astype(np.int16)
    f = rng.uniform(0, 1, n)
    aggs = [(dg.AGG_AVG_F64, f), (dg.AGG_COUNT, None)]
    t, kern = _run(aggs, [k1, k2], pu=pu, salt=5, G_cap=1 << 17)
    assert "partition" in kern, kern
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 5), [k1, k2], aggs))


def test_partition_equals_deferred_tier_on_c3_rows(monkeypatch):
    w = dg.WORKLOADS["C3"]
    cols = w.host_columns(0, 3_000_000)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    a, kern = _run(aggs, cols["keys"], pu=cols["pu"], salt=123, G_cap=1 << 21)
    assert "partition" in kern
    a = a.to_host()
    monkeypatch.delenv("PAC_PART")
    b, kern_b = _run(aggs, cols["keys"], pu=cols["pu"], salt=123, G_cap=1 << 21)
    assert "partition" not in kern_b
    assert_tables_equal(a, b.to_host())


def test_partition_capacity_reported():
    rng = np.random.default_rng(34)
    n = 1_100_000
    g = rng.integers(0, 5_000, n).astype(np.int32)
    aggs = [(dg.AGG_COUNT, None)]
    t, kern = _run(aggs, [g], pu=np.arange(n, dtype=np.int64), salt=1, G_cap=1024)
    assert "partition" in kern, kern
    assert int(t.status.item()) == pac._lib.PAC_E_CAPACITY
