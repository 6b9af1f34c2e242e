"""Deferred HBM tier (agg.cu k_spill_*): rows of groups without a CTA-local slot are recorded
and folded per group after the pass.  Parity with the oracle for every value column kind, with
the record capacity covering all tier rows, none (direct atomics) and part of them (overflow
rows take atomics)."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import assert_tables_equal, run_gpu

pytestmark = pytest.mark.gpu


def _case(seed, n, groups):
    rng = np.random.default_rng(seed)
    pu = rng.integers(0, 40_000, n).astype(np.int64)
    # Zipf-like skew: a few hot groups (CTA-local slots) and a long tail (the HBM tier)
    g = np.minimum(rng.zipf(1.2, n), groups).astype(np.int32) * 7 - 1000
    i1 = rng.integers(-10**6, 10**6, n).astype(np.int64)
    i2 = rng.integers(0, 2**40, n).astype(np.int64)
    f1 = rng.standard_normal(n) * 1e3
    f2 = rng.integers(1, 50, n).astype(np.float64)
    m = rng.standard_normal(n)
    aggs = [(dg.AGG_SUM_I64, i1), (dg.AGG_SUM_I64, i2), (dg.AGG_SUM_F64, f1), (dg.AGG_AVG_F64, f2),
            (dg.AGG_MIN_F64, m), (dg.AGG_MAX_F64, m), (dg.AGG_COUNT, None)]
    return pu, [g], aggs


@pytest.mark.parametrize("spill_rows", [None, 0, 20_000])
def test_spill_all_value_kinds_match_oracle(orc, spill_rows):
    pu, keys, aggs = _case(11, 300_001, 60_000)
    t, _ = run_gpu(aggs, keys, pu=pu, salt=9, G_cap=1 << 16, spill_rows=spill_rows)
    got = t.to_host()
    ref = orc.agg(orc.pac_hash(pu, 9), keys, aggs)
    assert got["G"] > 5_000
    assert_tables_equal(got, ref)


def test_spill_with_explicit_masks_and_hot_tail_group(orc):
    # one group with many rows that never gets a local slot in late CTAs: long runs in the
    # grouped records (several chunks of one slot)
    rng = np.random.default_rng(12)
    n = 400_000
    masks = rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64).astype(np.uint64)
    masks[::13] = 0  # R21: rows in no world are dropped
    g = rng.integers(0, 50_000, n).astype(np.int64)
    g[n // 2:][::3] = 123_456_789  # hot key appearing only in the second half
    iv = rng.integers(0, 1000, n).astype(np.int64)
    aggs = [(dg.AGG_SUM_I64, iv), (dg.AGG_COUNT, None)]
    t, _ = run_gpu(aggs, [g], masks=masks, G_cap=1 << 16)
    ref = orc.agg(masks, [g], aggs)
    assert_tables_equal(t.to_host(), ref)
