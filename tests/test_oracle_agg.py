"""Pins for the oracle's 64-world aggregation (O1 brute force, O2 single pass).

The independent reference is a *library* GROUP BY (pandas) run separately on each
world's filtered rows -- Eq. counter P:L249-253 / PAC aggregation P:L956-970 and
the PAC-DB m-fold semantics P:L852-894, with the library doing the grouping and the
arithmetic.  Plus the invariants the paper's construction implies.
"""
import numpy as np
import pandas as pd
import pytest

from datagen import AGG_AVG_F64, AGG_COUNT, AGG_MAX_F64, AGG_MIN_F64, AGG_SUM_F64, AGG_SUM_I64

ALL_AGGS = [AGG_COUNT, AGG_SUM_I64, AGG_SUM_F64, AGG_AVG_F64, AGG_MIN_F64, AGG_MAX_F64]


def _bits(masks):
    return np.unpackbits(masks.astype(np.uint64).view(np.uint8).reshape(-1, 8), axis=1,
                         bitorder="little").astype(bool)


def _random_case(rng, n, widths, n_pu=50, card=4):
    pu = rng.integers(-10**12, 10**12, n_pu)[rng.integers(0, n_pu, n)].astype(np.int64)
    keys = []
    for w in widths:
        dt = {1: np.int8, 2: np.int16, 4: np.int32, 8: np.int64}[w]
        lo = -card // 2
        keys.append(rng.integers(lo, lo + card, n).astype(dt))
    iv = rng.integers(-10**9, 10**9, n).astype(np.int64)
    fv = rng.normal(3.0, 10.0, n)
    return pu, keys, iv, fv


def _aggs(iv, fv):
    vals = {AGG_COUNT: None, AGG_SUM_I64: iv, AGG_SUM_F64: fv, AGG_AVG_F64: fv,
            AGG_MIN_F64: fv, AGG_MAX_F64: fv}
    return [(k, vals[k]) for k in ALL_AGGS]


def _pandas_world_tables(masks, keys, iv, fv):
    """Per world j: plain pandas GROUP BY over the rows with bit j set."""
    B = _bits(masks)
    df = pd.DataFrame({f"k{i}": k for i, k in enumerate(keys)})
    df["iv"] = iv
    df["fv"] = fv
    if not keys:
        df["k_"] = 0
    kcols = [c for c in df.columns if c.startswith("k")]
    out = []
    for j in range(64):
        sub = df[B[:, j]]
        out.append(sub.groupby(kcols).agg(cnt=("iv", "size"), isum=("iv", "sum"),
                                          fsum=("fv", "sum"), fmin=("fv", "min"),
                                          fmax=("fv", "max")))
    return out, kcols


def _unpack_group_key(packed, widths):
    vals, shift = [], 0
    for w in reversed(widths):
        bits = 8 * w
        u = (int(packed) >> shift) & ((1 << bits) - 1)
        u ^= 1 << (bits - 1)
        if u >= 1 << (bits - 1):
            u -= 1 << bits
        vals.append(u)
        shift += bits
    return tuple(reversed(vals))


@pytest.mark.parametrize("widths", [[], [1], [4], [8], [1, 1], [2, 4], [1, 2, 1]])
@pytest.mark.parametrize("method", ["o1", "o2"])
def test_world_tables_equal_per_world_pandas_groupby(orc, widths, method):
    rng = np.random.default_rng(len(widths) * 10 + (method == "o1"))
    n = 3000
    pu, keys, iv, fv = _random_case(rng, n, widths)
    masks = orc.pac_hash(pu, 777)
    t = orc.agg(masks, keys, _aggs(iv, fv), method=method)
    ref, kcols = _pandas_world_tables(masks, keys, iv, fv)
    # canonical order = ascending lexicographic signed key (R20)
    all_groups = sorted(set().union(*[set(r.index) for r in ref]))
    assert t["G"] == len(all_groups)
    for g in range(t["G"]):
        kv = _unpack_group_key(t["keys"][g], widths) if widths else (0,)
        gk = kv if len(kv) > 1 else kv[0]
        assert gk == all_groups[g]
        for j in range(64):
            r = ref[j]
            if gk in r.index:
                row = r.loc[gk]
                assert t["count"][g, j] == row.cnt
                assert t["world"][1][g, j] == row.isum
                np.testing.assert_allclose(t["world"][2][g, j], row.fsum, rtol=1e-12, atol=1e-9)
                np.testing.assert_allclose(t["world"][3][g, j], row.fsum, rtol=1e-12, atol=1e-9)
                assert t["world"][4][g, j] == row.fmin
                assert t["world"][5][g, j] == row.fmax
            else:
                assert t["count"][g, j] == 0
                assert t["world"][1][g, j] == 0
                assert t["world"][4][g, j] == np.inf
                assert t["world"][5][g, j] == -np.inf


def test_all_ones_masks_reduce_to_plain_group_by(orc):
    # S:L367 idea: with every row in every world, each world is the textbook GROUP BY.
    rng = np.random.default_rng(5)
    pu, keys, iv, fv = _random_case(rng, 5000, [4])
    masks = np.full(5000, 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
    t = orc.agg(masks, keys, _aggs(iv, fv))
    ref = pd.DataFrame({"k": keys[0], "iv": iv, "fv": fv}).groupby("k").agg(
        cnt=("iv", "size"), isum=("iv", "sum"), fmin=("fv", "min"), fmax=("fv", "max"),
        fmean=("fv", "mean"))
    assert t["G"] == len(ref)
    for g, (k, row) in enumerate(ref.iterrows()):
        assert np.all(t["count"][g] == row.cnt)
        assert np.all(t["world"][1][g] == row.isum)
        assert np.all(t["world"][4][g] == row.fmin)
        assert np.all(t["world"][5][g] == row.fmax)
        np.testing.assert_allclose(t["world"][3][g] / t["count"][g], row.fmean, rtol=1e-12)


def test_invariants_of_balanced_masks(orc):
    # Every row lands in exactly 32 worlds (P:L9), so per group
    # sum_j count_j = 32 rows and sum_j sum_j = 32 * sum(v) exactly; K = {j: count_j>0}
    # (P:L1654); max_j MAX_j = group max, min_j MIN_j = group min.
    rng = np.random.default_rng(9)
    pu, keys, iv, fv = _random_case(rng, 20000, [1, 1], n_pu=3000, card=3)
    masks = orc.pac_hash(pu, 4242)
    t = orc.agg(masks, keys, _aggs(iv, fv))
    df = pd.DataFrame({"a": keys[0], "b": keys[1], "iv": iv, "fv": fv}).groupby(["a", "b"]).agg(
        n=("iv", "size"), s=("iv", "sum"), mn=("fv", "min"), mx=("fv", "max"))
    for g in range(t["G"]):
        row = df.iloc[g]
        assert t["rows"][g] == row.n
        assert t["count"][g].sum() == 32 * row.n
        assert t["world"][1][g].sum() == 32 * row.s
        Kbits = _bits(np.array([t["K"][g]]))[0]
        assert np.array_equal(Kbits, t["count"][g] > 0)
        assert t["world"][5][g].max() == row.mx
        assert t["world"][4][g].min() == row.mn


def test_zero_masks_are_dropped_and_ungrouped_has_one_group(orc):
    # R21: rows with mask 0 are in no world and create no group; an
    # ungrouped aggregate always has exactly one group, even over zero rows.
    keys = [np.array([1, 2, 2, 3], dtype=np.int32)]
    masks = np.array([0, 0xFF, 0, 0], dtype=np.uint64)
    t = orc.agg(masks, keys, [(AGG_COUNT, None)])
    assert t["G"] == 1 and t["rows"][0] == 1
    assert list(t["count"][0, :8]) == [1] * 8 and t["count"][0, 8:].sum() == 0
    t0 = orc.agg(np.zeros(0, dtype=np.uint64), [], [(AGG_COUNT, None)])
    assert t0["G"] == 1 and t0["rows"][0] == 0 and t0["K"][0] == 0


def test_int64_overflow_is_reported(orc):
    iv = np.array([2**62, 2**62, 2**62], dtype=np.int64)
    masks = np.full(3, 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
    t = orc.agg(masks, [], [(AGG_SUM_I64, iv)])
    assert t["overflow"]


def test_restricting_to_sampled_groups_matches_full_table(orc):
    rng = np.random.default_rng(11)
    pu, keys, iv, fv = _random_case(rng, 8000, [4], card=40)
    masks = orc.pac_hash(pu, 1)
    full = orc.agg(masks, keys, _aggs(iv, fv))
    pick = full["keys"][[3, 17, 30]]
    part = orc.agg(masks, keys, _aggs(iv, fv), gkeys=pick)
    for i, g in enumerate([3, 17, 30]):
        assert np.array_equal(part["count"][i], full["count"][g])
        assert np.array_equal(part["world"][1][i], full["world"][1][g])
        assert np.array_equal(part["world"][5][i], full["world"][5][g])


def _total_order_key(v):
    # R31 (DuckDB's order on DOUBLE): NaN above every other value, all NaNs equal
    return (1, 0.0) if np.isnan(v) else (0, v)


def _fclass(x):
    return "nan" if np.isnan(x) else ("+inf" if x == np.inf else ("-inf" if x == -np.inf else "fin"))


@pytest.mark.parametrize("method", ["o1", "o2"])
def test_non_finite_values_follow_ieee_sums_and_total_order_extremes(orc, method):
    # R30: SUM/AVG of f64 is the IEEE sum (class order-independent: any NaN -> NaN,
    # +inf with -inf -> NaN, else the infinity); R31: MIN/MAX under the total order with
    # NaN largest.  Reference: per world, numpy's plain sum for the class and Python's
    # sorted() with the total-order key for the extremes, on the world's filtered rows.
    rng = np.random.default_rng(31)
    n = 400
    pu = rng.integers(0, 40, n).astype(np.int64)
    keys = [rng.integers(0, 3, n).astype(np.int32)]
    fv = rng.normal(0.0, 5.0, n)
    fv[rng.choice(n, 12, replace=False)] = np.nan
    fv[rng.choice(n, 8, replace=False)] = np.inf
    fv[rng.choice(n, 8, replace=False)] = -np.inf
    # group 3: only NaN rows; group 4: only +inf rows (a present world whose MIN is +inf)
    keys[0] = np.concatenate([keys[0], [3, 3, 4, 4]]).astype(np.int32)
    fv = np.concatenate([fv, [np.nan, np.nan, np.inf, np.inf]])
    pu = np.concatenate([pu, [100, 101, 102, 103]]).astype(np.int64)
    iv = np.zeros(len(fv), dtype=np.int64)
    masks = orc.pac_hash(pu, 99)
    t = orc.agg(masks, keys, [(AGG_COUNT, None), (AGG_SUM_F64, fv), (AGG_MIN_F64, fv), (AGG_MAX_F64, fv)],
                method=method)
    B = _bits(masks)
    for g in range(t["G"]):
        gk = _unpack_group_key(t["keys"][g], [4])[0]
        for j in range(64):
            sel = (keys[0] == gk) & B[:, j]
            vals = fv[sel]
            assert t["count"][g, j] == sel.sum()
            if sel.sum() == 0:
                assert t["world"][2][g, j] == np.inf and t["world"][3][g, j] == -np.inf
                continue
            ref_sum = float(np.sum(vals))
            got = t["world"][1][g, j]
            assert _fclass(got) == _fclass(ref_sum)
            if _fclass(ref_sum) == "fin":
                np.testing.assert_allclose(got, ref_sum, rtol=1e-12, atol=1e-9)
            srt = sorted(vals.tolist(), key=_total_order_key)
            for got_e, ref_e in ((t["world"][2][g, j], srt[0]), (t["world"][3][g, j], srt[-1])):
                assert _fclass(got_e) == _fclass(ref_e)
                if _fclass(ref_e) != "nan":
                    assert got_e == ref_e
    # the special groups, spelled out
    g3 = [g for g in range(t["G"]) if _unpack_group_key(t["keys"][g], [4])[0] == 3][0]
    present = t["count"][g3] > 0
    assert present.any() and np.all(np.isnan(t["world"][2][g3][present]))
    assert np.all(np.isnan(t["world"][3][g3][present]))
    g4 = [g for g in range(t["G"]) if _unpack_group_key(t["keys"][g], [4])[0] == 4][0]
    present = t["count"][g4] > 0
    assert np.all(t["world"][2][g4][present] == np.inf) and np.all(t["world"][1][g4][present] == np.inf)


def test_non_finite_sum_classes_are_exact(orc):
    # R30 closed forms on all-ones masks (every world = all rows)
    ones = np.full(3, 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
    for vals, cls in (([1.0, np.inf, 2.0], "+inf"), ([1.0, -np.inf], "-inf"), ([np.inf, -np.inf, 1.0], "nan"),
                      ([np.nan, 1.0, 2.0], "nan"), ([1e300, -1e300, 3.0], "fin")):
        v = np.array(vals)
        t = orc.agg(ones[:len(v)], [], [(AGG_SUM_F64, v), (AGG_MIN_F64, v), (AGG_MAX_F64, v)])
        assert all(_fclass(x) == cls for x in t["world"][0][0])
        srt = sorted(vals, key=_total_order_key)
        assert all(_fclass(x) == _fclass(srt[0]) for x in t["world"][1][0])
        assert all(_fclass(x) == _fclass(srt[-1]) for x in t["world"][2][0])
