"""Pins of the oracle's m = 128 extension (§8 f4, P:L92 footnote; readings R28, R29) against things
other than itself: exact popcount 64 and the fixed point of the balancing, per-bit / pairwise
statistics of a uniform balanced 128-bit word (rho = -1/127), j* uniform over 128 worlds,
the 128-world aggregation reducing to two 64-world aggregations of the mask halves and to a
plain pandas GROUP BY for all-ones masks, and finalize closed forms over 128 worlds."""
import numpy as np
import pytest

import oracle as orc

M = 128


def _bits(masks):
    return np.unpackbits(np.ascontiguousarray(masks).view(np.uint8).reshape(len(masks), 16), axis=1,
                         bitorder="little").astype(np.int8)


def test_hash128_balanced_and_fixed_point():
    keys = np.concatenate([np.arange(200_000, dtype=np.int64),
                           np.random.default_rng(0).integers(-(2**63), 2**63 - 1, 100_000, dtype=np.int64)])
    salt = 0x243F6A8885A308D3
    h = orc.pac_hash128(keys, salt)
    b = _bits(h)
    assert np.all(b.sum(1) == 64)
    # fixed point: a mixed word that is already balanced is returned unchanged
    lo = np.array([orc.fmix64((int(k) ^ salt) & 0xFFFFFFFFFFFFFFFF) for k in keys[:20_000]], dtype=np.uint64)
    hi = np.array([orc.fmix64(int(x) ^ 0x6A09E667F3BCC909) for x in lo], dtype=np.uint64)
    pc = np.array([bin(int(a)).count("1") + bin(int(c)).count("1") for a, c in zip(lo, hi)])
    bal = pc == 64
    assert bal.sum() > 1000
    np.testing.assert_array_equal(h[:20_000][bal, 0], lo[bal])
    np.testing.assert_array_equal(h[:20_000][bal, 1], hi[bal])
    # per-bit frequency 1/2 and pairwise correlation -1/127 of a uniform balanced word
    f = b.mean(0)
    assert np.all(np.abs(f - 0.5) < 0.006)
    c = np.corrcoef(b[:, :40].T.astype(np.float64))
    off = c[~np.eye(40, dtype=bool)]
    assert abs(off.mean() + 1 / 127) < 0.003 and np.abs(off + 1 / 127).max() < 0.02


def test_session128_jstar_uniform():
    js = np.array([orc.session128(s)[0] for s in range(12_800)])
    cnt = np.bincount(js, minlength=M)
    chi2 = ((cnt - 100.0) ** 2 / 100.0).sum()
    assert chi2 < 127 + 6 * np.sqrt(2 * 127)
    _, salt, P = orc.session128(7)
    assert salt == orc.session(7)[1] and np.allclose(P, 1 / 128)


def test_agg128_halves_are_two_m64_aggregations():
    rng = np.random.default_rng(3)
    n = 20_000
    h = orc.pac_hash128(rng.integers(0, 800, n).astype(np.int64), 5)
    h[:, 0] |= np.uint64(1)        # both halves nonzero: same group sets in all three tables
    h[:, 1] |= np.uint64(1)
    keys = [rng.integers(0, 5, n).astype(np.int8)]
    iv = rng.integers(-1000, 1000, n).astype(np.int64)
    fv = rng.normal(0, 1, n)
    aggs = [(orc.COUNT, None), (orc.SUM_I64, iv), (orc.AVG_F64, fv), (orc.MIN_F64, fv), (orc.MAX_F64, fv)]
    t = orc.agg128(h, keys, aggs)
    lo = orc.agg(np.ascontiguousarray(h[:, 0]), keys, aggs)
    hi = orc.agg(np.ascontiguousarray(h[:, 1]), keys, aggs)
    np.testing.assert_array_equal(t["keys"], lo["keys"])
    np.testing.assert_array_equal(t["rows"], lo["rows"])
    np.testing.assert_array_equal(t["K"][:, 0], lo["K"])
    np.testing.assert_array_equal(t["K"][:, 1], hi["K"])
    np.testing.assert_array_equal(t["count"][:, :64], lo["count"])
    np.testing.assert_array_equal(t["count"][:, 64:], hi["count"])
    for a in range(1, len(aggs)):
        np.testing.assert_allclose(t["world"][a][:, :64], lo["world"][a], rtol=1e-12)
        np.testing.assert_allclose(t["world"][a][:, 64:], hi["world"][a], rtol=1e-12)
    # invariants: sum_j count_j = 64 * rows for balanced masks without the forced bits
    h2 = orc.pac_hash128(rng.integers(0, 800, n).astype(np.int64), 6)
    t2 = orc.agg128(h2, keys, [(orc.COUNT, None)])
    np.testing.assert_array_equal(t2["count"].sum(1), 64 * t2["rows"])


def test_agg128_all_ones_is_group_by():
    import pandas as pd
    rng = np.random.default_rng(4)
    n = 5000
    h = np.full((n, 2), np.uint64(2**64 - 1), dtype=np.uint64)
    keys = [rng.integers(-3, 3, n).astype(np.int16)]
    iv = rng.integers(0, 100, n).astype(np.int64)
    t = orc.agg128(h, keys, [(orc.SUM_I64, iv)])
    ref = pd.DataFrame({"k": keys[0], "v": iv}).groupby("k")["v"].sum().sort_index()
    for j in (0, 63, 64, 127):
        np.testing.assert_array_equal(t["world"][0][:, j], ref.values)


def test_finalize128_closed_forms():
    seed = 9
    jstar, salt, P = orc.session128(seed)
    B = 1 / 128
    G = 1
    full = np.array([[2**64 - 1, 2**64 - 1]], dtype=np.uint64)
    # y_j = j: weighted population variance under uniform P = (128^2 - 1) / 12
    t = {"G": G, "kinds": [orc.MAX_F64], "K": full, "rows": np.array([1000]),
         "count": np.zeros((1, M), dtype=np.int64), "world": [np.arange(M, dtype=np.float64)[None, :]]}
    rel, isn, fl, d, P2 = orc.finalize128(seed, B, jstar, P, t)
    assert isn[0, 0] == 0 and abs(d[0, 0] - 1365.25 / (2 * B)) < 1e-9 and abs(P2.sum() - 1) < 1e-12
    # constant vector: exact release, posterior unchanged
    t["world"] = [np.full((1, M), 4.5)]
    rel, isn, fl, d, P3 = orc.finalize128(seed, B, jstar, P, t)
    assert rel[0, 0] == 4.5 and np.array_equal(P3, P)
    # NULL rate (128 - popcount K) / 128: K with 64 worlds -> 1/2
    nulls = []
    for r in range(4000):
        t["K"] = np.array([[2**64 - 1, 0]], dtype=np.uint64)
        _, isn, _, _, _ = orc.finalize128(seed, B, jstar, P, t, r)
        nulls.append(isn[0, 0])
    assert abs(np.mean(nulls) - 0.5) < 5 * np.sqrt(0.25 / 4000)
    t["K"] = np.zeros((1, 2), dtype=np.uint64)
    assert orc.finalize128(seed, B, jstar, P, t)[1][0, 0] == 1
