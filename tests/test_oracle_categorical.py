"""Pins of the oracle's categorical path (§8 f1; R22-R26) against things other than
itself: numpy's comparison operators, the bitwise truth table of pac_select (SPEC example),
binomial acceptance rates of pac_filter (Eq. pac-filter), algebraic identities of
vector lifting, closed forms of pac_noised on lifted vectors, and the paper's
ratio-lambda claim (noising the lifted ratio once beats noising twice)."""
import numpy as np
import pytest

import oracle as orc

FULL = (1 << 64) - 1
CMPS = {orc.CMP_LT: np.less, orc.CMP_LE: np.less_equal, orc.CMP_GT: np.greater,
        orc.CMP_GE: np.greater_equal, orc.CMP_EQ: np.equal}


def _bits_from_bool(b):
    return int(sum(1 << j for j in range(64) if b[j]))


@pytest.mark.parametrize("cmp", list(CMPS))
def test_cmp_bits_match_numpy(cmp):
    rng = np.random.default_rng(cmp)
    for t in range(300):
        c = rng.integers(-3, 4, 64).astype(np.float64)       # many ties
        if t % 3 == 0:
            c[rng.integers(0, 64, 5)] = np.nan                 # NaN worlds never compare true
        if t % 5 == 0:
            c[rng.integers(0, 64, 3)] = np.inf
        pres = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2)) if t % 4 else FULL
        v = float(rng.integers(-4, 5)) if t % 7 else [np.nan, -np.inf, np.inf, -0.0][t % 4]
        pres_b = np.array([(pres >> j) & 1 for j in range(64)], dtype=bool)
        want = _bits_from_bool(CMPS[cmp](v, c) & pres_b)
        assert orc.cmp_bits(cmp, v, c, pres) == want


def test_select_truth_table_and_identities():
    # SPEC example: pu = ...0101, b = ...0011 -> ...0001
    h = np.array([0b0101], dtype=np.uint64)
    assert orc.select(h, np.zeros(1, np.int32), np.array([0b0011], np.uint64))[0] == 0b0001
    rng = np.random.default_rng(1)
    h = rng.integers(0, 2**63, 1000, dtype=np.int64).astype(np.uint64) * np.uint64(2) + np.uint64(1)
    g = rng.integers(0, 3, 1000).astype(np.int32)
    bits = np.array([FULL, 0, 0x00000000FFFFFFFF], dtype=np.uint64)
    out = orc.select(h, g, bits)
    np.testing.assert_array_equal(out[g == 0], h[g == 0])                       # AND identity
    assert np.all(out[g == 1] == 0)                                             # annihilator
    np.testing.assert_array_equal(out[g == 2], h[g == 2] & np.uint64(0xFFFFFFFF))


def test_select_cmp_is_select_of_cmp_bits():
    rng = np.random.default_rng(2)
    G, n = 7, 5000
    c = rng.normal(0, 1, (G, 64))
    pres = rng.integers(0, 2**63, G, dtype=np.int64).astype(np.uint64)
    pres[0] = np.uint64(FULL)
    v = rng.normal(0, 1, n)
    g = rng.integers(0, G, n).astype(np.int32)
    h = orc.pac_hash(rng.integers(0, 10**6, n).astype(np.int64), 3)
    for cmp, op in CMPS.items():
        out = orc.select_cmp(cmp, h, v, g, c, pres)
        for i in range(0, n, 97):
            b = _bits_from_bool(op(v[i], c[g[i]]) & np.array([(int(pres[g[i]]) >> j) & 1 for j in range(64)],
                                                              dtype=bool))
            assert int(out[i]) == int(h[i]) & b


@pytest.mark.parametrize("pc", [0, 1, 16, 32, 48, 63, 64])
def test_filter_rate_is_popcount_over_64(pc):
    n = 100_000
    bits = np.full(n, (1 << pc) - 1 if pc < 64 else FULL, dtype=np.uint64)
    out = orc.pac_filter(1234, 0, bits)
    if pc in (0, 64):
        assert np.all(out == (pc == 64))           # exactly never / always
    else:
        p = pc / 64
        assert abs(out.mean() - p) < 5 * np.sqrt(p * (1 - p) / n)
    # the draw depends on the element, not on the bits: the same seed gives nested outcomes
    if 0 < pc < 64:
        more = orc.pac_filter(1234, 0, np.full(n, (1 << (pc + 1)) - 1, dtype=np.uint64))
        assert np.all(more >= out)


def test_filter_cmp_matches_filter_of_cmp_bits():
    rng = np.random.default_rng(4)
    G, n = 5, 20_000
    c = rng.normal(0, 1, (G, 64))
    pres = np.full(G, FULL, dtype=np.uint64)
    v = rng.normal(0, 1, n)
    g = rng.integers(0, G, n).astype(np.int32)
    bits = np.array([orc.cmp_bits(orc.CMP_LT, v[i], c[g[i]], FULL) for i in range(n)], dtype=np.uint64)
    np.testing.assert_array_equal(orc.filter_cmp(99, 2, orc.CMP_LT, v, g, c, pres), orc.pac_filter(99, 2, bits))


def test_lift_identities_and_presence():
    rng = np.random.default_rng(5)
    n = 50
    a = rng.integers(-10**6, 10**6, (n, 64)).astype(np.float64)     # integer-valued: exact arithmetic
    b = rng.integers(1, 10**6, (n, 64)).astype(np.float64)
    pa = rng.integers(0, 2**63, n, dtype=np.int64).astype(np.uint64) | np.uint64(1)
    pb = np.full(n, FULL, dtype=np.uint64)
    s, ps = orc.lift(orc.OP_ADD, (a, pa), (b, pb), n)
    d, pd = orc.lift(orc.OP_SUB, (s, ps), (b, pb), n)
    mask = np.array([[(int(p) >> j) & 1 for j in range(64)] for p in pa], dtype=bool)
    np.testing.assert_array_equal(pd, pa)                         # presence = AND
    np.testing.assert_array_equal(d[mask], a[mask])               # (a + b) - b == a exactly
    assert np.all(d[~mask] == 0)                                  # absent worlds hold 0 (R9)
    two, _ = orc.lift(orc.OP_MUL, (a, pb), 2.0, n)
    aa, _ = orc.lift(orc.OP_ADD, (a, pb), (a, pb), n)
    np.testing.assert_array_equal(two, aa)                        # 2*a == a + a
    q, pq = orc.lift(orc.OP_DIV, (b, pb), (b, pb), n)
    assert np.all(q == 1.0) and np.all(pq == np.uint64(FULL))     # b / b == 1
    mn, _ = orc.lift(orc.OP_MIN, (a, pb), 0.0, n)
    mx, _ = orc.lift(orc.OP_MAX, (a, pb), 0.0, n)
    np.testing.assert_array_equal(mn + mx, a)                     # min(a,0) + max(a,0) == a
    bits = orc.lift_cmp(orc.CMP_GT, (a, pa), 0.0, n)
    for i in range(n):
        assert int(bits[i]) == _bits_from_bool((a[i] > 0) & mask[i])


def test_noised_y_closed_forms():
    seed = 77
    jstar, salt, P = orc.session(seed)
    B = 1 / 128
    # y_j = j, full presence: s^2 = (64^2 - 1)/12 = 341.25 under uniform P
    y = np.arange(64, dtype=np.float64)[None, :]
    rel, isn, delta, P1 = orc.noised_y(seed, B, jstar, P, y, np.array([FULL], np.uint64))
    assert isn[0] == 0 and abs(delta[0] - 341.25 / (2 * B)) < 1e-9
    assert abs(P1.sum() - 1) < 1e-12
    # constant vector: exact release, no update
    rel, isn, delta, P2 = orc.noised_y(seed, B, jstar, P, np.full((1, 64), 3.5), np.array([FULL], np.uint64))
    assert rel[0] == 3.5 and delta[0] == 0.0 and np.array_equal(P2, P)
    # presence 0: always NULL
    rel, isn, _, _ = orc.noised_y(seed, B, jstar, P, np.ones((50, 64)), np.zeros(50, np.uint64))
    assert np.all(isn == 1) and np.all(np.isnan(rel))
    # a table cell noised as a world vector has the table finalize's variance (same P)
    rng = np.random.default_rng(3)
    pu = rng.integers(0, 300, 5000).astype(np.int64)
    keys = [np.zeros(5000, dtype=np.int8)]
    iv = rng.integers(1, 1000, 5000).astype(np.int64)
    t = orc.agg(orc.pac_hash(pu, salt), keys, [(orc.SUM_I64, iv)])
    yv, pres = orc.world_vectors(t, 0)
    _, n1, d1, _ = orc.noised_y(seed, B, jstar, P, yv, pres)
    _, n2, _, d2, _ = orc.finalize(seed, B, jstar, P, t)
    if n1[0] == 0 and n2[0, 0] == 0:
        assert abs(d1[0] - d2[0, 0]) <= 1e-12 * d2[0, 0]


def test_ratio_noised_once_beats_noised_twice():
    """P:L2074-2108 (Fig. ratio): the lifted ratio of two sums noised once has lower error
    than the ratio of the two separately noised sums."""
    rng = np.random.default_rng(11)
    n = 20_000
    pu = rng.integers(0, 2_000, n).astype(np.int64)
    e = rng.integers(1, 1000, n).astype(np.int64)
    sel = rng.random(n) < 0.3
    ei = np.where(sel, e, 0).astype(np.int64)
    keys = [np.zeros(n, dtype=np.int8)]
    exact = ei.sum() / e.sum()
    err_once, err_twice = [], []
    for seed in range(40):
        jstar, salt, P = orc.session(1000 + seed)
        t = orc.agg(orc.pac_hash(pu, salt), keys, [(orc.SUM_I64, ei), (orc.SUM_I64, e)])
        x, px = orc.world_vectors(t, 0)
        y, py = orc.world_vectors(t, 1)
        r, pr = orc.lift(orc.OP_DIV, (x, px), (y, py), 1)
        rel, isn, _, _ = orc.noised_y(1000 + seed, 1 / 128, jstar, P, r, pr)
        rel2, isn2, _, _, _ = orc.finalize(1000 + seed, 1 / 128, jstar, P, t)
        if isn[0] or isn2[0].any():
            continue
        err_once.append(abs(rel[0] - exact) / exact)
        err_twice.append(abs(rel2[0, 0] / rel2[0, 1] - exact) / exact)
    assert len(err_once) > 30
    assert np.mean(err_once) < np.mean(err_twice)
