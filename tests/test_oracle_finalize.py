"""Pins for the oracle's finalize (pac_noised) and posterior update.

References: closed forms of the weighted variance, numpy.average with weights,
scipy.stats.norm for the Gaussian likelihood in Bayes' rule, binomial / KS
statistics for the NULL mechanism and the calibrated noise
N(0, s^2/(2B)).
"""
import math

import numpy as np
import pytest
from scipy import stats

from datagen import AGG_AVG_F64, AGG_COUNT, AGG_MAX_F64, AGG_MIN_F64, AGG_SUM_I64

FULL = np.uint64(0xFFFFFFFFFFFFFFFF)
B = 1.0 / 128.0


def _table(kinds, K, rows, count, worlds):
    G = len(K)
    return {"G": G, "keys": np.arange(G, dtype=np.uint64), "rows": np.array(rows, dtype=np.int64),
            "K": np.array(K, dtype=np.uint64), "count": np.ascontiguousarray(count, dtype=np.int64),
            "world": [None if w is None else np.ascontiguousarray(w) for w in worlds],
            "kinds": list(kinds)}


def test_weighted_variance_matches_numpy_average(orc):
    rng = np.random.default_rng(0)
    for _ in range(50):
        P = rng.random(64)
        P /= P.sum()
        y = rng.normal(0, 100, 64)
        mu = np.average(y, weights=P)
        ref = np.average((y - mu) ** 2, weights=P)
        assert orc.weighted_var(P, y) == pytest.approx(ref, rel=1e-12)
    # closed form: y_j = j under uniform P -> (64^2 - 1)/12 = 341.25
    assert orc.weighted_var(np.full(64, 1 / 64), np.arange(64.0)) == pytest.approx(341.25, rel=1e-14)
    # zero-variance reading R11: equal y over the support -> exactly 0
    P = np.zeros(64); P[[3, 9]] = 0.5
    y = np.arange(64.0); y[3] = y[9] = 7.25
    assert orc.weighted_var(P, y) == 0.0


def test_posterior_update_is_gaussian_bayes(orc):
    # P <- P*W / sum(P*W), W_j the N(y_j, Delta) likelihood of y~.
    rng = np.random.default_rng(1)
    for _ in range(50):
        P = rng.random(64)
        P /= P.sum()
        y = rng.normal(0, 5, 64)
        delta = rng.uniform(0.5, 50)
        yt = rng.normal(0, 5)
        lik = stats.norm.pdf(yt, loc=y, scale=math.sqrt(delta))
        ref = P * lik / np.sum(P * lik)
        np.testing.assert_allclose(orc.posterior_update(P, y, yt, delta), ref, rtol=1e-10, atol=1e-300)


def test_posterior_two_world_closed_form(orc):
    # Two worlds with mass: posterior odds = prior odds * likelihood ratio.
    P = np.zeros(64); P[0], P[1] = 0.25, 0.75
    y = np.zeros(64); y[0], y[1] = 0.0, 2.0
    out = orc.posterior_update(P, y, 1.5, 1.0)
    lr = math.exp(-(1.5 ** 2) / 2) / math.exp(-(0.5 ** 2) / 2)
    odds = (0.25 / 0.75) * lr
    assert out[0] == pytest.approx(odds / (1 + odds), rel=1e-13)
    assert out[1] == pytest.approx(1 / (1 + odds), rel=1e-13)
    assert np.all(out[2:] == 0.0)


def test_single_pu_group_closed_form(orc):
    # One PU with value S: COUNT world vector y in {0, 2}, SUM y in {0, 2S}, 32 each,
    # K = the PU's mask (popcount 32) -> NULL w.p. 1/2; when released under uniform P,
    # s^2 = S^2 and Delta = S^2/(2B) = 64 S^2 for B = 1/128.
    mask = orc.pac_hash(np.array([99], dtype=np.int64), 5)[0]
    S = 1000
    cnt = np.zeros((1, 64), dtype=np.int64)
    sm = np.zeros((1, 64), dtype=np.int64)
    bits = np.array([(int(mask) >> j) & 1 for j in range(64)])
    cnt[0] = bits
    sm[0] = bits * S
    t = _table([AGG_SUM_I64], [mask], [1], cnt, [sm])
    nulls, deltas = 0, []
    for seed in range(400):
        jstar, _, P = orc.session(seed)
        rel, isn, flags, delta, P2 = orc.finalize(seed, B, jstar, P, t)
        if isn[0, 0]:
            nulls += 1
        else:
            deltas.append(delta[0, 0])
    assert stats.binomtest(nulls, 400, 0.5).pvalue > 1e-4
    np.testing.assert_allclose(deltas, 64.0 * S * S, rtol=1e-14)


def test_null_mechanism_rates(orc):
    # NULL with probability (64 - popcount K)/64, independent of the secret.
    K16 = np.uint64(0xFFFF)
    worlds = np.ones((3, 64), dtype=np.int64)
    t = _table([AGG_COUNT], [np.uint64(0), FULL, K16], [1, 100, 100], worlds, [None])
    counts = np.zeros(3)
    n = 2000
    for seed in range(n):
        jstar, _, P = orc.session(seed)
        _, isn, _, _, _ = orc.finalize(seed, B, jstar, P, t)
        counts += isn[:, 0]
    assert counts[0] == n          # K = 0 -> always NULL
    assert counts[1] == 0          # K full -> never NULL
    assert stats.binomtest(int(counts[2]), n, 0.75).pvalue > 1e-4


def test_noise_std_is_calibrated(orc):
    # y~ - y_{j*} ~ N(0, s^2/(2B)).  Over many sessions the standardised
    # noise has std 1 (within 3%) and passes a KS test.
    y = np.arange(64, dtype=np.int64)         # COUNT y_j = 2*j -> s^2 = 4*341.25
    t = _table([AGG_COUNT], [FULL], [1000], y.reshape(1, 64), [None])
    z = []
    for seed in range(6000):
        jstar, _, P = orc.session(seed)
        rel, isn, _, delta, _ = orc.finalize(seed, B, jstar, P, t)
        assert delta[0, 0] == pytest.approx(4 * 341.25 / (2 * B), rel=1e-13)
        z.append((rel[0, 0] - 2.0 * jstar) / math.sqrt(delta[0, 0]))
    z = np.array(z)
    assert abs(z.std() - 1.0) < 0.03
    assert stats.kstest(z, "norm").pvalue > 1e-4


def test_constant_vector_releases_exactly_and_keeps_posterior(orc):
    # R11 / S:L250: zero variance -> exact release, no Bayesian step.
    ext = np.full((1, 64), 12.5)
    t = _table([AGG_MAX_F64], [FULL], [500], np.ones((1, 64)), [ext])
    jstar, _, P = orc.session(7)
    rel, isn, _, delta, P2 = orc.finalize(7, B, jstar, P, t)
    assert isn[0, 0] == 0 and rel[0, 0] == 12.5 and delta[0, 0] == 0.0
    assert np.array_equal(P2, P)


def test_y_vector_scaling_and_unset_worlds(orc):
    # R7: COUNT/SUM doubled, AVG per-world mean, MIN/MAX raw; unset K bits read 0.
    K = np.uint64(0x00000000FFFFFFFF)
    cnt = np.arange(1, 65, dtype=np.int64).reshape(1, 64)
    s = (10 * np.arange(1, 65, dtype=np.int64)).reshape(1, 64)
    f = (0.5 * np.arange(1, 65, dtype=np.float64)).reshape(1, 64)
    t = _table([AGG_COUNT, AGG_SUM_I64, AGG_AVG_F64, AGG_MIN_F64], [K], [64], cnt, [None, s, f, f])
    y0, y1, y2, y3 = (orc.y_vector(t, a, 0) for a in range(4))
    assert np.array_equal(y0[:32], 2.0 * cnt[0, :32]) and np.all(y0[32:] == 0)
    assert np.array_equal(y1[:32], 2.0 * s[0, :32]) and np.all(y1[32:] == 0)
    assert np.array_equal(y2[:32], f[0, :32] / cnt[0, :32]) and np.all(y2[32:] == 0)
    assert np.array_equal(y3[:32], f[0, :32]) and np.all(y3[32:] == 0)


def test_posterior_stays_a_distribution_over_many_releases(orc):
    # sum P = 1 +- 1e-12 after thousands of chained releases (C5 reading R17).
    rng = np.random.default_rng(3)
    G = 100
    cnt = rng.integers(1000, 2000, (G, 64)).astype(np.int64)
    s = rng.integers(10**6, 10**7, (G, 64)).astype(np.int64)
    t = _table([AGG_SUM_I64, AGG_COUNT], [FULL] * G, [5000] * G, cnt, [s, None])
    jstar, _, P = orc.session(11)
    for rnd in range(20):
        _, _, _, _, P = orc.finalize(11, B, jstar, P, t, round_=rnd)
        assert abs(P.sum() - 1.0) < 1e-12 and np.all(P >= 0)
    # releases concentrate the posterior on the secret world (composition)
    assert np.argmax(P) == jstar


def test_diversity_flag(orc):
    # P:L1808-1810 with R18 thresholds: rows >= 64 and popcount K <= 34.
    m32 = orc.pac_hash(np.array([5], dtype=np.int64), 1)[0]
    t = _table([AGG_COUNT], [m32, m32, FULL], [1000, 3, 1000], np.ones((3, 64)), [None])
    _, _, flags, _, _ = orc.finalize(1, B, 0, np.full(64, 1 / 64), t)
    assert list(flags) == [1, 0, 0]
