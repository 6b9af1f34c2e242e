"""Pins of the oracle's approximate 64-world SUM (§8 f3; R35, R36).

Independent of the oracle's own arithmetic:
  - exact regime: every |v| < 2^12 (routed to level 0 unchanged) and no counter ever reaches 2^16
    (small inputs): the state decodes to the exact sum -- numpy's, world by world;
  - error bound (P:L1790 states 2^-12 per cascade; routing keeps >= 9 significant bits): for any
    input |y_j - 2 sum_j v| <= 2 (2^-8 + 2^-12) sum_j |v| -- checked against numpy's exact sums;
  - two-sided (R35): positive-only input leaves the negative side empty; the sides are independent
    (negating the input swaps them);
  - Table 1's contrast: on a mixed-sign column the single-sided sum (R36: the
    two's-complement pattern of a negative value has msb 63) fails -- error of the order of the
    negative mass -- while the two-sided one stays within the bound; on positive-only columns the
    two variants coincide."""
import numpy as np
import pytest


def _bits(masks):
    return np.unpackbits(masks.astype(np.uint64).view(np.uint8).reshape(-1, 8), axis=1, bitorder="little").astype(bool)


def _world_sums(masks, v):
    B = _bits(masks)
    return np.array([int(v[B[:, j]].astype(object).sum()) for j in range(64)], dtype=object), \
        np.array([int(np.abs(v[B[:, j]]).astype(object).sum()) for j in range(64)], dtype=object)


def test_exact_regime_equals_numpy_sum(orc):
    rng = np.random.default_rng(1)
    n = 60
    v = rng.integers(-4095, 4096, n).astype(np.int64)
    masks = orc.pac_hash(rng.integers(0, 50, n).astype(np.int64), 9)
    _, y = orc.approx_sum(masks, v, block_rows=16)  # blocks combined too
    exact, _ = _world_sums(masks, v)
    B = _bits(masks)
    checked = 0
    for j in range(64):  # a side's level 0 never overflows while its total stays below 2^16 - 2^12
        pos = int(v[B[:, j] & (v > 0)].sum())
        neg = int(-v[B[:, j] & (v < 0)].sum())
        if pos < 61440 and neg < 61440:
            assert y[j] == 2 * exact[j]
            checked += 1
    assert checked > 0
    # single-sided, positive values only: the same state as the two-sided pos side
    vp = np.abs(v) + 1
    c1, y1 = orc.approx_sum(masks, vp, block_rows=16, two_sided=False)
    c2, y2 = orc.approx_sum(masks, vp, block_rows=16, two_sided=True)
    assert np.array_equal(c1, c2) and np.array_equal(y1, y2)


@pytest.mark.parametrize("two_sided", [True, False])
@pytest.mark.parametrize("dist", ["uniform_int", "uniform_bigint", "exponential", "all_same"])
def test_error_bound(orc, two_sided, dist):  # positive columns: both variants within the bound
    if not two_sided and dist == "uniform_bigint":
        pytest.skip("world sums ~5e19 exceed int64: the single sum decodes modulo 2^64 (R36)")
    rng = np.random.default_rng(2)
    n = 200_000
    v = {"uniform_int": lambda: rng.integers(1, 2**31, n),
         "uniform_bigint": lambda: rng.integers(1, 2**50, n),
         "exponential": lambda: rng.exponential(1e6, n).astype(np.int64) + 1,
         "all_same": lambda: np.full(n, 123_456_789)}[dist]().astype(np.int64)
    masks = orc.pac_hash(rng.integers(0, 5000, n).astype(np.int64), 3)
    _, y = orc.approx_sum(masks, v, block_rows=4096, two_sided=two_sided)
    exact, absum = _world_sums(masks, v)
    for j in range(64):
        err = abs(float(y[j]) - 2.0 * float(exact[j]))
        assert err <= 2.0 * (2.0**-8 + 2.0**-12) * float(absum[j]) + 1e-6, (j, err, float(absum[j]))


def test_two_sided_sides(orc):
    rng = np.random.default_rng(3)
    n = 50_000
    v = rng.integers(1, 10**9, n).astype(np.int64)
    masks = orc.pac_hash(rng.integers(0, 900, n).astype(np.int64), 5)
    c, y = orc.approx_sum(masks, v, block_rows=1000)
    assert np.all(c[1] == 0) and np.any(c[0] != 0)
    c2, y2 = orc.approx_sum(masks, -v, block_rows=1000)
    assert np.array_equal(c2[1], c[0]) and np.all(c2[0] == 0)
    np.testing.assert_array_equal(y2, -y)


def test_table1_contrast_negative_mixed(orc):
    # P:L1968-1991 Table 1, "negative_mixed": two-sided keeps the error small where the single sum
    # (signed counters) fails -- large positive and negative values that cancel
    rng = np.random.default_rng(4)
    n = 400_000
    v = np.where(rng.random(n) < 0.5, rng.integers(10**8, 10**9, n), -rng.integers(10**8, 10**9, n)).astype(np.int64)
    masks = orc.pac_hash(rng.integers(0, 20_000, n).astype(np.int64), 7)
    exact, absum = _world_sums(masks, v)
    _, y1 = orc.approx_sum(masks, v, block_rows=65536, two_sided=False)
    _, y2 = orc.approx_sum(masks, v, block_rows=65536, two_sided=True)
    e1 = np.array([abs(float(y1[j]) - 2.0 * float(exact[j])) for j in range(64)])
    e2 = np.array([abs(float(y2[j]) - 2.0 * float(exact[j])) for j in range(64)])
    ab = np.array([float(a) for a in absum])
    assert np.all(e2 <= 2.0 * (2.0**-8 + 2.0**-12) * ab)
    assert np.all(e1 > 0.1 * ab)  # the single sum loses the negative values' low 52 bits
