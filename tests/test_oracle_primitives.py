"""Pins for the oracle's primitives: Philox4x32-10, fmix64, pac_hash, session.

Each check compares against something other than the oracle itself: published
known-answer vectors, closed forms of the uniform balanced-word distribution
(hypergeometric, via scipy), or invariants the paper states.
"""
import math

import numpy as np
import pytest
from scipy import stats

from conftest import golden_path


def _read_hex_rows(name):
    rows = []
    for line in open(golden_path(name)):
        line = line.split("#")[0].strip()
        if line:
            rows.append([int(t, 16) for t in line.split()])
    return rows


def test_philox_known_answer_vectors(orc):
    # tests/golden/philox4x32_10_kat.txt (Random123 kat_vectors, SC'11)
    for r in _read_hex_rows("philox4x32_10_kat.txt"):
        assert orc.philox(r[0:4], r[4:6]) == r[6:10]


def test_fmix64_is_splitmix64_finalizer(orc):
    # tests/golden/splitmix64_seed0.txt: SplitMix64 outputs for state 0
    outs = [r[0] for r in _read_hex_rows("splitmix64_seed0.txt")]
    gamma = 0x9E3779B97F4A7C15
    for k, ref in enumerate(outs, start=1):
        assert orc.fmix64((k * gamma) & 0xFFFFFFFFFFFFFFFF) == ref


SALT = 0x243F6A8885A308D3


def _popcount(a):
    a = a.astype(np.uint64)
    return np.unpackbits(a.view(np.uint8).reshape(-1, 8), axis=1).sum(axis=1)


def _bits(masks):
    """(n, 64) 0/1 matrix, column j = world j (LSB = world 0, reading R3)."""
    return np.unpackbits(masks.astype(np.uint64).view(np.uint8).reshape(-1, 8), axis=1,
                         bitorder="little").astype(np.int8)


@pytest.fixture(scope="module")
def seq_masks(orc):
    return orc.pac_hash(np.arange(1_000_000, dtype=np.int64), SALT)


def test_pac_hash_popcount_32_every_key(orc, seq_masks):
    # P:L93 (§2): "guaranteed to have 32 0- and 32 1-bits"
    assert np.all(_popcount(seq_masks) == 32)
    adversarial = np.array([0, -1, 1, 2, np.iinfo(np.int64).min, np.iinfo(np.int64).max,
                            0x5555555555555555, -0x5555555555555556], dtype=np.int64)
    for salt in (0, SALT, 0xFFFFFFFFFFFFFFFF):
        assert np.all(_popcount(orc.pac_hash(adversarial, salt)) == 32)
    rng = np.random.default_rng(1)
    rnd = rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, 200_000, dtype=np.int64)
    assert np.all(_popcount(orc.pac_hash(rnd, 12345)) == 32)


def test_pac_hash_fixed_point_and_majority_flips(orc):
    # Balancing only flips bits of the majority polarity, exactly |c-32| of them, and
    # leaves an already balanced hash alone ("transform ... guaranteed 32/32").
    keys = np.arange(-50_000, 50_000, dtype=np.int64)
    x = np.array([orc.fmix64(int(k) ^ SALT) for k in keys.view(np.uint64)], dtype=np.uint64)
    m = orc.pac_hash(keys, SALT)
    c = _popcount(x).astype(np.int64)
    flipped = x ^ m
    nflip = _popcount(flipped)
    assert np.all(nflip == np.abs(c - 32))
    fixed = c == 32
    assert fixed.sum() > 5000          # ~9.9% of keys are already balanced
    assert np.all(m[fixed] == x[fixed])
    maj_ones = c > 32
    # every flipped bit had the majority value in x
    assert np.all((flipped[maj_ones] & ~x[maj_ones]) == 0)
    assert np.all((flipped[~maj_ones & ~fixed] & x[~maj_ones & ~fixed]) == 0)


def test_pac_hash_matches_uniform_balanced_word_statistics(seq_masks):
    # §4: the induced subsets should be distributed like SamplePU's balanced
    # construction.  For a uniform balanced 64-bit word:
    #  * each bit is 1 w.p. 1/2;
    #  * two distinct bits have correlation -1/63;
    #  * the popcount of any fixed 8-bit window is hypergeometric(64, 32, 8).
    B = _bits(seq_masks).astype(np.float64)
    freq = B.mean(axis=0)
    assert np.max(np.abs(freq - 0.5)) < 0.005
    C = np.corrcoef(B, rowvar=False)
    off = C[~np.eye(64, dtype=bool)]
    assert np.max(np.abs(off + 1.0 / 63.0)) < 0.01
    hg = stats.hypergeom(64, 32, 8)
    for byte in (0, 3, 7):
        cnt = B[:, 8 * byte:8 * byte + 8].sum(axis=1).astype(int)
        obs = np.bincount(cnt, minlength=9)
        exp = np.array([hg.pmf(t) for t in range(9)]) * len(cnt)
        keep = exp > 5
        chi2 = (((obs - exp) ** 2) / exp)[keep].sum()
        assert chi2 < stats.chi2.ppf(0.9999, keep.sum() - 1)


def test_pac_hash_world_fractions_and_salt_independence(orc, seq_masks):
    # S:L203 idea: each world holds about half of a 1e4-PU population;
    # a new salt "virtually shuffles" the worlds -> ~50% agreement.
    B = _bits(seq_masks[:10_000])
    frac = B.mean(axis=0)
    assert frac.min() >= 0.48 and frac.max() <= 0.52
    other = orc.pac_hash(np.arange(1_000_000, dtype=np.int64), SALT ^ 0x1234567)
    agree = 1.0 - _popcount(seq_masks ^ other).mean() / 64.0
    assert abs(agree - 0.5) < 0.002


def test_pac_hash_deterministic(orc):
    k = np.array([7, 7, 123456789], dtype=np.int64)
    a = orc.pac_hash(k, 99)
    assert a[0] == a[1]
    assert np.array_equal(a, orc.pac_hash(k, 99))


def test_session_draws_and_uniform_prior(orc):
    # j* uniform over the m worlds, P = (1/m, ...).
    js = np.array([orc.session(s)[0] for s in range(6400)])
    assert js.min() == 0 and js.max() == 63
    obs = np.bincount(js, minlength=64)
    chi2 = ((obs - 100.0) ** 2 / 100.0).sum()
    assert chi2 < stats.chi2.ppf(0.9999, 63)
    j, salt, P = orc.session(42)
    assert np.all(P == 1.0 / 64)
    assert orc.session(42)[:2] == (j, salt)
    assert orc.session(43)[1] != salt


def test_box_muller_normal_is_standard_normal(orc):
    # R13 Box-Muller on Philox blocks -> N(0,1) (Kolmogorov-Smirnov vs scipy).
    z = np.array([orc.normal_from_block(orc.philox([i, 0, 7, 0], [5, 6])) for i in range(20000)])
    assert stats.kstest(z, "norm").pvalue > 1e-4
    assert abs(z.mean()) < 0.03 and abs(z.std() - 1.0) < 0.03
