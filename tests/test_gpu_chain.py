"""Release chain (a6-a7) edge behaviour against the oracle: the posterior collapsing to one
world (after which k_finalize_tail releases the rest cell-parallel, R11) and NaN world values
(R11's equality test as the oracle states it: every y_j with P_j > 0 equal to the first)."""
import numpy as np
import pytest

from gpu_helpers import assert_releases_close, to_dev

pytestmark = pytest.mark.gpu

import paper_2603_15023_b200 as pac  # noqa: E402

FULL = np.uint64(2**64 - 1)


def _dev_u64(a):
    return to_dev(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64))


def _single_pu_vectors(rng, n):
    """y_j = v * [j in a random 32-world set]: one PU per group, the C3 long tail's shape."""
    bits = np.zeros((n, 64))
    for i in range(n):
        bits[i, rng.permutation(64)[:32]] = 1.0
    return bits * rng.integers(1, 10**6, n)[:, None]


def _masked(y, pres):
    return np.where(((pres[:, None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)) == 1, y, 0.0)


def _run(orc, s, seed, jstar, P, y, pres, rnd):
    rel, isn, delta = pac.noised_y(s, to_dev(np.ascontiguousarray(y)), _dev_u64(pres), rnd)
    r_o, n_o, d_o, P = orc.noised_y(seed, 1 / 128, jstar, P, _masked(y, pres), pres, rnd)
    return rel.cpu().numpy(), isn.cpu().numpy(), delta.cpu().numpy(), r_o, n_o, d_o, P


def test_collapse_to_one_world_then_parallel_tail(orc):
    seed = 77
    jstar, _, P = orc.session(seed)
    s = pac.Session(seed)
    rng = np.random.default_rng(3)
    n = 4000
    y = _single_pu_vectors(rng, n)
    pres = np.full(n, FULL, dtype=np.uint64)
    pres[::7] = np.uint64(0xFFFFFFFF)  # NULL cells on both sides of the collapse
    for rnd in range(2):  # round 1 starts collapsed: the whole chain is the parallel tail
        rel, isn, delta, r_o, n_o, d_o, P = _run(orc, s, seed, jstar, P, y, pres, rnd)
        assert_releases_close(rel, r_o, d_o, isn, n_o)
        np.testing.assert_array_equal(np.isnan(delta), np.isnan(d_o))
        ok = n_o == 0
        np.testing.assert_allclose(delta[ok], d_o[ok], rtol=1e-9, atol=0)
        q = s.query()
        np.testing.assert_allclose(q["P"], P, rtol=0, atol=1e-9)
        assert (P > 0).sum() == 1  # the oracle's posterior collapsed in round 0
        if rnd == 0:
            released = q["releases"]
            assert 0 < released < n
            zv = np.flatnonzero(ok & (d_o == 0))
            assert zv.size > n // 2 and np.array_equal(rel[zv], _masked(y, pres)[zv, jstar])
        else:
            assert q["releases"] == released  # nothing released with noise after the collapse


def test_nan_world_values_follow_the_oracle(orc):
    seed = 5150
    jstar, _, P = orc.session(seed)
    s = pac.Session(seed)
    rng = np.random.default_rng(9)
    n = 1500
    y = _single_pu_vectors(rng, n)
    y[1000:1010, (jstar + 1) % 64] = np.nan  # after the collapse: only j*'s world is in the support
    y[1200:1205, jstar] = np.nan
    y[1400:, :] = np.where(rng.random((100, 64)) < 0.1, np.nan, y[1400:, :])
    pres = np.full(n, FULL, dtype=np.uint64)
    for rnd in range(2):
        rel, isn, delta, r_o, n_o, d_o, P = _run(orc, s, seed, jstar, P, y, pres, rnd)
        np.testing.assert_array_equal(isn, n_o)
        np.testing.assert_array_equal(np.isnan(rel), np.isnan(r_o))
        np.testing.assert_array_equal(np.isnan(delta), np.isnan(d_o))
        f = ~np.isnan(r_o)
        scale = np.maximum(np.maximum(np.abs(rel[f]), np.abs(r_o[f])), np.sqrt(np.abs(np.nan_to_num(d_o[f]))))
        assert np.all(np.abs(rel[f] - r_o[f]) <= 1e-9 * np.maximum(scale, 1e-300))
        np.testing.assert_allclose(s.query()["P"], P, rtol=0, atol=1e-9, equal_nan=True)


def test_nan_before_collapse_poisons_posterior_like_the_oracle(orc):
    seed = 99
    jstar, _, P = orc.session(seed)
    s = pac.Session(seed)
    rng = np.random.default_rng(4)
    n = 200
    y = _single_pu_vectors(rng, n)
    y[20, (jstar + 3) % 64] = np.nan  # support still has many worlds: Var = NaN, P -> NaN
    pres = np.full(n, FULL, dtype=np.uint64)
    rel, isn, delta, r_o, n_o, d_o, P = _run(orc, s, seed, jstar, P, y, pres, 0)
    np.testing.assert_array_equal(np.isnan(rel), np.isnan(r_o))
    np.testing.assert_array_equal(np.isnan(delta), np.isnan(d_o))
    f = ~np.isnan(r_o)
    np.testing.assert_allclose(rel[f], r_o[f], rtol=1e-9, atol=0)
    np.testing.assert_array_equal(np.isnan(s.query()["P"]), np.isnan(P))


def test_table_chain_collapse_and_tail_match_oracle(orc):
    """pac_finalize on a C3-shaped table (many small groups): the chain derives y from the table
    rows, the posterior collapses within the first call and k_finalize_tail releases the rest;
    the second call starts collapsed (tail only).  Parity with the oracle both times."""
    import datagen as dg
    from gpu_helpers import run_gpu, workload_aggs
    w = dg.WORKLOADS["C3"]
    cols = w.host_columns(0, 400_000)
    aggs = workload_aggs(w, cols)
    seed = 2024
    jstar, salt, P = orc.session(seed)
    s = pac.Session(seed, w.budget)
    t, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=salt, G_cap=1 << 17)
    ref = orc.agg(orc.pac_hash(cols["pu"], salt), cols["keys"], aggs)
    G = ref["G"]
    fin = pac.Finalizer(t.kinds, t.G_cap)
    for rnd in range(2):
        rel, isn, flags, delta = fin(s, t, rnd)
        r_o, n_o, f_o, d_o, P = orc.finalize(seed, w.budget, jstar, P, ref, rnd)
        rel = rel[:G].cpu().numpy()
        isn = isn[:G].cpu().numpy()
        assert_releases_close(rel, r_o, d_o, isn, n_o)
        np.testing.assert_array_equal(flags[:G].cpu().numpy(), f_o)
        np.testing.assert_allclose(s.query()["P"], P, rtol=0, atol=1e-9)
    assert (P > 0).sum() == 1  # collapsed: the tail kernel carried most of both calls
