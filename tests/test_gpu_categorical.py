"""-m gpu parity of the categorical path (§8 f1; R22-R26) through the C-ABI against the
oracle on the same inputs: world vectors of a table (exact), vector lifting (bit-exact: one
IEEE operation per world), lifted comparisons, the comparison index + fused row-parallel
pac_select_cmp / pac_filter_cmp (bit-exact masks and booleans, with ties, NaN, +-inf and
partial presence), pac_select / pac_filter, pac_noised of lifted vectors (releases per R16,
posterior 1e-9), the Q17-shaped chain (inner AVG -> select_cmp -> outer SUM through the
reduced masks), and the paper's ratio-lambda claim on the GPU path."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import REL_F64, assert_releases_close, assert_tables_equal, run_gpu, to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_15023_b200 as pac  # noqa: E402

FULL = (1 << 64) - 1
CMPS = [pac.CMP_LT, pac.CMP_LE, pac.CMP_GT, pac.CMP_GE, pac.CMP_EQ]


def _u64(t):
    return pac.as_u64(t)


def _dev_u64(a):
    return to_dev(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64))


def _table(orc, n=60_000, seed=1, G=6):
    rng = np.random.default_rng(seed)
    pu = rng.integers(0, 3000, n).astype(np.int64)
    keys = [rng.integers(0, G, n).astype(np.int16)]
    iv = rng.integers(1, 10**5, n).astype(np.int64)
    fv = rng.random(n)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv), (dg.AGG_AVG_F64, fv), (dg.AGG_MAX_F64, fv)]
    t, _ = run_gpu(aggs, keys, pu=pu, salt=5, G_cap=64)
    ref = orc.agg(orc.pac_hash(pu, 5), keys, aggs)
    return t, ref


def test_world_vectors_exact(orc):
    t, ref = _table(orc)
    G = ref["G"]
    for a in range(4):
        y, p = pac.world_vector(t, a)
        yo, po = orc.world_vectors(ref, a)
        if ref["kinds"][a] == dg.AGG_AVG_F64:   # f64 world sums: <= 1e-9 relative (R16)
            np.testing.assert_allclose(y[:G].cpu().numpy(), yo, rtol=REL_F64, atol=0)
        else:                                   # counts, int64 sums, extremes: exact
            np.testing.assert_array_equal(y[:G].cpu().numpy(), yo)
        np.testing.assert_array_equal(_u64(p[:G]), po)
        assert np.all(_u64(p[G:]) == 0)


@pytest.mark.parametrize("op", [pac.OP_ADD, pac.OP_SUB, pac.OP_MUL, pac.OP_DIV, pac.OP_MIN, pac.OP_MAX])
def test_lift_bit_exact(orc, op):
    rng = np.random.default_rng(op)
    n = 777
    a = rng.normal(0, 100, (n, 64))
    b = rng.normal(0, 100, (n, 64))
    b[::7, 3] = 0.0
    pa = rng.integers(0, 2**63, n, dtype=np.int64).astype(np.uint64) | np.uint64(1 << 63)
    pb = np.full(n, FULL, dtype=np.uint64)
    pb[::5] = rng.integers(0, 2**63, len(pb[::5]), dtype=np.int64).astype(np.uint64)
    for A, B, oa, ob in (((to_dev(a), _dev_u64(pa)), (to_dev(b), _dev_u64(pb)), (a, pa), (b, pb)),
                         ((to_dev(a), _dev_u64(pa)), 2.5, (a, pa), 2.5),
                         (-1.25, (to_dev(b), _dev_u64(pb)), -1.25, (b, pb))):
        y, p = pac.lift(op, A, B)
        yo, po = orc.lift(op, oa, ob, n)
        np.testing.assert_array_equal(_u64(p), po)
        np.testing.assert_array_equal(y.cpu().numpy().view(np.uint64), yo.view(np.uint64))


@pytest.mark.parametrize("cmp", CMPS)
def test_lift_cmp_bit_exact(orc, cmp):
    rng = np.random.default_rng(10 + cmp)
    n = 500
    a = rng.integers(-3, 4, (n, 64)).astype(np.float64)
    b = rng.integers(-3, 4, (n, 64)).astype(np.float64)
    a[::9, 5] = np.nan
    pa = rng.integers(0, 2**63, n, dtype=np.int64).astype(np.uint64)
    pb = np.full(n, FULL, dtype=np.uint64)
    bits = pac.lift_cmp(cmp, (to_dev(a), _dev_u64(pa)), (to_dev(b), _dev_u64(pb)))
    np.testing.assert_array_equal(_u64(bits), orc.lift_cmp(cmp, (a, pa), (b, pb), n))
    bits = pac.lift_cmp(cmp, (to_dev(a), _dev_u64(pa)), 0.0)
    np.testing.assert_array_equal(_u64(bits), orc.lift_cmp(cmp, (a, pa), 0.0, n))


def _cmp_case(seed, G=40, n=200_003):
    rng = np.random.default_rng(seed)
    c = rng.integers(-20, 21, (G, 64)).astype(np.float64) / 4      # many ties
    c[rng.integers(0, G, 30), rng.integers(0, 64, 30)] = np.nan
    c[rng.integers(0, G, 10), rng.integers(0, 64, 10)] = np.inf
    c[rng.integers(0, G, 10), rng.integers(0, 64, 10)] = -np.inf
    c[3] = 1.0                                                     # constant vector
    pres = rng.integers(0, 2**63, G, dtype=np.int64).astype(np.uint64) * np.uint64(2)
    pres[:G // 2] = np.uint64(FULL)
    pres[4] = 0                                                    # nothing present
    v = rng.integers(-24, 25, n).astype(np.float64) / 4
    v[::101] = np.nan
    v[::103] = np.inf
    v[::107] = -np.inf
    v[::109] = -0.0
    g = rng.integers(0, G, n).astype(np.int32)
    h = rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64).astype(np.uint64)
    return c, pres, v, g, h


@pytest.mark.parametrize("cmp", CMPS)
def test_select_cmp_bit_exact(orc, cmp):
    c, pres, v, g, h = _cmp_case(20 + cmp)
    ix = pac.cmp_index(to_dev(c), _dev_u64(pres))
    out = pac.select_cmp(cmp, _dev_u64(h), to_dev(v), to_dev(g), ix)
    np.testing.assert_array_equal(_u64(out), orc.select_cmp(cmp, h, v, g, c, pres))


@pytest.mark.parametrize("cmp", CMPS)
def test_filter_cmp_bit_exact(orc, cmp):
    c, pres, v, g, _ = _cmp_case(30 + cmp)
    seed = 4242
    s = pac.Session(seed)
    ix = pac.cmp_index(to_dev(c), _dev_u64(pres))
    got = pac.filter_cmp(s, cmp, to_dev(v), to_dev(g), ix, round_=3).cpu().numpy()
    np.testing.assert_array_equal(got, orc.filter_cmp(seed, 3, cmp, v, g, c, pres))


def test_select_and_filter_bit_exact(orc):
    rng = np.random.default_rng(7)
    n, G = 300_001, 17
    bits = rng.integers(-(2**63), 2**63 - 1, G, dtype=np.int64).astype(np.uint64)
    bits[0], bits[1] = np.uint64(FULL), np.uint64(0)
    g = rng.integers(0, G, n).astype(np.int32)
    h = orc.pac_hash(rng.integers(0, 10**6, n).astype(np.int64), 9)
    out = pac.select(_dev_u64(h), to_dev(g), _dev_u64(bits))
    np.testing.assert_array_equal(_u64(out), orc.select(h, g, bits))
    per_row = rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64).astype(np.uint64)
    per_row[:64] = [np.uint64((1 << k) - 1) for k in range(64)]
    s = pac.Session(99)
    got = pac.pac_filter(s, _dev_u64(per_row), round_=1).cpu().numpy()
    np.testing.assert_array_equal(got, orc.pac_filter(99, 1, per_row))


def test_noised_lifted_vectors_match_oracle(orc):
    t, ref = _table(orc, seed=3)
    G = ref["G"]
    seed = 31337
    jstar, salt, P = orc.session(seed)
    s = pac.Session(seed)
    # market-share-like ratio: SUM / (COUNT) per world, plus a scaled AVG
    x, px = pac.world_vector(t, 1)
    y, py = pac.world_vector(t, 0)
    r, pr = pac.lift(pac.OP_DIV, (x[:G], px[:G]), (y[:G], py[:G]))
    xo, pxo = orc.world_vectors(ref, 1)
    yo, pyo = orc.world_vectors(ref, 0)
    ro, pro = orc.lift(orc.OP_DIV, (xo, pxo), (yo, pyo), G)
    for rnd in range(3):
        rel, isn, delta = pac.noised_y(s, r, pr, rnd)
        r_o, n_o, d_o, P = orc.noised_y(seed, 1 / 128, jstar, P, ro, pro, rnd)
        assert_releases_close(rel.cpu().numpy(), r_o, d_o, isn.cpu().numpy(), n_o)
        np.testing.assert_allclose(s.query()["P"], P, rtol=0, atol=1e-9)


def test_q17_chain_inner_avg_select_outer_sum(orc):
    """Q17 shape: per part, 0.2 * AVG(qty) over the part's lineitems (unfused
    world vector); each lineitem keeps world j iff qty < 0.2 * avg_j (pac_select_lt with
    the constant folded); the outer SUM aggregates through the reduced masks."""
    rng = np.random.default_rng(17)
    n, parts = 120_000, 50
    pu = rng.integers(0, 5000, n).astype(np.int64)
    part = rng.integers(0, parts, n).astype(np.int32)
    qty = rng.integers(1, 51, n).astype(np.float64)
    price = rng.integers(100, 10_000, n).astype(np.int64)
    salt = 77
    # inner: AVG(qty) GROUP BY part
    t, _ = run_gpu([(dg.AGG_AVG_F64, qty)], [part], pu=pu, salt=salt, G_cap=parts)
    ref = orc.agg(orc.pac_hash(pu, salt), [part], [(dg.AGG_AVG_F64, qty)])
    assert t.check() == ref["G"] == parts                      # part keys 0..49 are all present
    avg, pavg = pac.world_vector(t, 0)
    thr, pthr = pac.lift(pac.OP_MUL, (avg[:parts], pavg[:parts]), 0.2)
    avg_o, pavg_o = orc.world_vectors(ref, 0)
    thr_o, pthr_o = orc.lift(orc.OP_MUL, (avg_o, pavg_o), 0.2, parts)
    np.testing.assert_allclose(thr.cpu().numpy(), thr_o, rtol=REL_F64, atol=0)  # f64 AVG (R16)
    np.testing.assert_array_equal(_u64(pthr), pthr_o)
    # from here both sides take the same threshold vectors (a comparison decides bits)
    thr_o = thr.cpu().numpy()
    # rows: keep world j iff qty < thr_j of the row's part (group index == part id here)
    h = pac.mask(to_dev(pu), salt)
    ix = pac.cmp_index(thr, pthr)
    hr = pac.select_cmp(pac.CMP_LT, h, to_dev(qty), to_dev(part), ix)
    hr_o = orc.select_cmp(orc.CMP_LT, orc.pac_hash(pu, salt), qty, part, thr_o, pthr_o)
    np.testing.assert_array_equal(_u64(hr), hr_o)
    # outer: SUM(price) over the reduced masks (rows with mask 0 dropped, R21)
    ag = pac.Aggregator([pac.SUM_I64], 1)
    tt = ag([to_dev(price)], [], mask=hr)
    ref2 = orc.agg(hr_o, [], [(dg.AGG_SUM_I64, price)])
    assert_tables_equal(tt.to_host(), ref2)


def test_ratio_noised_once_beats_twice_on_gpu(orc):
    rng = np.random.default_rng(11)
    n = 200_000
    pu = rng.integers(0, 20_000, n).astype(np.int64)
    e = rng.integers(1, 1000, n).astype(np.int64)
    ei = np.where(rng.random(n) < 0.3, e, 0).astype(np.int64)
    exact = ei.sum() / e.sum()
    once, twice = [], []
    for sd in range(40):
        s = pac.Session(500 + sd)
        t, _ = run_gpu([(dg.AGG_SUM_I64, ei), (dg.AGG_SUM_I64, e)], [], pu=pu, salt=s.salt, G_cap=1)
        x, px = pac.world_vector(t, 0)
        y, py = pac.world_vector(t, 1)
        r, pr = pac.lift(pac.OP_DIV, (x, px), (y, py))
        rel, isn, _ = pac.noised_y(s, r, pr)
        s2 = pac.Session(500 + sd)
        rel2, isn2, _, _ = pac.finalize(s2, t)
        if int(isn[0]) or int(isn2[0].sum()):
            continue
        once.append(abs(float(rel[0]) - exact) / exact)
        twice.append(abs(float(rel2[0, 0]) / float(rel2[0, 1]) - exact) / exact)
    assert len(once) > 30 and np.mean(once) < np.mean(twice)


def test_noised_chain_far_offsets_and_absent_secret_world(orc):
    """The release chain's variance: large offsets with a small spread (shifted one-pass about
    y_{j*}), the secret world absent (y_{j*} = 0 far from the mean: the two-pass branch), and
    single-outlier cells, chained over 3000 releases against the oracle's two-pass (R8, R16)."""
    seed = 4242
    jstar, _, P = orc.session(seed)
    s = pac.Session(seed)
    rng = np.random.default_rng(8)
    n = 3000
    kind = np.arange(n) % 3
    y = 1e12 + rng.standard_normal((n, 64)) * 1e3
    y[kind == 2] = rng.integers(0, 100, (int((kind == 2).sum()), 64)).astype(np.float64)
    y[kind == 2, 5] = 1e9  # one outlier world
    pres = rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64).astype(np.uint64)
    pres |= np.uint64(0xFFFF_FFFF_FFFF_0000)  # mostly present (NULL rate ~ (64 - pc) / 64)
    bit = np.uint64(1) << np.uint64(jstar)
    pres[kind == 1] &= ~bit  # y_{j*} reads 0 (R9) while the other worlds sit near 1e12
    pres[kind != 1] |= bit
    yo = np.where(((pres[:, None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)) == 1, y, 0.0)
    rel, isn, delta = pac.noised_y(s, to_dev(np.ascontiguousarray(y)), _dev_u64(pres))
    r_o, n_o, d_o, P_o = orc.noised_y(seed, 1 / 128, jstar, P, yo, pres)
    assert_releases_close(rel.cpu().numpy(), r_o, d_o, isn.cpu().numpy(), n_o)
    np.testing.assert_allclose(delta.cpu().numpy()[n_o == 0], d_o[n_o == 0], rtol=1e-9, atol=0)
    np.testing.assert_allclose(s.query()["P"], P_o, rtol=0, atol=1e-9)
