"""-m gpu parity of m = 128 worlds (§8 f4; readings R28, R29) through the C-ABI against the oracle:
the 128-bit balanced hash (bit-exact), the 128-world grouped aggregation on BASELINE-shaped
inputs and on explicit masks with one zero half / both halves zero (bit-exact integers,
f64 within 1e-9), and finalize over 128 worlds with an m = 128 session (releases per R16,
posterior 1e-9) over several rounds.  COUNT / SUM / AVG with G_cap <= 32 take the native single-pass
kernel (k_agg_tiles128): checked against the oracle, against the three-pass path
(PAC_NO_NATIVE128=1) and at its edges (32 groups, several tiles with a ragged tail, empty input,
capacity overflow)."""
import os

import numpy as np
import pytest

import datagen as dg
from gpu_helpers import REL_F64, assert_releases_close, to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_15023_b200 as pac  # noqa: E402


def _dev_vals(aggs):
    """one device copy per host column (aggregates may share a column, e.g. MIN + MAX)"""
    cache = {}
    out = []
    for _, v in aggs:
        if v is None:
            out.append(None)
        else:
            if id(v) not in cache:
                cache[id(v)] = to_dev(v)
            out.append(cache[id(v)])
    return out


def _cmp(got, ref):
    assert got["G"] == ref["G"]
    np.testing.assert_array_equal(got["keys"], ref["keys"])
    np.testing.assert_array_equal(got["rows"], ref["rows"])
    np.testing.assert_array_equal(got["K"], ref["K"])
    if ref["count"] is not None and got["count"] is not None:
        np.testing.assert_array_equal(got["count"], ref["count"])
    for a, k in enumerate(ref["kinds"]):
        if k == dg.AGG_COUNT:
            continue
        if k in (dg.AGG_SUM_I64, dg.AGG_MIN_F64, dg.AGG_MAX_F64):
            np.testing.assert_array_equal(got["world"][a], ref["world"][a])
        else:
            np.testing.assert_allclose(got["world"][a], ref["world"][a], rtol=REL_F64, atol=1e-300)


def test_mask128_bit_exact(orc):
    rng = np.random.default_rng(0)
    keys = np.concatenate([np.arange(300_000, dtype=np.int64),
                           rng.integers(-(2**63), 2**63 - 1, 300_001, dtype=np.int64),
                           np.array([0, -1, np.iinfo(np.int64).min], dtype=np.int64)])
    for salt in (0x243F6A8885A308D3, 0):
        got = pac.as_u64(pac.mask128(to_dev(keys), salt)).reshape(-1, 2)
        np.testing.assert_array_equal(got, orc.pac_hash128(keys, salt))


@pytest.mark.parametrize("cfg,n,G_cap", [("C2", 300_007, 8), ("C5", 200_003, 128), ("C1", 100_001, 1)])
def test_agg128_workloads(orc, cfg, n, G_cap):
    w = dg.WORKLOADS[cfg]
    cols = w.host_columns(0, n)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    salt = 0x5EED
    ag = pac.Aggregator128([k for k, _ in aggs], G_cap)
    t = ag(_dev_vals(aggs), [to_dev(k) for k in cols["keys"]],
           pu_key=to_dev(cols["pu"]), salt=salt)
    _cmp(t.to_host(), orc.agg128(orc.pac_hash128(cols["pu"], salt), cols["keys"], aggs))


def test_agg128_explicit_masks_with_zero_halves(orc):
    rng = np.random.default_rng(4)
    n = 120_000
    m = orc.pac_hash128(rng.integers(0, 2000, n).astype(np.int64), 3)
    m[::7, 0] = 0                  # worlds 0..63 empty for these rows
    m[3::11, 1] = 0                # worlds 64..127 empty
    m[5::13] = 0                   # in no world: dropped (R21)
    keys = [rng.integers(0, 6, n).astype(np.int8)]
    keys[0][5::13] = 99            # a group reached only by dropped rows: absent
    iv = rng.integers(-10**6, 10**6, n).astype(np.int64)
    fv = rng.normal(3, 1, n)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv), (dg.AGG_AVG_F64, fv), (dg.AGG_MIN_F64, fv),
            (dg.AGG_MAX_F64, fv)]
    ag = pac.Aggregator128([k for k, _ in aggs], 16)
    t = ag(_dev_vals(aggs), [to_dev(keys[0])],
           mask2=to_dev(np.ascontiguousarray(m).view(np.int64)))
    _cmp(t.to_host(), orc.agg128(m, keys, aggs))


def test_finalize128_matches_oracle(orc):
    w = dg.WORKLOADS["C2"]
    cols = w.host_columns(0, 150_000)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    seed = 2718
    jstar, salt, P = orc.session128(seed)
    s = pac.Session(seed, w.budget, m=128)
    assert (s.salt, s.jstar) == (salt, jstar)
    ag = pac.Aggregator128([k for k, _ in aggs], 8)
    t = ag(_dev_vals(aggs), [to_dev(k) for k in cols["keys"]],
           pu_key=to_dev(cols["pu"]), salt=salt)
    ref = orc.agg128(orc.pac_hash128(cols["pu"], salt), cols["keys"], aggs)
    G = ref["G"]
    fin = pac.Finalizer(t.kinds, t.G_cap)
    for rnd in range(3):
        rel, isn, flags, delta = fin(s, t, rnd)
        r_o, n_o, f_o, d_o, P = orc.finalize128(seed, w.budget, jstar, P, ref, rnd)
        assert_releases_close(rel[:G].cpu().numpy(), r_o, d_o, isn[:G].cpu().numpy(), n_o)
        np.testing.assert_array_equal(flags[:G].cpu().numpy(), f_o)
        np.testing.assert_allclose(s.query()["P"], P, rtol=0, atol=1e-9)


def test_m_mismatch_is_rejected():
    s64 = pac.Session(1)
    ag = pac.Aggregator128([pac.COUNT], 4)
    t = ag([None], [], pu_key=to_dev(np.arange(100, dtype=np.int64)), salt=1)
    with pytest.raises(pac.PacError):
        pac.Finalizer(t.kinds, t.G_cap)(s64, t)


def _last_kernel(fn):
    pac.profile_enable(True)
    try:
        out = fn()
        torch.cuda.synchronize()
        return out, pac.profile_last_kernel()
    finally:
        pac.profile_enable(False)


@pytest.mark.parametrize("n", [0, 1, 1023, 1025, 333_333])
def test_native128_explicit_masks_32_groups(orc, n):
    """the native kernel at its slot limit (32 groups), 2 int64 + 2 f64 columns, zero halves"""
    rng = np.random.default_rng(n + 17)
    m = orc.pac_hash128(rng.integers(0, 5000, n).astype(np.int64), 9)
    if n:
        m[::5, 0] = 0
        m[2::9, 1] = 0
        m[4::17] = 0
    keys = [rng.integers(0, 32, n).astype(np.int16)]
    i1 = rng.integers(-(2**40), 2**40, n).astype(np.int64)   # |v| >= 2^26: the GENERIC run body
    i2 = rng.integers(-100, 100, n).astype(np.int64)
    f1 = rng.normal(0, 1e3, n)
    f2 = rng.uniform(0, 1, n)
    aggs = [(dg.AGG_SUM_I64, i1), (dg.AGG_COUNT, None), (dg.AGG_SUM_I64, i2), (dg.AGG_AVG_F64, f1),
            (dg.AGG_SUM_F64, f2)]
    ag = pac.Aggregator128([k for k, _ in aggs], 32)
    call = lambda: ag(_dev_vals(aggs), [to_dev(keys[0])],  # noqa: E731
                      mask2=to_dev(np.ascontiguousarray(m).view(np.int64)))
    t, kern = _last_kernel(call)
    if n:
        assert kern.startswith("k_agg_tiles128<2,2>")
    _cmp(t.to_host(), orc.agg128(m, keys, aggs))


@pytest.mark.parametrize("cfg,n,G_cap", [("C2", 2_000_003, 8), ("C1", 70_001, 1)])
def test_native128_matches_three_pass(cfg, n, G_cap):
    """same table from the native kernel and from the three 64-world passes (integers bit-exact)"""
    w = dg.WORKLOADS[cfg]
    cols = w.host_columns(0, n)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    ag = pac.Aggregator128([k for k, _ in aggs], G_cap)
    dv, dk, pu = _dev_vals(aggs), [to_dev(k) for k in cols["keys"]], to_dev(cols["pu"])
    t1, kern = _last_kernel(lambda: ag(dv, dk, pu_key=pu, salt=77))
    assert kern.startswith("k_agg_tiles128")
    a = t1.to_host()
    os.environ["PAC_NO_NATIVE128"] = "1"
    try:
        b = ag(dv, dk, pu_key=pu, salt=77).to_host()
    finally:
        del os.environ["PAC_NO_NATIVE128"]
    _cmp(a, b)


def test_native128_capacity_reported():
    rng = np.random.default_rng(3)
    n = 50_000
    keys = rng.integers(0, 9, n).astype(np.int8)
    ag = pac.Aggregator128([pac.COUNT, pac.SUM_I64], 4)
    t = ag([None, to_dev(np.ones(n, dtype=np.int64))], [to_dev(keys)],
           pu_key=to_dev(np.arange(n, dtype=np.int64)), salt=5)
    torch.cuda.synchronize()
    assert int(t.status.item()) == pac._lib.PAC_E_CAPACITY
