"""-m gpu parity: libpac (through the C-ABI binding) vs the CPU oracle, element by element,
on the same seeded input bytes.  Bit-exact for masks, counts, integer sums, MIN/MAX, K,
rows, NULL flags; <= 1e-9 relative for f64 sums / AVG; releases per R16."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import (REL_F64, assert_delta_close, assert_releases_close, assert_tables_equal,
                         run_gpu, to_dev, workload_aggs)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_15023_b200 as pac  # noqa: E402

SALT = 0x243F6A8885A308D3


# ------------------------------------------------------------------ mask (a2)
def test_mask_bit_exact(orc):
    rng = np.random.default_rng(0)
    keys = np.concatenate([
        np.arange(1_000_000, dtype=np.int64),
        rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, 1_000_003, dtype=np.int64),
        np.array([0, -1, 1, np.iinfo(np.int64).min, np.iinfo(np.int64).max], dtype=np.int64)])
    for salt in (SALT, 0, 0xFFFFFFFFFFFFFFFF):
        got = pac.as_u64(pac.mask(to_dev(keys), salt))
        ref = orc.pac_hash(keys, salt)
        np.testing.assert_array_equal(got, ref)
    pc = np.unpackbits(got.view(np.uint8).reshape(-1, 8), axis=1).sum(1)
    assert np.all(pc == 32)


def test_mask_empty():
    out = pac.mask(torch.zeros(0, dtype=torch.int64, device="cuda"), 1)
    assert out.numel() == 0


# ------------------------------------------------------------------ aggregation (a3-a5)
@pytest.mark.parametrize("cfg,n", [("C1", 100_003), ("C2", 200_017), ("C3", 150_001), ("C4", 300_007),
                                   ("C5", 250_009)])
def test_workload_tables_match_oracle(orc, cfg, n):
    w = dg.WORKLOADS[cfg]
    cols = w.host_columns(0, n)
    aggs = workload_aggs(w, cols)
    G_cap = 1 << 17
    t, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=SALT, G_cap=G_cap)
    got = t.to_host()
    ref = orc.agg(orc.pac_hash(cols["pu"], SALT), cols["keys"], aggs)
    assert_tables_equal(got, ref)


def test_brute_force_o1_equals_gpu_on_tiny_input(orc):
    rng = np.random.default_rng(1)
    n = 3000
    pu = rng.integers(0, 40, n).astype(np.int64)
    keys = [rng.integers(-2, 2, n).astype(np.int16), rng.integers(0, 3, n).astype(np.int8)]
    iv = rng.integers(-10**12, 10**12, n).astype(np.int64)
    fv = rng.normal(0, 1e3, n)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv), (dg.AGG_SUM_F64, fv), (dg.AGG_AVG_F64, fv),
            (dg.AGG_MIN_F64, fv), (dg.AGG_MAX_F64, fv)]
    t, _ = run_gpu(aggs, keys, pu=pu, salt=7, G_cap=64)
    ref = orc.agg(orc.pac_hash(pu, 7), keys, aggs, method="o1")
    assert_tables_equal(t.to_host(), ref)


@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 2047, 2048, 2049, 4097])
def test_ragged_and_tiny_sizes(orc, n):
    rng = np.random.default_rng(n)
    pu = rng.integers(0, 1000, n).astype(np.int64)
    keys = [rng.integers(0, 5, n).astype(np.int32)]
    iv = rng.integers(1, 10**6, n).astype(np.int64)
    fv = rng.random(n)
    aggs = [(dg.AGG_SUM_I64, iv), (dg.AGG_AVG_F64, fv), (dg.AGG_COUNT, None)]
    t, _ = run_gpu(aggs, keys, pu=pu, salt=3, G_cap=16)
    ref = orc.agg(orc.pac_hash(pu, 3), keys, aggs)
    assert_tables_equal(t.to_host(), ref)


def test_ungrouped_zero_rows_has_one_empty_group(orc):
    e = np.zeros(0, dtype=np.int64)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, e)]
    t, _ = run_gpu(aggs, [], pu=e, salt=1, G_cap=1)
    got = t.to_host()
    assert got["G"] == 1 and got["rows"][0] == 0 and got["K"][0] == 0
    assert_tables_equal(got, orc.agg(np.zeros(0, dtype=np.uint64), [], aggs))


def test_explicit_masks_zero_and_all_ones(orc):
    rng = np.random.default_rng(2)
    n = 20_000
    masks = orc.pac_hash(rng.integers(0, 500, n).astype(np.int64), 11)
    masks[::11] = np.uint64(0xFFFFFFFFFFFFFFFF)      # in every world
    masks[5::13] &= np.uint64(0x00FF00FF00FF00FF)    # pac_select-style reduced masks
    masks[::7] = 0                                   # R21: dropped rows
    keys = [rng.integers(0, 9, n).astype(np.int8)]
    keys[0][::7] = 100                               # a group whose rows all have mask 0
    fv = rng.normal(10, 3, n)
    iv = rng.integers(-5, 5, n).astype(np.int64)
    for aggs in ([(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv), (dg.AGG_MAX_F64, fv)],
                 [(dg.AGG_MIN_F64, fv), (dg.AGG_MAX_F64, fv)]):
        t, _ = run_gpu(aggs, keys, masks=masks, G_cap=32)
        ref = orc.agg(masks, keys, aggs)
        assert 100 not in [int(k) ^ 0x80 for k in ref["keys"]]
        assert_tables_equal(t.to_host(), ref)


def test_many_groups_use_global_tier_and_radix_sort(orc):
    # > local smem slots and > single-CTA sort size: HBM dictionary + radix path
    rng = np.random.default_rng(4)
    n = 400_000
    pu = rng.integers(0, 50_000, n).astype(np.int64)
    keys = [rng.integers(-30_000, 30_000, n).astype(np.int32)]
    iv = rng.integers(0, 1000, n).astype(np.int64)
    aggs = [(dg.AGG_SUM_I64, iv), (dg.AGG_COUNT, None)]
    t, _ = run_gpu(aggs, keys, pu=pu, salt=5, G_cap=70_000)
    got = t.to_host()
    ref = orc.agg(orc.pac_hash(pu, 5), keys, aggs)
    assert got["G"] > 4096
    assert_tables_equal(got, ref)


def test_capacity_exceeded_is_reported():
    n = 10_000
    keys = [to_dev(np.arange(n, dtype=np.int64) % 100)]
    pu = to_dev(np.arange(n, dtype=np.int64))
    ag = pac.Aggregator([pac.COUNT], 50)
    t = ag([None], keys, pu_key=pu, salt=1)
    with pytest.raises(pac.PacError) as e:
        t.check()
    assert e.value.rc == 2


def test_composite_keys_all_widths(orc):
    rng = np.random.default_rng(6)
    n = 60_000
    pu = rng.integers(0, 5000, n).astype(np.int64)
    for keys in ([rng.integers(-3, 3, n).astype(np.int8), rng.integers(-2, 2, n).astype(np.int16),
                  rng.integers(-2, 2, n).astype(np.int32)],
                 [rng.integers(-(2**40), 2**40, n).astype(np.int64) % 7 - 3]):
        aggs = [(dg.AGG_COUNT, None)]
        t, _ = run_gpu(aggs, keys, pu=pu, salt=9, G_cap=512)
        assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 9), keys, aggs))


# ------------------------------------------------------------------ finalize (a6, a7)
def _finalize_case(orc, cfg, n, seed, rounds=1):
    w = dg.WORKLOADS[cfg]
    cols = w.host_columns(0, n)
    aggs = workload_aggs(w, cols)
    jstar, salt, P = orc.session(seed)
    s = pac.Session(seed, w.budget)
    assert (s.salt, s.jstar) == (salt, jstar)
    t, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=salt, G_cap=1 << 15)
    ref = orc.agg(orc.pac_hash(cols["pu"], salt), cols["keys"], aggs)
    fin = pac.Finalizer(t.kinds, t.G_cap)
    G = ref["G"]
    assert t.check() == G
    A = len(aggs)
    ymax = np.array([[np.abs(orc.y_vector(ref, a, g)).max() for a in range(A)] for g in range(G)])
    for rnd in range(rounds):
        rel, isn, flags, delta = fin(s, t, rnd)
        r_o, n_o, f_o, d_o, P = orc.finalize(seed, w.budget, jstar, P, ref, rnd)
        rel = rel[:G].cpu().numpy()
        isn = isn[:G].cpu().numpy()
        assert_releases_close(rel, r_o, d_o, isn, n_o)
        np.testing.assert_array_equal(flags[:G].cpu().numpy(), f_o)
        dg_ = delta[:G].cpu().numpy()
        ok = n_o == 0
        assert_delta_close(dg_[ok], d_o[ok], ymax[ok], w.budget)
        Pg = s.query()["P"]
        np.testing.assert_allclose(Pg, P, rtol=0, atol=1e-9)
    return s


@pytest.mark.parametrize("cfg,n,seed", [("C1", 100_000, 1), ("C2", 120_000, 2), ("C4", 100_000, 3),
                                        ("C3", 60_000, 4)])
def test_finalize_matches_oracle(orc, cfg, n, seed):
    _finalize_case(orc, cfg, n, seed)


def test_finalize_twenty_rounds_chain(orc):
    # R17: C5-shaped table, 20 rounds of 300 chained releases
    s = _finalize_case(orc, "C5", 200_000, 5, rounds=20)
    assert s.query()["releases"] > 0


def test_posterior_update_matches_oracle(orc):
    rng = np.random.default_rng(8)
    s = pac.Session(99)
    P = rng.random(64)
    P[[3, 17]] = 0.0
    P /= P.sum()
    s.set_posterior(P)
    for _ in range(10):
        y = rng.normal(0, 10, 64)
        yt, d = float(rng.normal(0, 10)), float(rng.uniform(1, 100))
        pac.posterior_update(s, to_dev(y), yt, d)
        P = orc.posterior_update(P, y, yt, d)
        np.testing.assert_allclose(s.query()["P"], P, rtol=0, atol=1e-12)


def test_null_and_zero_variance_edge_cells(orc):
    # one PU per group: y in {0, 2S}; single-row groups; constant MAX column
    n = 64
    pu = np.repeat(np.arange(8, dtype=np.int64), 8)
    keys = [np.arange(n, dtype=np.int32) // 8]
    iv = np.full(n, 5, dtype=np.int64)
    fv = np.full(n, 2.5)
    aggs = [(dg.AGG_SUM_I64, iv), (dg.AGG_MAX_F64, fv), (dg.AGG_COUNT, None)]
    seed = 77
    jstar, salt, P = orc.session(seed)
    s = pac.Session(seed)
    t, _ = run_gpu(aggs, keys, pu=pu, salt=salt, G_cap=16)
    ref = orc.agg(orc.pac_hash(pu, salt), keys, aggs)
    rel, isn, flags, delta = pac.finalize(s, t, 0)
    r_o, n_o, f_o, d_o, P = orc.finalize(seed, 1 / 128, jstar, P, ref, 0)
    G = ref["G"]
    assert_releases_close(rel[:G].cpu().numpy(), r_o, d_o, isn[:G].cpu().numpy(), n_o)
    np.testing.assert_allclose(s.query()["P"], P, atol=1e-12)


# ------------------------------------------------------------------ merge kernels (a5, e)
def test_shard_remap_merge_rederive_matches_unsharded(orc):
    """Two row shards aggregated separately, laid out on the union dictionary with
    pac_table_remap, summed / min-maxed (what the NCCL allreduce does across GPUs), then K
    re-derived with pac_table_rederive_presence: equals the unsharded oracle table."""
    rng = np.random.default_rng(12)
    n = 120_000
    pu = rng.integers(0, 9000, n).astype(np.int64)
    g = rng.integers(0, 300, n).astype(np.int32)
    g[n // 2:][g[n // 2:] == 5] = 6          # shard 1 lacks group 5
    iv = rng.integers(-10**9, 10**9, n).astype(np.int64)
    fv = rng.normal(0, 10, n)
    for kinds in ([dg.AGG_COUNT, dg.AGG_SUM_I64, dg.AGG_AVG_F64], [dg.AGG_MIN_F64, dg.AGG_MAX_F64]):
        vals = {dg.AGG_COUNT: None, dg.AGG_SUM_I64: iv, dg.AGG_AVG_F64: fv, dg.AGG_MIN_F64: fv,
                dg.AGG_MAX_F64: fv}
        parts = []
        for lo, hi in ((0, n // 2), (n // 2, n)):
            shard = {id(iv): iv[lo:hi].copy(), id(fv): fv[lo:hi].copy()}  # one copy per column
            aggs = [(k, None if vals[k] is None else shard[id(vals[k])]) for k in kinds]
            t, _ = run_gpu(aggs, [g[lo:hi].copy()], pu=pu[lo:hi].copy(), salt=77, G_cap=512)
            t.check()
            parts.append((t, aggs))
        keys = np.union1d(pac.as_u64(parts[0][0].group_key[:parts[0][0].check()]),
                          pac.as_u64(parts[1][0].group_key[:parts[1][0].check()]))
        ukeys = to_dev(keys.view(np.int64))
        mapped = [pac.remap(t, ukeys, [(k, to_dev(v) if v is not None else None) for k, v in aggs])
                  for t, aggs in parts]
        a, b = mapped
        a.rows += b.rows
        if a.count is not None:
            a.count += b.count
        for i, k in enumerate(kinds):
            if k in (dg.AGG_SUM_I64, dg.AGG_AVG_F64):
                a.world[i] += b.world[i]
            elif k == dg.AGG_MIN_F64:
                torch.minimum(a.world[i], b.world[i], out=a.world[i])
            elif k == dg.AGG_MAX_F64:
                torch.maximum(a.world[i], b.world[i], out=a.world[i])
        a.presence.zero_()
        pac.rederive_presence(a, [(k, None) for k in kinds])
        full_aggs = [(k, vals[k]) for k in kinds]
        ref = orc.agg(orc.pac_hash(pu, 77), [g], full_aggs)
        assert_tables_equal(a.to_host(), ref)
