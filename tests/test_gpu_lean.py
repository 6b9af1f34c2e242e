"""-m gpu parity of k_agg_lean (csrc/agg_lean.cuh: every group in a CTA-local slot, packed key
<= 4 bytes, COUNT / int64 SUM / f64 SUM-AVG over hashed pu keys -- BASELINE C1, C2, C5) against
the CPU oracle, element by element on the same seeded inputs: both TMEM table modes (private
copies for small tables, slot owners for up to 128 groups), every (int64, f64) column count the
kernel instantiates, the three key specs (none, one int32 column, 1-4 narrow columns), ragged
tails and unaligned columns (thread-staged tiles), skewed groups, straggler queues, the generic
(big int64 / non-finite f64) run bodies and capacity overflow; plus an A/B check against the
general tile kernels (PAC_NO_LEAN)."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import assert_tables_equal, run_gpu, to_dev, workload_aggs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

SALT = 0x243F6A8885A308D3


def _last_kernel(aggs, keys, **kw):
    import paper_2603_15023_b200 as pac
    pac.profile_enable(True)
    try:
        t, _ = run_gpu(aggs, keys, **kw)
        torch.cuda.synchronize()
        name = pac.profile_last_kernel()
        pac.profile_read()
    finally:
        pac.profile_enable(False)
    return t, name


@pytest.mark.parametrize("cfg,n,G_cap", [("C1", 1_000_000, 1), ("C2", 2_000_017, 8), ("C5", 3_000_001, 100),
                                         ("C5", 400_000, 128)])
def test_workloads(orc, cfg, n, G_cap):
    w = dg.WORKLOADS[cfg]
    cols = w.host_columns(0, n)
    aggs = workload_aggs(w, cols)
    t, name = _last_kernel(aggs, cols["keys"], pu=cols["pu"], salt=SALT, G_cap=G_cap)
    assert name.startswith("k_agg_lean"), name
    ref = orc.agg(orc.pac_hash(cols["pu"], SALT), cols["keys"], aggs)
    assert_tables_equal(t.to_host(), ref)


@pytest.mark.parametrize("n", [1, 2, 31, 33, 2047, 2048, 2049, 4095, 4097, 70_001])
@pytest.mark.parametrize("G_cap,ng", [(8, 6), (100, 100)])
def test_ragged(orc, n, G_cap, ng):
    rng = np.random.default_rng(7 * n + G_cap)
    pu = rng.integers(0, 5000, n).astype(np.int64)
    keys = [rng.integers(-50, -50 + ng, n).astype(np.int32)]
    iv = rng.integers(-10**6, 10**6, n).astype(np.int64)
    fv = rng.normal(3, 1, n)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv), (dg.AGG_AVG_F64, fv)]
    t, name = _last_kernel(aggs, keys, pu=pu, salt=11, G_cap=G_cap)
    assert name.startswith("k_agg_lean"), name
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 11), keys, aggs))


# (int64 columns, f64 columns) the kernel instantiates (ni + nf <= 3)
@pytest.mark.parametrize("ni,nf", [(0, 0), (0, 1), (0, 2), (1, 0), (1, 1), (1, 2), (2, 0), (2, 1)])
@pytest.mark.parametrize("G_cap", [4, 100])
def test_column_counts(orc, ni, nf, G_cap):
    rng = np.random.default_rng(100 * ni + 10 * nf + G_cap)
    n = 123_457
    pu = rng.integers(0, 20_000, n).astype(np.int64)
    keys = [rng.integers(0, G_cap, n).astype(np.int32)]
    aggs = [(dg.AGG_COUNT, None)]
    for c in range(ni):
        aggs.append((dg.AGG_SUM_I64, rng.integers(-(10**5), 10**7, n).astype(np.int64)))
    for c in range(nf):
        aggs.append((dg.AGG_AVG_F64 if c == 0 else dg.AGG_SUM_F64, rng.random(n) * (c + 1)))
    t, name = _last_kernel(aggs, keys, pu=pu, salt=5, G_cap=G_cap)
    assert name.startswith("k_agg_lean<%d,%d," % (ni, nf)), name
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 5), keys, aggs))


@pytest.mark.parametrize("dtypes,G_cap", [([np.int8, np.int8], 8), ([np.int16, np.int8, np.int8], 64),
                                          ([np.int8] * 4, 128), ([np.int16, np.int16], 100), ([np.int16], 30)])
def test_narrow_key_columns(orc, dtypes, G_cap):
    rng = np.random.default_rng(len(dtypes) + G_cap)
    n = 200_003
    pu = rng.integers(0, 9000, n).astype(np.int64)
    # a small key domain (<= G_cap distinct packed keys), including negative values
    combos = rng.integers(-3, 3, (G_cap, len(dtypes)))
    pick = rng.integers(0, G_cap, n)
    keys = [combos[pick, c].astype(dt) for c, dt in enumerate(dtypes)]
    iv = rng.integers(1, 10**6, n).astype(np.int64)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv)]
    t, name = _last_kernel(aggs, keys, pu=pu, salt=9, G_cap=G_cap)
    assert name.startswith("k_agg_lean") and name.split("<")[1].split(",")[2] == "2", name
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 9), keys, aggs))


def test_unaligned_columns_thread_staged(orc):
    # column views offset by one element: not 16-byte aligned, so no TMA -- every tile is staged
    # by the threads
    rng = np.random.default_rng(3)
    n = 50_001
    pu = rng.integers(0, 3000, n + 1).astype(np.int64)
    k = rng.integers(0, 90, n + 1).astype(np.int32)
    iv = rng.integers(0, 1000, n + 1).astype(np.int64)
    fv = rng.random(n + 1)
    import paper_2603_15023_b200 as pac
    ag = pac.Aggregator([pac.COUNT, pac.SUM_I64, pac.AVG_F64], 100)
    dk, dpu, di, df = to_dev(k), to_dev(pu), to_dev(iv), to_dev(fv)
    pac.profile_enable(True)
    t = ag([None, di[1:], df[1:]], [dk[1:]], pu_key=dpu[1:], salt=2)
    torch.cuda.synchronize()
    name = pac.profile_last_kernel()
    pac.profile_read()
    pac.profile_enable(False)
    assert name.startswith("k_agg_lean"), name
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv[1:]), (dg.AGG_AVG_F64, fv[1:])]
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu[1:], 2), [k[1:]], aggs))


def test_skewed_groups_owner_mode(orc):
    # Zipf-like: one group holds most rows (many runs for one owner warp), a long tail of small ones
    rng = np.random.default_rng(21)
    n = 600_000
    g = np.minimum(rng.zipf(1.3, n) - 1, 119).astype(np.int32)
    pu = rng.integers(0, 50_000, n).astype(np.int64)
    iv = rng.integers(1, 10**6, n).astype(np.int64)
    fv = rng.random(n)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv), (dg.AGG_AVG_F64, fv)]
    t, name = _last_kernel(aggs, [g], pu=pu, salt=33, G_cap=120)
    assert name.startswith("k_agg_lean"), name
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 33), [g], aggs))


@pytest.mark.parametrize("G_cap", [4, 100])
def test_generic_run_bodies(orc, G_cap):
    # |v| >= 2^26 (int64 subset tables) and +-inf / nan (select-built f64 tables) in some tiles
    rng = np.random.default_rng(G_cap)
    n = 150_000
    pu = rng.integers(0, 3000, n).astype(np.int64)
    keys = [rng.integers(0, G_cap, n).astype(np.int32)]
    iv = rng.integers(-1000, 1000, n).astype(np.int64)
    iv[rng.integers(0, n, 40)] = rng.integers(-(2**40), 2**40, 40)
    fv = rng.random(n)
    fv[rng.integers(0, n, 5)] = np.inf
    fv[rng.integers(0, n, 3)] = -np.inf
    fv[rng.integers(0, n, 2)] = np.nan
    aggs = [(dg.AGG_SUM_I64, iv), (dg.AGG_COUNT, None), (dg.AGG_SUM_F64, fv)]
    t, name = _last_kernel(aggs, keys, pu=pu, salt=3, G_cap=G_cap)
    assert name.startswith("k_agg_lean"), name
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 3), keys, aggs))


@pytest.mark.parametrize("G_cap,ng", [(8, 20), (100, 150), (128, 300)])
def test_capacity_exceeded_reported(G_cap, ng):
    import paper_2603_15023_b200 as pac
    n = 40_000
    keys = [to_dev(np.arange(n, dtype=np.int32) % ng)]
    pu = to_dev(np.arange(n, dtype=np.int64))
    ag = pac.Aggregator([pac.COUNT], G_cap)
    t = ag([None], keys, pu_key=pu, salt=1)
    with pytest.raises(pac.PacError) as e:
        t.check()
    assert e.value.rc == 2


@pytest.mark.parametrize("cfg,n,G_cap", [("C2", 1_000_000, 8), ("C5", 1_000_000, 100)])
def test_lean_and_tile_kernels_agree(orc, monkeypatch, cfg, n, G_cap):
    w = dg.WORKLOADS[cfg]
    cols = w.host_columns(0, n)
    aggs = workload_aggs(w, cols)
    t1, name1 = _last_kernel(aggs, cols["keys"], pu=cols["pu"], salt=SALT, G_cap=G_cap)
    monkeypatch.setenv("PAC_NO_LEAN", "1")
    t2, name2 = _last_kernel(aggs, cols["keys"], pu=cols["pu"], salt=SALT, G_cap=G_cap)
    assert name1.startswith("k_agg_lean") and not name2.startswith("k_agg_lean"), (name1, name2)
    assert_tables_equal(t1.to_host(), t2.to_host())
