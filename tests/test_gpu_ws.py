"""-m gpu parity of the warp-specialized kernel k_agg_ws (agg_ws.cuh: TMA chunk ring, hasher
warps appending finished rows to per-slot 32-row run buffers, consumer warps aggregating full
runs into Tensor Memory) against the CPU oracle -- the path pac_agg_grouped takes for
COUNT/SUM/AVG tables whose groups all fit the CTA-local slots (BASELINE C1, C2, C5).  Covers
every (int64 SUM, f64 SUM/AVG) column count, 1 / few / 100 / 128 groups, ragged sizes (partial
runs, partial chunks, unaligned columns read from HBM), explicit masks with zeros, runs holding
large int64 or non-finite values (the generic run_body), and an A/B against the tile kernels
(without PAC_WS)."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import assert_tables_equal, run_gpu, to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_15023_b200 as pac  # noqa: E402


@pytest.fixture(autouse=True)
def _ws_on(monkeypatch):
    monkeypatch.setenv("PAC_WS", "1")  # the kernel is opt-in


@pytest.mark.parametrize("ni,nf", [(0, 0), (1, 0), (0, 1), (1, 1), (2, 1), (1, 2), (2, 2)])
@pytest.mark.parametrize("groups,G_cap", [(1, 1), (6, 8), (100, 100), (128, 128)])
def test_column_counts_and_group_counts(orc, monkeypatch, capfd, ni, nf, groups, G_cap):
    monkeypatch.setenv("PAC_DEBUG", "1")
    rng = np.random.default_rng(ni * 10 + nf + groups)
    n = 300_017
    pu = rng.integers(0, 20_000, n).astype(np.int64)
    keys = [rng.integers(0, groups, n).astype(np.int32)] if groups > 1 else []
    aggs = [(dg.AGG_COUNT, None)]
    for c in range(ni):
        aggs.append((dg.AGG_SUM_I64, rng.integers(-10**6, 10**6, n).astype(np.int64)))
    for c in range(nf):
        aggs.append((dg.AGG_AVG_F64 if c == 0 else dg.AGG_SUM_F64, rng.normal(3, 2, n)))
    t, _ = run_gpu(aggs, keys, pu=pu, salt=13, G_cap=G_cap)
    got = t.to_host()
    err = capfd.readouterr().err
    if G_cap <= 100 and ni + nf <= 2:  # fits the TMEM columns and shared memory of k_agg_ws
        assert "k_agg_ws" in err, err
    assert_tables_equal(got, orc.agg(orc.pac_hash(pu, 13), keys, aggs))


@pytest.mark.parametrize("cfg", ["C1", "C2", "C5"])
@pytest.mark.parametrize("n", [1, 31, 63, 64, 65, 4097, 1_000_003])
def test_baseline_shapes_ragged(orc, cfg, n):
    w = dg.WORKLOADS[cfg]
    cols = w.host_columns(12345, n)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    G_cap = {"C1": 1, "C2": 8, "C5": 100}[cfg]
    t, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=21, G_cap=G_cap)
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(cols["pu"], 21), cols["keys"], aggs))


def test_unaligned_columns_and_explicit_masks(orc):
    rng = np.random.default_rng(7)
    n = 100_001
    masks = orc.pac_hash(rng.integers(0, 500, n + 1).astype(np.int64), 3)
    masks[::7] = 0
    masks[::11] &= np.uint64(0x00FF00FF00FF00FF)
    g = rng.integers(0, 40, n + 1).astype(np.int16)
    iv = rng.integers(0, 1000, n + 1).astype(np.int64)
    # offset-by-one views: no 16-byte alignment, so the hashers read HBM directly (no TMA)
    dm = to_dev(masks.view(np.int64))[1:]
    dg_ = to_dev(g)[1:]
    di = to_dev(iv)[1:]
    ag = pac.Aggregator([pac.COUNT, pac.SUM_I64], 64)
    t = ag([None, di], [dg_], mask=dm)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv[1:])]
    assert_tables_equal(t.to_host(), orc.agg(masks[1:], [g[1:]], aggs))


def test_big_and_nonfinite_runs(orc):
    rng = np.random.default_rng(8)
    n = 200_000
    pu = rng.integers(0, 3000, n).astype(np.int64)
    g = rng.integers(0, 20, n).astype(np.int32)
    iv = rng.integers(-1000, 1000, n).astype(np.int64)
    iv[rng.choice(n, 60, replace=False)] = rng.integers(-(2**45), 2**45, 60)
    fv = rng.random(n)
    fv[rng.choice(n, 9, replace=False)] = np.inf
    fv[rng.choice(n, 4, replace=False)] = np.nan
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv), (dg.AGG_AVG_F64, fv)]
    t, _ = run_gpu(aggs, [g], pu=pu, salt=4, G_cap=32)
    assert_tables_equal(t.to_host(), orc.agg(orc.pac_hash(pu, 4), [g], aggs))


def test_ws_and_tile_kernels_agree(orc, monkeypatch):
    w = dg.WORKLOADS["C5"]
    cols = w.host_columns(0, 2_000_000)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    t1, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=5, G_cap=100)
    a = t1.to_host()
    monkeypatch.delenv("PAC_WS")
    t2, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=5, G_cap=100)
    assert_tables_equal(a, t2.to_host())
