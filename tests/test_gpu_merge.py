"""-m gpu tests of the cross-GPU merge kernels (pac_merge_pack / pac_merge_unpack, §8 a5/e) on
one device: two row shards are aggregated separately, packed, reduced exactly as the three
NCCL all_reduce calls would (SUM, SUM, MIN -- done here with torch on the device), unpacked,
and compared with the unsharded table and the oracle.  Also: presence of MIN/MAX-only tables
survives the merge (worlds holding only +inf / -inf), a dictionary mismatch is caught on the
device (PAC_E_MERGE), a rank's CAPACITY status propagates, and pac_finalize releases nothing
from an invalid table (every cell NULL, flags bit 1, posterior unchanged)."""
import numpy as np
import pytest

import datagen as dg
from gpu_helpers import assert_tables_equal, run_gpu, to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_15023_b200 as pac  # noqa: E402


def _reduce(bufs_list):
    """What all_reduce(SUM), all_reduce(SUM), all_reduce(MIN) leave in every rank's buffers."""
    b0 = bufs_list[0]
    for b in bufs_list[1:]:
        b0.i64_sum += b.i64_sum
        b0.f64_sum += b.f64_sum
        torch.minimum(b0.i64_min, b.i64_min, out=b0.i64_min)
    return b0


def _shards(aggs, keys, pu, salt, G_cap, cut):
    tabs = []
    for lo, hi in ((0, cut), (cut, len(pu))):
        sl = {id(v): v[lo:hi] for _, v in aggs if v is not None}  # aggregates sharing a column keep sharing it
        a = [(k, None if v is None else sl[id(v)]) for k, v in aggs]
        t, _ = run_gpu(a, [k[lo:hi] for k in keys], pu=pu[lo:hi], salt=salt, G_cap=G_cap)
        tabs.append(t)
    return tabs


def _merge(tabs):
    bufs = [pac.api.MergeBuffers(t.kinds, t.G_cap, t.rows.device) for t in tabs]
    for t, b in zip(tabs, bufs):
        pac.api.merge_pack(t, b)
    b = _reduce(bufs)
    pac.api.merge_unpack(tabs[0], b)
    return tabs[0]


@pytest.mark.parametrize("cfg", ["C2", "C5"])
def test_two_shard_merge_equals_unsharded(orc, cfg):
    w = dg.WORKLOADS[cfg]
    n = 600_000
    cols = w.host_columns(0, n)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    G_cap = {"C2": 8, "C5": 100}[cfg]
    tabs = _shards(aggs, cols["keys"], cols["pu"], 77, G_cap, 250_001)
    merged = _merge(tabs).to_host()
    full, _ = run_gpu(aggs, cols["keys"], pu=cols["pu"], salt=77, G_cap=G_cap)
    assert_tables_equal(merged, full.to_host())
    assert_tables_equal(merged, orc.agg(orc.pac_hash(cols["pu"], 77), cols["keys"], aggs))


def test_minmax_only_presence_survives_the_merge(orc):
    rng = np.random.default_rng(3)
    n = 200_000
    pu = rng.integers(0, 3000, n).astype(np.int64)
    g = rng.integers(0, 10, n).astype(np.int32)
    v = rng.normal(0, 1, n)
    v[g == 3] = np.inf    # MIN of group 3 is +inf in every present world
    v[g == 4] = -np.inf   # MAX of group 4 is -inf in every present world
    v[rng.choice(n, 50, replace=False)] = np.nan
    aggs = [(dg.AGG_MIN_F64, v), (dg.AGG_MAX_F64, v)]
    tabs = _shards(aggs, [g], pu, 5, 16, 99_999)
    merged = _merge(tabs).to_host()
    ref = orc.agg(orc.pac_hash(pu, 5), [g], aggs)
    assert_tables_equal(merged, ref)
    assert bin(int(merged["K"][3])).count("1") == 64 and bin(int(merged["K"][4])).count("1") == 64


def test_dictionary_mismatch_is_caught_on_device():
    rng = np.random.default_rng(4)
    n = 100_000
    pu = rng.integers(0, 3000, n).astype(np.int64)
    g = rng.integers(0, 10, n).astype(np.int32)
    g[n // 2:][g[n // 2:] == 7] = 8  # shard 2 lacks group 7: a different dictionary
    iv = rng.integers(0, 100, n).astype(np.int64)
    aggs = [(dg.AGG_COUNT, None), (dg.AGG_SUM_I64, iv)]
    tabs = _shards(aggs, [g], pu, 5, 16, n // 2)
    m = _merge(tabs)
    assert int(m.status.item()) == pac._lib.PAC_E_MERGE
    # nothing is released from it
    s = pac.Session(11, 1 / 128)
    P0 = s.query()["P"]
    rel, isn, flags, _ = pac.finalize(s, m, 0)
    G = int(m.num_groups.item())
    assert np.all(isn[:G].cpu().numpy() == 1) and np.all((flags[:G].cpu().numpy() & 2) == 2)
    assert np.all(np.isnan(rel[:G].cpu().numpy()))
    assert np.array_equal(s.query()["P"], P0)


def test_capacity_status_propagates_and_blocks_release():
    n = 50_000
    keys = [to_dev((np.arange(n) % 12).astype(np.int64))]
    pu = to_dev(np.arange(n, dtype=np.int64))
    ag = pac.Aggregator([pac.COUNT], 8)
    t = ag([None], keys, pu_key=pu, salt=1)
    assert int(t.status.item()) == pac._lib.PAC_E_CAPACITY
    s = pac.Session(12, 1 / 128)
    P0 = s.query()["P"]
    rel, isn, flags, _ = pac.finalize(s, t, 0)
    assert np.all(isn[:8].cpu().numpy() == 1) and np.all((flags[:8].cpu().numpy() & 2) == 2)
    assert np.array_equal(s.query()["P"], P0)
    # merged with a valid shard, the CAPACITY status wins
    ok = pac.Aggregator([pac.COUNT], 8)([None], [to_dev((np.arange(n) % 8).astype(np.int64))], pu_key=pu, salt=1)
    bufs = [pac.api.MergeBuffers([pac.COUNT], 8, ok.rows.device) for _ in range(2)]
    pac.api.merge_pack(ok, bufs[0])
    pac.api.merge_pack(t, bufs[1])
    pac.api.merge_unpack(ok, _reduce(bufs))
    assert int(ok.status.item()) in (pac._lib.PAC_E_CAPACITY, pac._lib.PAC_E_MERGE)
