"""Host-side checks of the synthetic input generators (datagen/)."""
import numpy as np

import datagen as dg


def test_counter_based_rows_do_not_depend_on_sharding():
    spec = dg.WORKLOADS["C2"].values[0]
    a = dg.gen_column(spec, 7, 0, 1000)
    b = np.concatenate([dg.gen_column(spec, 7, 0, 400), dg.gen_column(spec, 7, 400, 600)])
    assert np.array_equal(a, b)


def test_ranges_and_distinctness():
    w = dg.WORKLOADS["C2"]
    cols = w.host_columns(0, 200_000)
    g1, g2 = cols["keys"]
    assert g1.dtype == np.int8 and set(np.unique(g1)) == {0, 1, 2}
    assert set(np.unique(g2)) == {0, 1}
    cents, disc = cols["values"]
    assert cents.min() >= 100 and cents.max() <= 10_000_000
    assert disc.min() >= 0.0 and disc.max() < 0.1
    # pu keys: at most 1.5M distinct scrambled ids
    assert len(np.unique(cols["pu"])) <= 1_500_000


def test_scrambles_are_bijective():
    r = np.arange(1 << 16, dtype=np.uint64)
    assert len(np.unique(dg.scramble32(r))) == r.size
    assert len(np.unique(dg.scramble64(r))) == r.size


def test_mulhi64_matches_python_ints():
    rng = np.random.default_rng(0)
    a = rng.integers(0, 2**63, 1000, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    for b in (3, 1_500_000, 2**40 + 17, 2**63 - 1):
        ref = np.array([(int(x) * b) >> 64 for x in a], dtype=np.uint64)
        assert np.array_equal(dg.mulhi64(a, b), ref)


def test_zipf_rank_frequencies():
    spec = dg.ColSpec("g", dg.KIND_ZIPF_KEY32, col=1, n_distinct=1000, zipf_s=1.1)
    keys = dg.gen_column(spec, 3, 0, 400_000)
    _, counts = np.unique(keys, return_counts=True)
    counts = np.sort(counts)[::-1]
    H = np.sum(np.arange(1, 1001) ** -1.1)
    assert abs(counts[0] / 400_000 - 1.0 / H) < 0.01
    assert abs(counts[1] / counts[0] - 2 ** -1.1) < 0.03


def test_normal_moments():
    spec = dg.WORKLOADS["C4"].values[0]
    v = dg.gen_column(spec, 4, 0, 200_000)
    assert abs(v.mean() - 1000) < 3 and abs(v.std() - 250) < 3
