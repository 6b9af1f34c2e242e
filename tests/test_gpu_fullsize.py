"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (same
workload, same Aggregator capacity, hence the same kernel instance and grid): C2 (6e7 rows, the
bench line), C3 (1e8 rows, 1e6 Zipf groups: the deferred HBM tier at scale) and C4 (2e8 rows,
MIN/MAX with pruning).

The oracle cannot run the whole O2 aggregation in test time, so the comparison is on samples and
on properties that hold at any size, all computed from the oracle's pac_hash of every row and
plain definitions (np.unique / bincount / index_add of the grouped sums):
  - the group keys (sorted, R20 packing) and each group's row count, exactly;
  - for sampled worlds j: COUNT, int64 SUM, MIN and MAX per group exactly, the f64 sum within
    1e-9, K bit j;
  - for every group: sum over worlds of COUNT = 32 x rows (every PU is in 32 worlds)."""
import numpy as np
import pytest
import torch

import datagen as dg
from gpu_helpers import to_dev

pytestmark = pytest.mark.gpu

import paper_2603_15023_b200 as pac  # noqa: E402

WORLDS = [0, 17, 42, 63]
BENCH_G_CAP = {"C2": 8, "C3": 1 << 21, "C4": 1024}  # bench.py's capacity hints


def _combined_key(keys):
    """R20 packing as an integer: first column most significant, each column sign-flipped."""
    out = np.zeros(len(keys[0]), dtype=np.int64)
    for k in keys:
        bits = 8 * k.dtype.itemsize
        out = (out << bits) | (k.astype(np.int64) + (1 << (bits - 1)))
    return out


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4"])
def test_full_size_sampled_parity(orc, cfg):
    w = dg.WORKLOADS[cfg]
    cols = w.host_columns(0, w.n_rows)
    kinds = [k for k, _ in w.aggs]
    vals = [None if i < 0 else cols["values"][i] for _, i in w.aggs]
    ag = pac.Aggregator(kinds, BENCH_G_CAP[cfg])
    seed = 0x5EED
    s = pac.Session(seed, w.budget)
    dev = {}  # one device copy per column (MIN and MAX of C4 read the same column)
    dvals = [None if v is None else dev.setdefault(id(v), to_dev(v)) for v in vals]
    t = ag(dvals, [to_dev(k) for k in cols["keys"]], pu_key=to_dev(cols["pu"]), salt=s.salt)
    G = t.check()
    got = t.to_host()

    uniq, inv = np.unique(_combined_key(cols["keys"]), return_inverse=True)
    assert G == len(uniq)
    np.testing.assert_array_equal(got["keys"].view(np.int64), uniq)
    rows = np.bincount(inv, minlength=G)
    np.testing.assert_array_equal(got["rows"], rows)
    if got["count"] is not None:
        np.testing.assert_array_equal(got["count"].sum(axis=1), 32 * rows)

    masks = orc.pac_hash(cols["pu"], s.salt)
    inv_t = torch.from_numpy(inv)
    for j in WORLDS:
        sel = ((masks >> np.uint64(j)) & np.uint64(1)).astype(bool)
        cnt = np.bincount(inv[sel], minlength=G)
        if got["count"] is not None:
            np.testing.assert_array_equal(got["count"][:, j], cnt)
        np.testing.assert_array_equal((got["K"] >> np.uint64(j)) & np.uint64(1), (cnt > 0).astype(np.uint64))
        sel_t = torch.from_numpy(sel)
        for a, (k, v) in enumerate(zip(kinds, vals)):
            if k == dg.AGG_SUM_I64:
                ref = torch.zeros(G, dtype=torch.int64).index_add_(0, inv_t[sel_t], torch.from_numpy(v)[sel_t])
                np.testing.assert_array_equal(got["world"][a][:, j], ref.numpy())
            elif k in (dg.AGG_SUM_F64, dg.AGG_AVG_F64):
                ref = torch.zeros(G, dtype=torch.float64).index_add_(0, inv_t[sel_t], torch.from_numpy(v)[sel_t])
                np.testing.assert_allclose(got["world"][a][:, j], ref.numpy(), rtol=1e-9, atol=0)
            elif k in (dg.AGG_MIN_F64, dg.AGG_MAX_F64):  # exact; +inf / -inf for a world with no row
                red = "amin" if k == dg.AGG_MIN_F64 else "amax"
                empty = np.inf if k == dg.AGG_MIN_F64 else -np.inf
                ref = torch.full((G,), empty, dtype=torch.float64).scatter_reduce_(
                    0, inv_t[sel_t], torch.from_numpy(v)[sel_t], reduce=red, include_self=True)
                np.testing.assert_array_equal(got["world"][a][:, j], ref.numpy())
