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


def _threads():
    import os
    return max(1, os.cpu_count() or 1)


def test_c2_full_table_all_worlds_and_releases(orc):
    """C2 at 6e7 rows (bench launch configuration): the complete 64-world table against O2 (row
    ranges on every host core, partial tables combined in thread order -- f64 sums within R16),
    then one finalize round: releases, NULL flags, diversity flags and the posterior."""
    from gpu_helpers import assert_delta_close, assert_releases_close, assert_tables_equal
    w = dg.WORKLOADS["C2"]
    cols = w.host_columns(0, w.n_rows)
    aggs = [(k, None if i < 0 else cols["values"][i]) for k, i in w.aggs]
    seed = 0x5EED
    s = pac.Session(seed, w.budget)
    ag = pac.Aggregator([k for k, _ in aggs], BENCH_G_CAP["C2"])
    t = ag([None if v is None else to_dev(v) for _, v in aggs], [to_dev(k) for k in cols["keys"]],
           pu_key=to_dev(cols["pu"]), salt=s.salt)
    got = t.to_host()
    n = _threads()
    ref = orc.agg_mt(orc.pac_hash_mt(cols["pu"], s.salt, n), cols["keys"], aggs, n)
    assert_tables_equal(got, ref)
    jstar, salt, P = orc.session(seed)
    rel, isn, flags, delta = pac.finalize(s, t, 0)
    r_o, n_o, f_o, d_o, P = orc.finalize(seed, w.budget, jstar, P, ref, 0)
    G = ref["G"]
    assert_releases_close(rel[:G].cpu().numpy(), r_o, d_o, isn[:G].cpu().numpy(), n_o)
    np.testing.assert_array_equal(flags[:G].cpu().numpy(), f_o)
    ok = n_o == 0
    ymax = np.abs(r_o[ok]).max() if ok.any() else 1.0
    assert_delta_close(delta[:G].cpu().numpy()[ok], d_o[ok], ymax, w.budget)
    np.testing.assert_allclose(s.query()["P"], P, rtol=0, atol=1e-9)


def test_c5_full_size_sampled_groups_and_twenty_rounds(orc):
    """C5 at 1.2e9 rows in bench.py's launch configuration (G_cap = 100; device-generated columns,
    as bench.py times them).  Every group: rows and sum_j COUNT_j = 32 rows.  Two sampled groups:
    the rows of those groups are selected on the device, copied to the host, and the oracle
    (pac_hash + O2 on every host core) recomputes their complete 64-world tables.  Then all 20
    finalize rounds of a session over the sampled groups' table (GPU kernels on the GPU table,
    orc_finalize on the oracle's)."""
    from gpu_helpers import assert_releases_close, assert_tables_equal
    w = dg.WORKLOADS["C5"]
    cols = dg.device_columns(w, 0, w.n_rows)
    kinds = [k for k, _ in w.aggs]
    vals = [None if i < 0 else cols["values"][i] for _, i in w.aggs]
    seed = 0x5EED
    s = pac.Session(seed, w.budget)
    ag = pac.Aggregator(kinds, 100)
    t = ag(vals, cols["keys"], pu_key=cols["pu"], salt=s.salt)
    got = t.to_host()
    g = cols["keys"][0]
    rows = torch.bincount(g.long(), minlength=100).cpu().numpy()
    assert got["G"] == 100
    np.testing.assert_array_equal(got["rows"], rows)
    np.testing.assert_array_equal(got["count"].sum(axis=1), 32 * rows)
    pick = [7, 64]
    sel = (g == pick[0]) | (g == pick[1])
    sub_pu = cols["pu"][sel].cpu().numpy()
    sub_g = g[sel].cpu().numpy()
    sub_v = {i: v[sel].cpu().numpy() for i, v in enumerate(cols["values"])}
    del cols, vals, sel
    aggs = [(k, None if i < 0 else sub_v[i]) for k, i in w.aggs]
    n = _threads()
    ref = orc.agg_mt(orc.pac_hash_mt(sub_pu, s.salt, n), [sub_g], aggs, n)
    assert ref["G"] == 2
    gi = [int(np.searchsorted(got["keys"], k)) for k in ref["keys"]]
    sub = {"G": 2, "keys": got["keys"][gi], "rows": got["rows"][gi], "K": got["K"][gi], "count": got["count"][gi],
           "world": [None if x is None else x[gi] for x in got["world"]], "kinds": got["kinds"]}
    assert_tables_equal(sub, ref)
    # the sampled groups as a table of their own on the device: 20 finalize rounds
    t2 = pac.PacTable.allocate(kinds, 2, t.rows.device)
    idx = torch.tensor(gi, device=t.rows.device)
    t2.num_groups.fill_(2)
    t2.status.zero_()
    t2.group_key.copy_(t.group_key[idx])
    t2.rows.copy_(t.rows[idx])
    t2.presence.copy_(t.presence[idx])
    t2.count.copy_(t.count[idx])
    for a, x in enumerate(t.world):
        if x is not None:
            t2.world[a].copy_(x[idx])
    s2 = pac.Session(seed + 1, w.budget)
    jstar, _, P = orc.session(seed + 1)
    fin = pac.Finalizer(kinds, 2)
    for r in range(w.rounds):
        rel, isn, _, _ = fin(s2, t2, r)
        r_o, n_o, _, d_o, P = orc.finalize(seed + 1, w.budget, jstar, P, ref, r)
        assert_releases_close(rel.cpu().numpy(), r_o, d_o, isn.cpu().numpy(), n_o)
    np.testing.assert_allclose(s2.query()["P"], P, rtol=0, atol=1e-9)
