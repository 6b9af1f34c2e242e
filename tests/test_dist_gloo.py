"""Multi-process (world_size 2, gloo, CPU) test of the row-sharded merge plumbing
(paper analogue: thread-local partial aggregates + combine).

Each rank builds the partial 64-world table of its contiguous row shard (the oracle stands
in for the per-GPU kernel here), then the product's torch.distributed plumbing --
union dictionary, all_reduce ops per array -- merges them.  The merged table must equal
the unsharded table exactly (integers, MIN/MAX) or to 1e-12 (f64 sums)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen as dg

KINDS = [dg.AGG_COUNT, dg.AGG_SUM_I64, dg.AGG_AVG_F64, dg.AGG_MIN_F64, dg.AGG_MAX_F64]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(n=40_000, seed=3):
    rng = np.random.default_rng(seed)
    pu = rng.integers(0, 3000, n).astype(np.int64)
    g = rng.integers(0, 40, n).astype(np.int32)
    iv = rng.integers(-10**6, 10**6, n).astype(np.int64)
    fv = rng.normal(5, 2, n)
    return pu, g, iv, fv


def _aggs(iv, fv):
    vals = {dg.AGG_COUNT: None, dg.AGG_SUM_I64: iv, dg.AGG_AVG_F64: fv, dg.AGG_MIN_F64: fv,
            dg.AGG_MAX_F64: fv}
    return [(k, vals[k]) for k in KINDS]


MIN_EMPTY = np.int64(0x7FFFFFFFFFFFFFFF)
MAX_EMPTY = np.int64(-0x8000000000000000)


def _enc(v):
    """include/pac.h's order-preserving encoding (R31): NaN -> one value above +inf."""
    b = np.ascontiguousarray(v, dtype=np.float64).view(np.int64).copy()
    nan = np.isnan(v)
    b = np.where(b >= 0, b, b ^ np.int64(0x7FFFFFFFFFFFFFFF))
    return np.where(nan, np.int64(0x7FF8000000000000), b)


def _dec(e):
    b = np.where(e >= 0, e, e ^ np.int64(0x7FFFFFFFFFFFFFFF))
    return b.view(np.float64)


def _pack(G, rows, count, worlds, K):
    """The flat-buffer layout of include/pac.h (pac_merge_pack), written from the header:
    i64_sum = rows | count | SUM_I64 worlds; f64_sum = SUM/AVG worlds; i64_min = f, ~f,
    ~status, MIN encodings, ~MAX encodings (sentinel for worlds outside K)."""
    Kb = ((K[:, None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)).astype(bool)
    i64 = [rows, count.ravel()]
    f64, mn = [], [np.array([12345, ~12345, ~0], dtype=np.int64)]
    for a, k in enumerate(KINDS):
        if k == dg.AGG_SUM_I64:
            i64.append(worlds[a].ravel())
        elif k in (dg.AGG_SUM_F64, dg.AGG_AVG_F64):
            f64.append(worlds[a].ravel())
        elif k == dg.AGG_MIN_F64:
            mn.append(np.where(Kb, _enc(worlds[a]), MIN_EMPTY).ravel())
        elif k == dg.AGG_MAX_F64:
            mn.append(~np.where(Kb, _enc(worlds[a]), MAX_EMPTY).ravel())
    return (torch.from_numpy(np.concatenate(i64).astype(np.int64)), torch.from_numpy(np.concatenate(f64)),
            torch.from_numpy(np.concatenate(mn).astype(np.int64)))


def _unpack(G, i64, f64, mn):
    i64, f64, mn = i64.numpy(), f64.numpy(), mn.numpy()
    rows, count = i64[:G], i64[G:G + 64 * G].reshape(G, 64)
    oi, of, om = G + 64 * G, 0, 3
    worlds = []
    for k in KINDS:
        if k == dg.AGG_COUNT:
            worlds.append(None)
        elif k == dg.AGG_SUM_I64:
            worlds.append(i64[oi:oi + 64 * G].reshape(G, 64)); oi += 64 * G
        elif k in (dg.AGG_SUM_F64, dg.AGG_AVG_F64):
            worlds.append(f64[of:of + 64 * G].reshape(G, 64)); of += 64 * G
        elif k == dg.AGG_MIN_F64:
            e = mn[om:om + 64 * G].reshape(G, 64); om += 64 * G
            worlds.append(np.where(e == MIN_EMPTY, np.inf, _dec(e)))
        else:
            e = ~mn[om:om + 64 * G].reshape(G, 64); om += 64 * G
            worlds.append(np.where(e == MAX_EMPTY, -np.inf, _dec(e)))
    assert mn[0] == ~mn[1]  # every rank packed the same dictionary fingerprint
    return rows, count, worlds


def _worker(rank, world, port, q):
    try:
        import time

        import oracle
        from paper_2603_15023_b200 import dist as pdist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        pu, g, iv, fv = _case()
        n = len(pu)
        lo, hi = rank * n // world, (rank + 1) * n // world
        # rank 1 drops a group entirely so the union dictionary differs from the local one
        sel = np.arange(lo, hi)
        if rank == 1:
            sel = sel[g[sel] != 7]
        masks = oracle.pac_hash(pu[sel], 99)
        part = oracle.agg(masks, [g[sel]], _aggs(iv[sel], fv[sel]))
        local_keys = torch.from_numpy(part["keys"].view(np.int64).copy())
        union, same = pdist.union_keys(local_keys)
        assert not same
        ukeys = union.numpy().view(np.uint64)
        # lay the partial table out on the union dictionary (the device does this with
        # pac_table_remap; here plain numpy on the oracle's arrays)
        G = len(ukeys)
        idx = np.searchsorted(ukeys, part["keys"])
        rows = np.zeros(G, dtype=np.int64)
        count = np.zeros((G, 64), dtype=np.int64)
        K = np.zeros(G, dtype=np.uint64)
        worlds = []
        rows[idx] = part["rows"]
        count[idx] = part["count"]
        K[idx] = part["K"]
        for a, k in enumerate(KINDS):
            if k == dg.AGG_COUNT:
                worlds.append(None)
                continue
            fill = {dg.AGG_MIN_F64: np.inf, dg.AGG_MAX_F64: -np.inf}.get(k, 0)
            w = np.full((G, 64), fill, dtype=np.int64 if k == dg.AGG_SUM_I64 else np.float64)
            w[idx] = part["world"][a]
            worlds.append(w)
        i64, f64, mn = _pack(G, rows, count, worlds, K)
        pdist.merge_flat(i64, f64, mn)
        rows, count, worlds = _unpack(G, i64, f64, mn)
        # the merge's collectives alone, at BASELINE C5's table size (100 groups, COUNT + SUM + AVG)
        b = (torch.zeros(100 + 2 * 6400, dtype=torch.int64), torch.zeros(6400, dtype=torch.float64),
             torch.zeros(3, dtype=torch.int64))
        for _ in range(5):
            pdist.merge_flat(*b)
        t0 = time.perf_counter()
        for _ in range(50):
            pdist.merge_flat(*b)
        us = (time.perf_counter() - t0) / 50 * 1e6
        q.put((rank, ukeys, rows, count, worlds, us))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure to the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()))


def test_row_sharded_merge_equals_unsharded_table(orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for o in out:
        assert not (isinstance(o[1], str) and o[1] == "error"), o
    pu, g, iv, fv = _case()
    n = len(pu)
    keep = np.ones(n, dtype=bool)
    keep[n // 2:] &= g[n // 2:] != 7   # the rows rank 1 left out
    pu, g, iv, fv = pu[keep], g[keep], iv[keep], fv[keep]
    ref = orc.agg(orc.pac_hash(pu, 99), [g], _aggs(iv, fv))
    for rank, ukeys, rows, count, worlds, us in out:
        np.testing.assert_array_equal(ukeys, ref["keys"])
        np.testing.assert_array_equal(rows, ref["rows"])
        np.testing.assert_array_equal(count, ref["count"])
        # K from the merged counts (NCCL has no OR reduction) equals the OR
        K = np.array([sum(1 << j for j in range(64) if c[j] > 0) for c in count], dtype=np.uint64)
        np.testing.assert_array_equal(K, ref["K"])
        for a, k in enumerate(KINDS):
            if k == dg.AGG_COUNT:
                continue
            if k == dg.AGG_AVG_F64:
                np.testing.assert_allclose(worlds[a], ref["world"][a], rtol=1e-12)
            else:
                np.testing.assert_array_equal(worlds[a], ref["world"][a])
        print(f"rank {rank}: merge collectives at C5 table size {us:.0f} us (gloo, CPU)")


def test_reduce_ops_follow_aggregate_kind():
    from paper_2603_15023_b200 import dist as pdist
    assert pdist.reduce_ops_for(KINDS) == ["none", "sum", "sum", "min", "max"]
