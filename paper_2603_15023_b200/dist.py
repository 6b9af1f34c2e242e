"""Row-sharded multi-GPU merge (the paper's analogue is DuckDB's thread-local
partial aggregates + state.combine).

Each rank aggregates its contiguous row shard with the same salt, then the partial 64-world
tables are merged over NCCL (NVLink / NVSwitch):
  1. common layout: every rank's table must sit on one group dictionary.  Dense domains
     (every rank holds every group, e.g. BASELINE C5's 100 groups) already do -- pass
     `same_keys=True` and nothing is exchanged or synchronised for it; the dictionary
     fingerprint that travels with the data catches a wrong claim on the device
     (PAC_E_MERGE in the table status).  Otherwise the ranks allgather their keys, take the
     sorted union and libpac remaps each table onto it (pac_table_remap) -- host syncs, the
     general path;
  2. libpac packs the table into three flat buffers (pac_merge_pack);
  3. three all_reduce calls, issued back to back: SUM on the int64 buffer {rows, counts,
     SUM_I64 worlds}, SUM on the f64 buffer {SUM_F64 / AVG_F64 worlds}, MIN on the int64
     buffer {fingerprint, status, order-preserving MIN encodings, bit-inverted MAX encodings};
  4. libpac unpacks into the table (pac_merge_unpack): K from the merged counts, or for
     MIN/MAX-only tables from the merged extremes (NCCL has no OR; the encoding carries it).
Finalize then runs identically on every rank (same table, same session seed).

The communication helpers work on any torch.distributed backend (NCCL on the GPU box, gloo in
the CPU tests); they only move tensors -- no method arithmetic here.
"""
from __future__ import annotations

from typing import Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from ._lib import AVG_F64, COUNT, MAX_F64, MIN_F64, SUM_F64, SUM_I64


def reduce_ops_for(kinds: Sequence[int]):
    """The reduction each aggregate's world array takes in the merge (documentation / tests)."""
    ops = []
    for k in kinds:
        if k == COUNT:
            ops.append("none")
        elif k in (SUM_I64, SUM_F64, AVG_F64):
            ops.append("sum")
        elif k == MIN_F64:
            ops.append("min")
        elif k == MAX_F64:
            ops.append("max")
        else:
            raise ValueError(k)
    return ops


def union_keys(local_keys: torch.Tensor, group=None) -> Tuple[torch.Tensor, bool]:
    """Sorted union (as unsigned 64-bit order) of every rank's group keys (int64 bit
    patterns).  Returns (union, same) where `same` is True when every rank already holds
    exactly the union (no remap needed).  Synchronises with the host (sizes)."""
    ws = dist.get_world_size(group)
    n = torch.tensor([local_keys.numel()], dtype=torch.int64, device=local_keys.device)
    sizes = [torch.zeros_like(n) for _ in range(ws)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes) if sizes else 0
    pad = torch.zeros(mx, dtype=torch.int64, device=local_keys.device)
    pad[:local_keys.numel()] = local_keys
    bufs = [torch.zeros_like(pad) for _ in range(ws)]
    dist.all_gather(bufs, pad, group=group)
    allk = torch.cat([b[:s] for b, s in zip(bufs, sizes)])
    # unsigned order: flip the sign bit, sort as signed, flip back
    flip = torch.tensor(-(2 ** 63), dtype=torch.int64, device=allk.device)
    u = torch.unique(allk ^ flip, sorted=True) ^ flip
    same = all(s == u.numel() for s in sizes) and bool(
        torch.equal(local_keys, u)) if local_keys.numel() == u.numel() else False
    # every rank must agree on `same`
    f = torch.tensor([1 if same else 0], dtype=torch.int64, device=local_keys.device)
    dist.all_reduce(f, op=dist.ReduceOp.MIN, group=group)
    return u, bool(f.item())


def merge_flat(i64_sum: torch.Tensor, f64_sum: torch.Tensor, i64_min: torch.Tensor, group=None) -> None:
    """The three reductions of the flat merge buffers (in place, issued back to back)."""
    works = [dist.all_reduce(i64_sum, op=dist.ReduceOp.SUM, group=group, async_op=True)]
    if f64_sum.numel():
        works.append(dist.all_reduce(f64_sum, op=dist.ReduceOp.SUM, group=group, async_op=True))
    works.append(dist.all_reduce(i64_min, op=dist.ReduceOp.MIN, group=group, async_op=True))
    for w in works:
        w.wait()


_BUFS = {}


def merge_table(table, aggs, group=None, same_keys: bool = False, bufs=None):
    """Merge a libpac PacTable across the process group; returns the merged table (the input
    table itself unless a remap onto the union dictionary was needed).

    same_keys=True: the caller asserts every rank's table already has the same groups in the
    same order (dense domains); then the merge is pack + three all_reduce + unpack with no
    host synchronisation, and a wrong assertion ends in PAC_E_MERGE in the table status."""
    from . import api
    t = table
    if not same_keys:
        G = table.check()
        u, same = union_keys(table.group_key[:G], group)
        if not same:
            t = api.remap(table, u, aggs)
    if bufs is None:
        key = (tuple(t.kinds), t.G_cap, str(t.rows.device))
        bufs = _BUFS.get(key)
        if bufs is None:
            bufs = _BUFS[key] = api.MergeBuffers(t.kinds, t.G_cap, t.rows.device)
    api.merge_pack(t, bufs)
    merge_flat(bufs.i64_sum, bufs.f64_sum, bufs.i64_min, group)
    api.merge_unpack(t, bufs)
    return t
