"""Row-sharded multi-GPU merge (the paper's analogue is DuckDB's thread-local
partial aggregates + state.combine).

Each rank aggregates its contiguous row shard with the same salt, then the partial
64-world tables are merged over NCCL (NVLink / NVSwitch):
  1. union dictionary: all ranks allgather their group keys; the sorted union is the common
     layout (skipped when every rank already has the same keys, e.g. dense group domains);
  2. libpac remaps each table onto the union layout (pac_table_remap);
  3. one coalesced set of all_reduce calls: SUM on int64 {rows, count, SUM_I64 worlds} and
     f64 {SUM_F64 / AVG_F64 worlds}, MIN / MAX on the f64 extremes;
  4. NCCL has no bitwise-OR reduction, so K is re-derived on the device from the merged
     counts or extremes (pac_table_rederive_presence).
Finalize then runs identically on every rank (same table, same session seed).

The communication helpers work on any torch.distributed backend (NCCL on the GPU box,
gloo in the CPU tests); they only move tensors -- no method arithmetic here.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import torch
import torch.distributed as dist

from ._lib import AVG_F64, COUNT, MAX_F64, MIN_F64, SUM_F64, SUM_I64


def reduce_ops_for(kinds: Sequence[int]) -> List[str]:
    """all_reduce op per world array of a table with these aggregate kinds."""
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


_OPS = {"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}


def union_keys(local_keys: torch.Tensor, group=None) -> Tuple[torch.Tensor, bool]:
    """Sorted union (as unsigned 64-bit order) of every rank's group keys (int64 bit
    patterns).  Returns (union, same) where `same` is True when every rank already holds
    exactly the union (no remap needed)."""
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


def allreduce_table_tensors(rows: torch.Tensor, count, worlds: Sequence, kinds: Sequence[int],
                            group=None) -> None:
    """In-place merge of one table laid out on the common dictionary."""
    dist.all_reduce(rows, op=dist.ReduceOp.SUM, group=group)
    if count is not None:
        dist.all_reduce(count, op=dist.ReduceOp.SUM, group=group)
    for w, op in zip(worlds, reduce_ops_for(kinds)):
        if w is None or op == "none":
            continue
        dist.all_reduce(w, op=_OPS[op], group=group)


def merge_table(table, aggs, group=None):
    """Merge a libpac PacTable across the process group; returns the merged table (the
    input table itself when no remap was needed)."""
    from . import api
    G = table.check()
    keys = table.group_key[:G]
    u, same = union_keys(keys, group)
    t = table if same else api.remap(table, u, aggs)
    Gu = u.numel()
    worlds = [None if w is None else w[:Gu] for w in t.world]
    allreduce_table_tensors(t.rows[:Gu], None if t.count is None else t.count[:Gu], worlds, t.kinds, group)
    api.rederive_presence(t, aggs)
    return t
