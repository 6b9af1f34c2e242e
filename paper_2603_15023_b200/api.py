"""Python binding of libpac (include/pac.h): the same calls, torch tensors in, argument
marshalling only.  Every step of the hot path runs in libpac's sm_100a kernels; this
module only allocates device memory (torch), passes pointers and the current stream.

Bit patterns (masks, packed group keys, presence K) travel in int64 tensors; use
`as_u64` to view them as unsigned on the host.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib as L
from ._lib import AVG_F64, COUNT, MAX_F64, MIN_F64, SUM_F64, SUM_I64, PAC_M, PacError, check

_DEV_KEY_BYTES = {torch.int8: 1, torch.int16: 2, torch.int32: 4, torch.int64: 8}


def _stream(dev=None) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def as_u64(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(a).view(np.uint64)


def _require_cuda(*ts):
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise ValueError("libpac takes contiguous CUDA tensors")


# ------------------------------------------------------------------ session (a1)
class Session:
    """pac_session: salt, secret world j*, posterior P on the device."""

    def __init__(self, seed: int, budget: float = 1.0 / 128.0, m: int = PAC_M):
        h = ctypes.c_void_p()
        check("pac_session_create_m", L.lib().pac_session_create_m(seed & 0xFFFFFFFFFFFFFFFF, float(budget), int(m),
                                                                     ctypes.byref(h)))
        self._h = h
        self.m = int(m)
        self.seed = seed & 0xFFFFFFFFFFFFFFFF
        self.budget = float(budget)
        q = self.query()
        self.salt, self.jstar = q["salt"], q["jstar"]

    @property
    def handle(self):
        return self._h

    def query(self) -> dict:
        salt, js, rel, seed = ctypes.c_uint64(), ctypes.c_int32(), ctypes.c_uint64(), ctypes.c_uint64()
        B = ctypes.c_double()
        P = np.zeros(self.m, dtype=np.float64)
        check("pac_session_query", L.lib().pac_session_query(
            self._h, ctypes.byref(salt), ctypes.byref(js), P.ctypes.data, ctypes.byref(rel),
            ctypes.byref(seed), ctypes.byref(B)))
        return {"salt": salt.value, "jstar": js.value, "P": P, "releases": rel.value,
                "seed": seed.value, "budget": B.value}

    def set_posterior(self, P: np.ndarray) -> None:
        P = np.ascontiguousarray(P, dtype=np.float64)
        check("pac_session_set_posterior", L.lib().pac_session_set_posterior(self._h, P.ctypes.data))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            L.lib().pac_session_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ mask (a2)
def mask(pu_keys: torch.Tensor, salt: int, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """pac_hash of every key: int64 tensor holding the 64-bit masks."""
    _require_cuda(pu_keys)
    if pu_keys.dtype != torch.int64:
        raise ValueError("pu_keys must be int64")
    n = pu_keys.numel()
    if out is None:
        out = torch.empty(n, dtype=torch.int64, device=pu_keys.device)
    check("pac_mask", L.lib().pac_mask(_ptr(pu_keys), n, salt & 0xFFFFFFFFFFFFFFFF, _ptr(out),
                                        _stream(pu_keys.device)))
    return out


# ------------------------------------------------------------------ table (a3-a5)
@dataclass
class PacTable:
    kinds: List[int]
    G_cap: int
    num_groups: torch.Tensor
    status: torch.Tensor
    group_key: torch.Tensor
    rows: torch.Tensor
    presence: torch.Tensor
    count: Optional[torch.Tensor]
    world: List[Optional[torch.Tensor]]
    _struct: Optional[L.Table] = field(default=None, repr=False)

    m: int = PAC_M

    @staticmethod
    def allocate(kinds: Sequence[int], G_cap: int, device, m: int = PAC_M) -> "PacTable":
        """m = 64, or 128 (§8 f4: presence [G_cap, 2], count / worlds [G_cap, 128])."""
        kinds = list(kinds)
        mm_only = all(k in (MIN_F64, MAX_F64) for k in kinds)
        z = lambda *s, dt=torch.int64: torch.zeros(*s, dtype=dt, device=device)
        world = []
        for k in kinds:
            if k == COUNT:
                world.append(None)
            elif k == SUM_I64:
                world.append(z(G_cap, m))
            else:
                world.append(z(G_cap, m, dt=torch.float64))
        pres = z(G_cap) if m == PAC_M else z(G_cap, m // 64)
        return PacTable(kinds, G_cap, z(1), z(1, dt=torch.int32), z(G_cap), z(G_cap), pres,
                        None if mm_only else z(G_cap, m), world, m=m)

    def struct(self) -> L.Table:
        if self._struct is None:
            t = L.Table()
            t.d_num_groups = self.num_groups.data_ptr()
            t.d_status = self.status.data_ptr()
            t.d_group_key = self.group_key.data_ptr()
            t.d_rows = self.rows.data_ptr()
            t.d_presence = self.presence.data_ptr()
            t.d_count = self.count.data_ptr() if self.count is not None else None
            for a, w in enumerate(self.world):
                t.d_world[a] = w.data_ptr() if w is not None else None
            t.m = self.m
            self._struct = t
        return self._struct

    def check(self) -> int:
        """Synchronizing: number of groups; raises PacError on CAPACITY / OVERFLOW."""
        G = ctypes.c_int64()
        rc = L.lib().pac_table_check(ctypes.byref(self.struct()), ctypes.byref(G), _stream(self.rows.device))
        if rc != L.PAC_OK:
            raise PacError("pac_table_check", rc)
        return int(G.value)

    def to_host(self) -> dict:
        G = self.check()
        return {
            "G": G,
            "keys": as_u64(self.group_key[:G]),
            "rows": self.rows[:G].cpu().numpy(),
            "K": as_u64(self.presence[:G]) if self.m == PAC_M else as_u64(self.presence[:G].contiguous()).reshape(G, self.m // PAC_M),
            "count": None if self.count is None else self.count[:G].cpu().numpy(),
            "world": [None if w is None else w[:G].cpu().numpy() for w in self.world],
            "kinds": list(self.kinds),
        }


def _agg_specs(aggs: Sequence[Tuple[int, Optional[torch.Tensor]]]):
    arr = (L.AggSpec * max(1, len(aggs)))()
    for a, (k, v) in enumerate(aggs):
        if v is not None:
            _require_cuda(v)
            want = torch.int64 if k == SUM_I64 else torch.float64
            if v.dtype != want:
                raise ValueError(f"aggregate {a}: values must be {want}")
        arr[a].kind = int(k)
        arr[a].d_values = None if v is None else v.data_ptr()
    return arr


def _key_cols(keys: Sequence[torch.Tensor]):
    arr = (L.KeyCol * max(1, len(keys)))()
    for c, k in enumerate(keys):
        _require_cuda(k)
        if k.dtype not in _DEV_KEY_BYTES:
            raise ValueError("group key columns must be int8/16/32/64")
        arr[c].d_col = k.data_ptr()
        arr[c].elem_bytes = _DEV_KEY_BYTES[k.dtype]
    return arr


class Aggregator:
    """pac_agg_grouped with a cached workspace and output table (reused across calls)."""

    def __init__(self, kinds: Sequence[int], G_cap: int, device="cuda", spill_rows: Optional[int] = None):
        """spill_rows: record capacity of the deferred HBM tier (default: every row of the call;
        0: direct atomics; fewer than the tier rows: the rest take atomics)."""
        self.kinds = list(kinds)
        self.G_cap = int(G_cap)
        self.device = torch.device(device)
        self.table = PacTable.allocate(self.kinds, self.G_cap, self.device)
        self.spill_rows = spill_rows
        self._ws = None

    def _workspace(self, specs, n_aggs, n_rows):
        nb = ctypes.c_size_t()
        rows = n_rows if self.spill_rows is None else min(n_rows, int(self.spill_rows))
        check("pac_agg_workspace_size_rows", L.lib().pac_agg_workspace_size_rows(
            specs, n_aggs, self.G_cap, rows, ctypes.byref(nb)))
        if self._ws is None or self._ws.numel() < nb.value:
            self._ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=self.device)
        return self._ws, nb.value

    def __call__(self, values: Sequence[Optional[torch.Tensor]], keys: Sequence[torch.Tensor] = (),
                 pu_key: Optional[torch.Tensor] = None, mask: Optional[torch.Tensor] = None,
                 salt: int = 0) -> PacTable:
        if len(values) != len(self.kinds):
            raise ValueError("one value tensor (or None for COUNT) per aggregate")
        aggs = list(zip(self.kinds, values))
        specs = _agg_specs(aggs)
        kc = _key_cols(keys)
        _require_cuda(pu_key, mask)
        n = (pu_key if pu_key is not None else mask).numel()
        ws, nb = self._workspace(specs, len(aggs), n)
        t = self.table
        check("pac_agg_grouped", L.lib().pac_agg_grouped(
            _ptr(pu_key), _ptr(mask), salt & 0xFFFFFFFFFFFFFFFF, kc, len(keys), specs, len(aggs), n,
            ctypes.byref(t.struct()), self.G_cap, _ptr(ws), nb, _stream(self.device)))
        return t


class Aggregator128:
    """pac_agg_grouped128 (§8 f4): grouped aggregation over m = 128 worlds (R29)."""

    def __init__(self, kinds: Sequence[int], G_cap: int, device="cuda"):
        self.kinds = list(kinds)
        self.G_cap = int(G_cap)
        self.device = torch.device(device)
        self.table = PacTable.allocate(self.kinds, self.G_cap, self.device, m=128)
        self._ws = None

    def __call__(self, values: Sequence[Optional[torch.Tensor]], keys: Sequence[torch.Tensor] = (),
                 pu_key: Optional[torch.Tensor] = None, mask2: Optional[torch.Tensor] = None,
                 salt: int = 0) -> PacTable:
        aggs = list(zip(self.kinds, values))
        specs = _agg_specs(aggs)
        kc = _key_cols(keys)
        _require_cuda(pu_key, mask2)
        n = pu_key.numel() if pu_key is not None else mask2.shape[0]
        nb = ctypes.c_size_t()
        check("pac_agg_workspace_size128", L.lib().pac_agg_workspace_size128(
            specs, len(aggs), self.G_cap, n, 1 if pu_key is not None else 0, ctypes.byref(nb)))
        if self._ws is None or self._ws.numel() < nb.value:
            self._ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=self.device)
        t = self.table
        check("pac_agg_grouped128", L.lib().pac_agg_grouped128(
            _ptr(pu_key), _ptr(mask2), salt & 0xFFFFFFFFFFFFFFFF, kc, len(keys), specs, len(aggs), n,
            ctypes.byref(t.struct()), self.G_cap, _ptr(self._ws), nb.value, _stream(self.device)))
        return t


def mask128(pu_keys: torch.Tensor, salt: int) -> torch.Tensor:
    """pac_hash over 128 worlds (R28): int64 [n, 2] bit patterns (lo, hi)."""
    _require_cuda(pu_keys)
    out = torch.empty(pu_keys.numel(), 2, dtype=torch.int64, device=pu_keys.device)
    check("pac_mask128", L.lib().pac_mask128(_ptr(pu_keys), pu_keys.numel(), salt & 0xFFFFFFFFFFFFFFFF, _ptr(out),
                                              _stream(pu_keys.device)))
    return out


def agg_grouped(aggs: Sequence[Tuple[int, Optional[torch.Tensor]]], keys: Sequence[torch.Tensor] = (),
                pu_key: Optional[torch.Tensor] = None, mask: Optional[torch.Tensor] = None, salt: int = 0,
                G_cap: int = 1024) -> PacTable:
    dev = (pu_key if pu_key is not None else mask).device
    ag = Aggregator([k for k, _ in aggs], G_cap, dev)
    return ag([v for _, v in aggs], keys, pu_key=pu_key, mask=mask, salt=salt)


def rederive_presence(table: PacTable, aggs) -> None:
    specs = _agg_specs([(k, v) for k, v in aggs])
    check("pac_table_rederive_presence", L.lib().pac_table_rederive_presence(
        ctypes.byref(table.struct()), specs, len(aggs), table.G_cap, _stream(table.rows.device)))


def remap(table: PacTable, union_keys: torch.Tensor, aggs) -> PacTable:
    """Lay `table` out on the ascending union dictionary `union_keys` (int64 bit patterns)."""
    Gu = union_keys.numel()
    out = PacTable.allocate(table.kinds, max(Gu, 1), table.rows.device)
    specs = _agg_specs([(k, v) for k, v in aggs])
    check("pac_table_remap", L.lib().pac_table_remap(
        ctypes.byref(table.struct()), _ptr(union_keys), Gu, specs, len(aggs), table.G_cap,
        ctypes.byref(out.struct()), _stream(table.rows.device)))
    return out


class MergeBuffers:
    """The three flat buffers of pac_merge_pack / pac_merge_unpack for tables of these kinds and
    capacity: i64_sum (all_reduce SUM), f64_sum (SUM, may be empty), i64_min (MIN)."""

    def __init__(self, kinds: Sequence[int], G_cap: int, device):
        self.kinds = list(kinds)
        self.G_cap = int(G_cap)
        specs = _agg_specs([(k, None) for k in self.kinds])
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check("pac_merge_sizes", L.lib().pac_merge_sizes(specs, len(self.kinds), self.G_cap, ctypes.byref(a),
                                                          ctypes.byref(b), ctypes.byref(c)))
        self.i64_sum = torch.empty(a.value, dtype=torch.int64, device=device)
        self.f64_sum = torch.empty(b.value, dtype=torch.float64, device=device)
        self.i64_min = torch.empty(c.value, dtype=torch.int64, device=device)


def merge_pack(table: PacTable, bufs: MergeBuffers) -> None:
    specs = _agg_specs([(k, None) for k in table.kinds])
    check("pac_merge_pack", L.lib().pac_merge_pack(
        ctypes.byref(table.struct()), specs, len(table.kinds), bufs.G_cap, _ptr(bufs.i64_sum),
        _ptr(bufs.f64_sum) if bufs.f64_sum.numel() else None, _ptr(bufs.i64_min), _stream(table.rows.device)))


def merge_unpack(table: PacTable, bufs: MergeBuffers) -> None:
    specs = _agg_specs([(k, None) for k in table.kinds])
    check("pac_merge_unpack", L.lib().pac_merge_unpack(
        ctypes.byref(table.struct()), specs, len(table.kinds), bufs.G_cap, _ptr(bufs.i64_sum),
        _ptr(bufs.f64_sum) if bufs.f64_sum.numel() else None, _ptr(bufs.i64_min), _stream(table.rows.device)))


# ------------------------------------------------------------------ finalize (a6, a7)
class Finalizer:
    """pac_finalize with cached workspace/outputs."""

    def __init__(self, kinds: Sequence[int], G_cap: int, device="cuda"):
        self.kinds = list(kinds)
        self.G_cap = int(G_cap)
        dev = torch.device(device)
        A = len(self.kinds)
        nb = ctypes.c_size_t()
        check("pac_finalize_workspace_size", L.lib().pac_finalize_workspace_size(self.G_cap, A,
                                                                                   ctypes.byref(nb)))
        self.ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
        self.ws_bytes = nb.value
        self.release = torch.empty(self.G_cap, A, dtype=torch.float64, device=dev)
        self.is_null = torch.empty(self.G_cap, A, dtype=torch.uint8, device=dev)
        self.flags = torch.empty(self.G_cap, dtype=torch.uint8, device=dev)
        self.delta = torch.empty(self.G_cap, A, dtype=torch.float64, device=dev)

    def __call__(self, session: Session, table: PacTable, round_: int = 0):
        specs = _agg_specs([(k, w) for k, w in zip(table.kinds, table.world)])
        check("pac_finalize", L.lib().pac_finalize(
            session.handle, ctypes.byref(table.struct()), specs, len(self.kinds), self.G_cap, int(round_),
            _ptr(self.release), _ptr(self.is_null), _ptr(self.flags), _ptr(self.delta), _ptr(self.ws),
            self.ws_bytes, _stream(self.release.device)))
        return self.release, self.is_null, self.flags, self.delta


def finalize(session: Session, table: PacTable, round_: int = 0):
    return Finalizer(table.kinds, table.G_cap, table.rows.device)(session, table, round_)


def posterior_update(session: Session, y64: torch.Tensor, y_tilde: float, delta: float) -> None:
    _require_cuda(y64)
    check("pac_posterior_update", L.lib().pac_posterior_update(session.handle, _ptr(y64), float(y_tilde),
                                                                float(delta), _stream(y64.device)))


# ------------------------------------------------------------------ categorical path (§8 f1)
# World vectors are (y, presence) pairs: y float64 [n, 64] in the released scale (R22),
# presence int64 [n] holding the 64-bit masks.  A Python number is a broadcast scalar.
from ._lib import (CMP_EQ, CMP_GE, CMP_GT, CMP_LE, CMP_LT, OP_ADD, OP_DIV, OP_MAX,  # noqa: E402
                   OP_MIN, OP_MUL, OP_SUB)


def world_vector(table: PacTable, a: int) -> Tuple[torch.Tensor, torch.Tensor]:
    """pac_world_vector: the y-vectors of aggregate a of every group (R22)."""
    dev = table.rows.device
    y = torch.empty(table.G_cap, PAC_M, dtype=torch.float64, device=dev)
    pres = torch.empty(table.G_cap, dtype=torch.int64, device=dev)
    specs = _agg_specs([(k, w) for k, w in zip(table.kinds, table.world)])
    check("pac_world_vector", L.lib().pac_world_vector(ctypes.byref(table.struct()), specs, len(table.kinds), a,
                                                        table.G_cap, _ptr(y), _ptr(pres), _stream(dev)))
    return y, pres


def _wvec(x):
    w = L.WVec()
    if isinstance(x, tuple):
        y, p = x
        _require_cuda(y, p)
        w.d_y, w.d_presence, w.scalar = y.data_ptr(), p.data_ptr(), 0.0
        return w, y.shape[0], y.device
    w.d_y, w.d_presence, w.scalar = None, None, float(x)
    return w, None, None


def _operands(a, b):
    wa, na, da = _wvec(a)
    wb, nb, db = _wvec(b)
    n = na if na is not None else nb
    if n is None:
        raise ValueError("at least one operand must be a world vector")
    if na is not None and nb is not None and na != nb:
        raise ValueError("world vector operands differ in length")
    return wa, wb, n, da if da is not None else db


def lift(op: int, a, b) -> Tuple[torch.Tensor, torch.Tensor]:
    """pac_lift: pointwise a OP b over world vectors / broadcast scalars (R23)."""
    wa, wb, n, dev = _operands(a, b)
    out = torch.empty(n, PAC_M, dtype=torch.float64, device=dev)
    pres = torch.empty(n, dtype=torch.int64, device=dev)
    check("pac_lift", L.lib().pac_lift(int(op), ctypes.byref(wa), ctypes.byref(wb), n, _ptr(out), _ptr(pres),
                                        _stream(dev)))
    return out, pres


def lift_cmp(cmp: int, a, b) -> torch.Tensor:
    """pac_lift_cmp: world booleans (int64 bit patterns) of a CMP b (R23, R26)."""
    wa, wb, n, dev = _operands(a, b)
    bits = torch.empty(n, dtype=torch.int64, device=dev)
    check("pac_lift_cmp", L.lib().pac_lift_cmp(int(cmp), ctypes.byref(wa), ctypes.byref(wb), n, _ptr(bits),
                                                _stream(dev)))
    return bits


class NoisedY:
    """pac_noised_y with a cached workspace (R24)."""

    def __init__(self, n: int, device="cuda"):
        self.n = int(n)
        dev = torch.device(device)
        nb = ctypes.c_size_t()
        check("pac_noised_y_workspace_size", L.lib().pac_noised_y_workspace_size(self.n, ctypes.byref(nb)))
        self.ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=dev)
        self.ws_bytes = nb.value
        self.release = torch.empty(self.n, dtype=torch.float64, device=dev)
        self.is_null = torch.empty(self.n, dtype=torch.uint8, device=dev)
        self.delta = torch.empty(self.n, dtype=torch.float64, device=dev)

    def __call__(self, session: Session, y: torch.Tensor, presence: torch.Tensor, round_: int = 0):
        _require_cuda(y, presence)
        n = presence.numel()
        if n > self.n:
            raise ValueError("more vectors than the NoisedY capacity")
        check("pac_noised_y", L.lib().pac_noised_y(
            session.handle, _ptr(y), _ptr(presence), n, int(round_), _ptr(self.release), _ptr(self.is_null),
            _ptr(self.delta), _ptr(self.ws), self.ws_bytes, _stream(y.device)))
        return self.release[:n], self.is_null[:n], self.delta[:n]


def noised_y(session: Session, y: torch.Tensor, presence: torch.Tensor, round_: int = 0):
    return NoisedY(presence.numel(), y.device)(session, y, presence, round_)


def cmp_index(c: torch.Tensor, presence: torch.Tensor) -> torch.Tensor:
    """pac_cmp_index: sorted world values + suffix masks per group, for select_cmp / filter_cmp."""
    _require_cuda(c, presence)
    G = presence.numel()
    ix = torch.empty(G, L.PAC_CMP_INDEX_WORDS, dtype=torch.int64, device=c.device)
    check("pac_cmp_index", L.lib().pac_cmp_index(_ptr(c), _ptr(presence), G, _ptr(ix), _stream(c.device)))
    return ix


def select(h: torch.Tensor, gidx: torch.Tensor, bits: torch.Tensor, out: Optional[torch.Tensor] = None):
    """pac_select: h AND bits[gidx] (Eq. pac-select) -- reduced masks for an upstream aggregate."""
    _require_cuda(h, gidx, bits)
    out = torch.empty_like(h) if out is None else out
    check("pac_select", L.lib().pac_select(_ptr(h), _ptr(gidx), _ptr(bits), h.numel(), _ptr(out),
                                            _stream(h.device)))
    return out


def select_cmp(cmp: int, h: torch.Tensor, v: torch.Tensor, gidx: torch.Tensor, index: torch.Tensor,
               out: Optional[torch.Tensor] = None):
    """pac_select_<cmp>: h AND [v CMP c_j] against the row group's world vector."""
    _require_cuda(h, v, gidx, index)
    out = torch.empty_like(h) if out is None else out
    check("pac_select_cmp", L.lib().pac_select_cmp(int(cmp), _ptr(h), _ptr(v), _ptr(gidx), _ptr(index), h.numel(),
                                                    _ptr(out), _stream(h.device)))
    return out


def pac_filter(session: Session, bits: torch.Tensor, round_: int = 0) -> torch.Tensor:
    """pac_filter: 1 with probability popcount(b)/64 (Eq. pac-filter, R25)."""
    _require_cuda(bits)
    out = torch.empty(bits.numel(), dtype=torch.uint8, device=bits.device)
    check("pac_filter", L.lib().pac_filter(session.handle, _ptr(bits), bits.numel(), int(round_), _ptr(out),
                                            _stream(bits.device)))
    return out


def filter_cmp(session: Session, cmp: int, v: torch.Tensor, gidx: torch.Tensor, index: torch.Tensor,
               round_: int = 0) -> torch.Tensor:
    """pac_filter_<cmp>: pac_filter of [v CMP c_j]."""
    _require_cuda(v, gidx, index)
    out = torch.empty(v.numel(), dtype=torch.uint8, device=v.device)
    check("pac_filter_cmp", L.lib().pac_filter_cmp(session.handle, int(cmp), _ptr(v), _ptr(gidx), _ptr(index),
                                                    v.numel(), int(round_), _ptr(out), _stream(v.device)))
    return out


# ------------------------------------------------------------------ PU-key join (§8 f2)
class JoinTable:
    """pac_join_build: primary key -> next foreign key of one table on the FK chain (R27)."""

    def __init__(self, pk: torch.Tensor, nxt: torch.Tensor):
        _require_cuda(pk, nxt)
        if pk.dtype != torch.int64 or nxt.dtype != torch.int64 or pk.numel() != nxt.numel():
            raise ValueError("pk and next must be int64 tensors of one length")
        nb = ctypes.c_size_t()
        check("pac_join_table_bytes", L.lib().pac_join_table_bytes(pk.numel(), ctypes.byref(nb)))
        self.buf = torch.empty((nb.value + 15) // 16 * 2, dtype=torch.int64, device=pk.device)
        self.nbytes = nb.value
        check("pac_join_build", L.lib().pac_join_build(_ptr(pk), _ptr(nxt), pk.numel(), _ptr(self.buf),
                                                        self.nbytes, _stream(pk.device)))

    def status(self) -> int:
        return int(L.lib().pac_join_table_status(_ptr(self.buf), _stream(self.buf.device)))


def join_mask(tables: Sequence[JoinTable], fk: torch.Tensor, salt: int, want_pu: bool = False):
    """pac_join_mask: masks of the rows' PU keys reached along the FK chain (join elimination)."""
    _require_cuda(fk)
    k = len(tables)
    arr = (ctypes.c_void_p * max(1, k))(*[t.buf.data_ptr() for t in tables])
    mask = torch.empty_like(fk)
    pu = torch.empty_like(fk) if want_pu else None
    check("pac_join_mask", L.lib().pac_join_mask(arr, k, _ptr(fk), fk.numel(), salt & 0xFFFFFFFFFFFFFFFF,
                                                  _ptr(mask), _ptr(pu), _stream(fk.device)))
    return (mask, pu) if want_pu else mask


# ------------------------------------------------------------------ approximate SUM (§8 f3)
def approx_sum(values: torch.Tensor, pu_key: Optional[torch.Tensor] = None, mask: Optional[torch.Tensor] = None,
               salt: int = 0, two_sided: bool = True, block_rows: int = 65536):
    """pac_approx_sum (R35/R36): ungrouped approximate 64-world SUM.  Returns (counters uint16
    [2, 64, 25] as int16 bit patterns in an int16 tensor, y float64 [64])."""
    _require_cuda(values, pu_key, mask)
    n = values.numel()
    nb = ctypes.c_size_t()
    check("pac_approx_sum_workspace_size", L.lib().pac_approx_sum_workspace_size(n, int(block_rows), ctypes.byref(nb)))
    ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=values.device)
    cnt = torch.zeros(2, PAC_M, 25, dtype=torch.int16, device=values.device)
    y = torch.empty(PAC_M, dtype=torch.float64, device=values.device)
    check("pac_approx_sum", L.lib().pac_approx_sum(_ptr(pu_key), _ptr(mask), salt & 0xFFFFFFFFFFFFFFFF, _ptr(values), n,
                                                    1 if two_sided else 0, int(block_rows), _ptr(cnt), _ptr(y), _ptr(ws),
                                                    nb.value, _stream(values.device)))
    return cnt, y


# ------------------------------------------------------------------ runtime
def launch_count() -> int:
    return int(L.lib().pac_launch_count())


def profile_enable(on: bool) -> None:
    L.lib().pac_profile_enable(1 if on else 0)


def profile_read() -> Tuple[float, int]:
    ms, n = ctypes.c_double(), ctypes.c_int64()
    check("pac_profile_read", L.lib().pac_profile_read(ctypes.byref(ms), ctypes.byref(n)))
    return float(ms.value), int(n.value)


def profile_last_kernel() -> str:
    return L.lib().pac_profile_last_kernel().decode()


def version() -> str:
    return L.lib().pac_version().decode()
