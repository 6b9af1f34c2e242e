"""ctypes wrapper of the CPU oracle (oracle/pac_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product path
(paper_2603_15023_b200) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "pac_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

COUNT, SUM_I64, SUM_F64, AVG_F64, MIN_F64, MAX_F64 = range(6)
M = 64


def build(force: bool = False) -> str:
    """Compile the oracle with the host compiler (plain C, -O2, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", LIB, SRC, "-lm"])
    return LIB


_lib = None
_P = ctypes.c_void_p


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        L.orc_philox4x32_10.argtypes = [_P, _P, _P]
        L.orc_fmix64.restype = ctypes.c_uint64
        L.orc_fmix64.argtypes = [ctypes.c_uint64]
        L.orc_pac_hash.restype = ctypes.c_uint64
        L.orc_pac_hash.argtypes = [ctypes.c_int64, ctypes.c_uint64]
        L.orc_pac_hash_n.argtypes = [_P, ctypes.c_int64, ctypes.c_uint64, _P]
        L.orc_session_init.argtypes = [ctypes.c_uint64, _P, _P, _P]
        L.orc_pack_key.restype = ctypes.c_uint64
        L.orc_group_keys.restype = ctypes.c_int64
        L.orc_group_keys.argtypes = [_P, _P, ctypes.c_int, _P, ctypes.c_int64, _P, ctypes.c_int64]
        for f in (L.orc_agg_o1, L.orc_agg_o2):
            f.restype = ctypes.c_int
            f.argtypes = [_P, ctypes.c_int64, _P, _P, ctypes.c_int, _P, ctypes.c_int64, _P, _P,
                          ctypes.c_int, _P, _P, _P, _P]
        L.orc_y_vector.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, _P, _P, _P]
        L.orc_weighted_var.restype = ctypes.c_double
        L.orc_weighted_var.argtypes = [_P, _P]
        L.orc_normal.restype = ctypes.c_double
        L.orc_normal.argtypes = [_P]
        L.orc_posterior_update.argtypes = [_P, _P, ctypes.c_double, ctypes.c_double]
        L.orc_lift.argtypes = [ctypes.c_int, ctypes.c_int64, _P, _P, ctypes.c_double, _P, _P, ctypes.c_double,
                               _P, _P]
        L.orc_lift_cmp.argtypes = [ctypes.c_int, ctypes.c_int64, _P, _P, ctypes.c_double, _P, _P,
                                   ctypes.c_double, _P]
        L.orc_cmp_bits.restype = ctypes.c_uint64
        L.orc_cmp_bits.argtypes = [ctypes.c_int, ctypes.c_double, _P, ctypes.c_uint64]
        L.orc_select.argtypes = [ctypes.c_int64, _P, _P, _P, _P]
        L.orc_select_cmp.argtypes = [ctypes.c_int, ctypes.c_int64, _P, _P, _P, _P, _P, _P]
        L.orc_filter.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64, _P, _P]
        L.orc_filter_cmp.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_int64, _P, _P,
                                     _P, _P, _P]
        L.orc_join_chain_mask.argtypes = [ctypes.c_int, _P, _P, _P, _P, ctypes.c_int64, ctypes.c_uint64, _P, _P, _P]
        L.orc_pac_hash128_n.argtypes = [_P, ctypes.c_int64, ctypes.c_uint64, _P]
        L.orc_session_init128.argtypes = [ctypes.c_uint64, _P, _P, _P]
        L.orc_agg128.restype = ctypes.c_int
        L.orc_agg128.argtypes = [_P, ctypes.c_int64, _P, _P, ctypes.c_int, _P, ctypes.c_int64, _P, _P,
                                 ctypes.c_int, _P, _P, _P, _P]
        L.orc_finalize128.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_int, _P, ctypes.c_int64,
                                      ctypes.c_int, _P, _P, _P, _P, _P, ctypes.c_uint32, _P, _P, _P, _P]
        L.orc_noised_y.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_int, _P, ctypes.c_int64, _P, _P,
                                   ctypes.c_uint32, _P, _P, _P]
        L.orc_finalize.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_int, _P, ctypes.c_int64,
                                   ctypes.c_int, _P, _P, _P, _P, _P, ctypes.c_uint32, _P, _P, _P, _P]
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


# ------------------------------------------------------------------ primitives

def philox(ctr: Sequence[int], key: Sequence[int]) -> List[int]:
    c = np.array(ctr, dtype=np.uint32)
    k = np.array(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    _load().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(o))
    return [int(v) for v in o]


def fmix64(z: int) -> int:
    return int(_load().orc_fmix64(z & 0xFFFFFFFFFFFFFFFF))


def pac_hash(keys: np.ndarray, salt: int) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    out = np.empty(keys.shape[0], dtype=np.uint64)
    _load().orc_pac_hash_n(_ptr(keys), keys.shape[0], salt & 0xFFFFFFFFFFFFFFFF, _ptr(out))
    return out


def session(seed: int):
    """(jstar, salt, P) for a session seed (R13)."""
    j = ctypes.c_int(0)
    s = ctypes.c_uint64(0)
    P = np.zeros(M, dtype=np.float64)
    _load().orc_session_init(seed & 0xFFFFFFFFFFFFFFFF, ctypes.byref(j), ctypes.byref(s), _ptr(P))
    return int(j.value), int(s.value), P


def normal_from_block(x: Sequence[int]) -> float:
    a = np.array(x, dtype=np.uint32)
    return float(_load().orc_normal(_ptr(a)))


def weighted_var(P: np.ndarray, y: np.ndarray) -> float:
    P = np.ascontiguousarray(P, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return float(_load().orc_weighted_var(_ptr(P), _ptr(y)))


def posterior_update(P: np.ndarray, y: np.ndarray, ytilde: float, delta: float) -> np.ndarray:
    P = np.array(P, dtype=np.float64, copy=True)
    y = np.ascontiguousarray(y, dtype=np.float64)
    _load().orc_posterior_update(_ptr(P), _ptr(y), float(ytilde), float(delta))
    return P


# ------------------------------------------------------------------ tables

class _Cols:
    def __init__(self, key_cols: Sequence[np.ndarray]):
        self.arrs = [np.ascontiguousarray(c) for c in key_cols]
        self.ptrs = (ctypes.c_void_p * max(1, len(self.arrs)))(*[a.ctypes.data for a in self.arrs])
        self.eb = np.array([a.dtype.itemsize for a in self.arrs] or [0], dtype=np.int32)
        self.n = len(self.arrs)


def pack_keys(key_cols: Sequence[np.ndarray]) -> np.ndarray:
    """Packed composite key per row (R20), via the oracle."""
    cols = _Cols(key_cols)
    n = cols.arrs[0].shape[0] if cols.n else 0
    L = _load()
    L.orc_pack_key.argtypes = [_P, _P, ctypes.c_int, ctypes.c_int64]
    return np.array([L.orc_pack_key(cols.ptrs, _ptr(cols.eb), cols.n, i) for i in range(n)],
                    dtype=np.uint64)


def group_keys(key_cols: Sequence[np.ndarray], masks: np.ndarray) -> np.ndarray:
    cols = _Cols(key_cols)
    masks = np.ascontiguousarray(masks, dtype=np.uint64)
    n = masks.shape[0]
    L = _load()
    G = L.orc_group_keys(cols.ptrs, _ptr(cols.eb), cols.n, _ptr(masks), n, None, 0)
    out = np.zeros(max(G, 1), dtype=np.uint64)
    L.orc_group_keys(cols.ptrs, _ptr(cols.eb), cols.n, _ptr(masks), n, _ptr(out), G)
    return out[:G]


def agg(masks: np.ndarray, key_cols: Sequence[np.ndarray], aggs: Sequence[tuple],
        gkeys: Optional[np.ndarray] = None, method: str = "o2") -> dict:
    """Run O1/O2 on explicit masks.  aggs = [(kind, values or None)].
    gkeys (sorted uint64) restricts the output to those groups (others skipped)."""
    masks = np.ascontiguousarray(masks, dtype=np.uint64)
    n = masks.shape[0]
    cols = _Cols(key_cols)
    if gkeys is None:
        gkeys = group_keys(key_cols, masks)
    gkeys = np.ascontiguousarray(gkeys, dtype=np.uint64)
    G = gkeys.shape[0]
    kinds = np.array([k for k, _ in aggs], dtype=np.int32)
    vals = [None if v is None else np.ascontiguousarray(v) for _, v in aggs]
    vptr = (ctypes.c_void_p * max(1, len(aggs)))(*[None if v is None else v.ctypes.data for v in vals])
    rows = np.zeros(G, dtype=np.int64)
    K = np.zeros(G, dtype=np.uint64)
    count = np.zeros((G, M), dtype=np.int64)
    worlds = []
    for k, _ in aggs:
        if k == COUNT:
            worlds.append(None)
        elif k == SUM_I64:
            worlds.append(np.zeros((G, M), dtype=np.int64))
        else:
            worlds.append(np.zeros((G, M), dtype=np.float64))
    wptr = (ctypes.c_void_p * max(1, len(aggs)))(*[None if w is None else w.ctypes.data for w in worlds])
    fn = _load().orc_agg_o1 if method == "o1" else _load().orc_agg_o2
    ovf = fn(_ptr(masks), n, cols.ptrs, _ptr(cols.eb), cols.n, _ptr(gkeys), G, _ptr(kinds), vptr,
             len(aggs), _ptr(rows), _ptr(K), _ptr(count), wptr)
    return {"G": G, "keys": gkeys, "rows": rows, "K": K, "count": count, "world": worlds,
            "kinds": [k for k, _ in aggs], "overflow": bool(ovf)}


def _table_ptrs(t):
    return (t["rows"], t["K"], t["count"],
            (ctypes.c_void_p * max(1, len(t["world"])))(*[None if w is None else w.ctypes.data for w in t["world"]]))


def combine(a: dict, b: dict) -> dict:
    """a <- a (+) b (state.combine, P:L1966 / P:L2010) for two partial tables over the same
    groups; returns a."""
    assert a["G"] == b["G"] and np.array_equal(a["keys"], b["keys"])
    kinds = np.array(a["kinds"], dtype=np.int32)
    ra, Ka, ca, wa = _table_ptrs(a)
    rb, Kb, cb, wb = _table_ptrs(b)
    L = _load()
    L.orc_combine.restype = ctypes.c_int
    L.orc_combine.argtypes = [ctypes.c_int64, _P, ctypes.c_int, _P, _P, _P, _P, _P, _P, _P, _P]
    ovf = L.orc_combine(a["G"], _ptr(kinds), len(kinds), _ptr(ra), _ptr(Ka), _ptr(ca), wa,
                        _ptr(rb), _ptr(Kb), _ptr(cb), wb)
    a["overflow"] = bool(a["overflow"] or b["overflow"] or ovf)
    return a


def _ranges(n: int, parts: int):
    parts = max(1, min(parts, max(1, n)))
    return [(n * i // parts, n * (i + 1) // parts) for i in range(parts)]


def pac_hash_mt(keys: np.ndarray, salt: int, threads: int) -> np.ndarray:
    """pac_hash on `threads` host threads (contiguous row ranges; ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    out = np.empty(keys.shape[0], dtype=np.uint64)
    L = _load()

    def run(r):
        a, b = r
        if b > a:
            L.orc_pac_hash_n(keys[a:].ctypes.data, b - a, salt & 0xFFFFFFFFFFFFFFFF, out[a:].ctypes.data)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, _ranges(len(keys), threads)))
    return out


def agg_mt(masks: np.ndarray, key_cols: Sequence[np.ndarray], aggs: Sequence[tuple], threads: int) -> dict:
    """O2 on `threads` host threads: each thread runs O2 on a contiguous row range (group keys per
    range, then their sorted union), the partial tables are combined in thread order (SURVEY
    §8c O2 "per-thread states, merged in thread order").  CPU-baseline timing only."""
    from concurrent.futures import ThreadPoolExecutor
    masks = np.ascontiguousarray(masks, dtype=np.uint64)
    key_cols = [np.ascontiguousarray(c) for c in key_cols]
    aggs = [(k, None if v is None else np.ascontiguousarray(v)) for k, v in aggs]
    rng = _ranges(masks.shape[0], threads)
    with ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(lambda r: group_keys([c[r[0]:r[1]] for c in key_cols], masks[r[0]:r[1]]), rng))
    gk = np.unique(np.concatenate(parts)) if parts else np.zeros(0, dtype=np.uint64)
    if not key_cols:
        gk = np.zeros(1, dtype=np.uint64)
    sub = lambda r: agg(masks[r[0]:r[1]], [c[r[0]:r[1]] for c in key_cols],
                        [(k, None if v is None else v[r[0]:r[1]]) for k, v in aggs], gkeys=gk)
    with ThreadPoolExecutor(threads) as ex:
        tabs = list(ex.map(sub, rng))
    out = tabs[0]
    for t in tabs[1:]:
        combine(out, t)
    return out


def agg_from_keys(pu_keys: np.ndarray, salt: int, key_cols, aggs, gkeys=None, method="o2") -> dict:
    return agg(pac_hash(pu_keys, salt), key_cols, aggs, gkeys=gkeys, method=method)


def y_vector(table: dict, a: int, g: int) -> np.ndarray:
    y = np.zeros(M, dtype=np.float64)
    w = table["world"][a]
    _load().orc_y_vector(table["kinds"][a], g, int(table["K"][g]), _ptr(table["count"]),
                         _ptr(w) if w is not None else None, _ptr(y))
    return y


def finalize(seed: int, B: float, jstar: int, P: np.ndarray, table: dict, round_: int = 0):
    """pac_noised over all cells of `table` (one round).  Returns
    (release[G,A], is_null[G,A], flags[G], delta[G,A], P_after)."""
    G = table["G"]
    A = len(table["kinds"])
    P = np.array(P, dtype=np.float64, copy=True)
    kinds = np.array(table["kinds"], dtype=np.int32)
    wptr = (ctypes.c_void_p * max(1, A))(*[None if w is None else w.ctypes.data for w in table["world"]])
    release = np.zeros((G, A), dtype=np.float64)
    is_null = np.zeros((G, A), dtype=np.uint8)
    flags = np.zeros(G, dtype=np.uint8)
    delta = np.zeros((G, A), dtype=np.float64)
    _load().orc_finalize(seed & 0xFFFFFFFFFFFFFFFF, float(B), int(jstar), _ptr(P), G, A, _ptr(kinds),
                         _ptr(table["K"]), _ptr(table["rows"]), _ptr(table["count"]), wptr,
                         int(round_), _ptr(release), _ptr(is_null), _ptr(flags), _ptr(delta))
    return release, is_null, flags, delta, P


# ------------------------------------------------------------------ categorical path (§8 f1)
OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_MIN, OP_MAX = range(6)
CMP_LT, CMP_LE, CMP_GT, CMP_GE, CMP_EQ = range(5)


def world_vectors(table: dict, a: int):
    """(y[G,64], presence[G]) of aggregate a of every group (R22)."""
    G = table["G"]
    y = np.stack([y_vector(table, a, g) for g in range(G)]) if G else np.zeros((0, M))
    return y, np.array(table["K"], dtype=np.uint64).copy()


def _vec(x):
    """(pointer to y or None, pointer to presence or None, scalar) of a lift operand:
    a (y, presence) pair or a Python scalar."""
    if isinstance(x, tuple):
        y = np.ascontiguousarray(x[0], dtype=np.float64)
        p = np.ascontiguousarray(x[1], dtype=np.uint64)
        return y, p, 0.0
    return None, None, float(x)


def lift(op: int, a, b, n: int):
    ya, pa, sa = _vec(a)
    yb, pb, sb = _vec(b)
    out = np.zeros((n, M), dtype=np.float64)
    pout = np.zeros(n, dtype=np.uint64)
    _load().orc_lift(op, n, _ptr(ya), _ptr(pa), sa, _ptr(yb), _ptr(pb), sb, _ptr(out), _ptr(pout))
    return out, pout


def lift_cmp(cmp: int, a, b, n: int) -> np.ndarray:
    ya, pa, sa = _vec(a)
    yb, pb, sb = _vec(b)
    bits = np.zeros(n, dtype=np.uint64)
    _load().orc_lift_cmp(cmp, n, _ptr(ya), _ptr(pa), sa, _ptr(yb), _ptr(pb), sb, _ptr(bits))
    return bits


def cmp_bits(cmp: int, v: float, c: np.ndarray, presence: int) -> int:
    c = np.ascontiguousarray(c, dtype=np.float64)
    return int(_load().orc_cmp_bits(cmp, float(v), _ptr(c), presence & 0xFFFFFFFFFFFFFFFF))


def select(h: np.ndarray, gidx: np.ndarray, bits: np.ndarray) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.uint64)
    gidx = np.ascontiguousarray(gidx, dtype=np.int32)
    bits = np.ascontiguousarray(bits, dtype=np.uint64)
    out = np.zeros(len(h), dtype=np.uint64)
    _load().orc_select(len(h), _ptr(h), _ptr(gidx), _ptr(bits), _ptr(out))
    return out


def select_cmp(cmp: int, h, v, gidx, c, presence) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.uint64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    gidx = np.ascontiguousarray(gidx, dtype=np.int32)
    c = np.ascontiguousarray(c, dtype=np.float64)
    presence = np.ascontiguousarray(presence, dtype=np.uint64)
    out = np.zeros(len(h), dtype=np.uint64)
    _load().orc_select_cmp(cmp, len(h), _ptr(h), _ptr(v), _ptr(gidx), _ptr(c), _ptr(presence), _ptr(out))
    return out


def pac_filter(seed: int, round_: int, bits) -> np.ndarray:
    bits = np.ascontiguousarray(bits, dtype=np.uint64)
    out = np.zeros(len(bits), dtype=np.uint8)
    _load().orc_filter(seed & 0xFFFFFFFFFFFFFFFF, round_, len(bits), _ptr(bits), _ptr(out))
    return out


def filter_cmp(seed: int, round_: int, cmp: int, v, gidx, c, presence) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.float64)
    gidx = np.ascontiguousarray(gidx, dtype=np.int32)
    c = np.ascontiguousarray(c, dtype=np.float64)
    presence = np.ascontiguousarray(presence, dtype=np.uint64)
    out = np.zeros(len(v), dtype=np.uint8)
    _load().orc_filter_cmp(seed & 0xFFFFFFFFFFFFFFFF, round_, cmp, len(v), _ptr(v), _ptr(gidx), _ptr(c),
                           _ptr(presence), _ptr(out))
    return out


def noised_y(seed: int, B: float, jstar: int, P: np.ndarray, y: np.ndarray, presence: np.ndarray,
             round_: int = 0):
    """pac_noised of given world vectors (R24).  Returns (release[n], is_null[n], delta[n], P_after)."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    presence = np.ascontiguousarray(presence, dtype=np.uint64)
    n = len(presence)
    P = np.array(P, dtype=np.float64, copy=True)
    release = np.zeros(n, dtype=np.float64)
    is_null = np.zeros(n, dtype=np.uint8)
    delta = np.zeros(n, dtype=np.float64)
    _load().orc_noised_y(seed & 0xFFFFFFFFFFFFFFFF, float(B), int(jstar), _ptr(P), n, _ptr(y), _ptr(presence),
                         int(round_), _ptr(release), _ptr(is_null), _ptr(delta))
    return release, is_null, delta, P


# ------------------------------------------------------------------ PU-key join (§8 f2)
def join_chain_mask(tables, fk: np.ndarray, salt: int):
    """tables: [(pk, next)] along the FK chain (R27).  Returns (mask, found, pu_key)."""
    k = len(tables)
    pks = [np.ascontiguousarray(t[0], dtype=np.int64) for t in tables]
    nxt = [np.ascontiguousarray(t[1], dtype=np.int64) for t in tables]
    pk_p = (ctypes.c_void_p * max(1, k))(*[a.ctypes.data for a in pks])
    nx_p = (ctypes.c_void_p * max(1, k))(*[a.ctypes.data for a in nxt])
    nb = np.array([len(a) for a in pks], dtype=np.int64)
    fk = np.ascontiguousarray(fk, dtype=np.int64)
    n = len(fk)
    mask = np.zeros(n, dtype=np.uint64)
    found = np.zeros(n, dtype=np.uint8)
    pu = np.zeros(n, dtype=np.int64)
    _load().orc_join_chain_mask(k, pk_p, nx_p, _ptr(nb), _ptr(fk), n, salt & 0xFFFFFFFFFFFFFFFF, _ptr(mask),
                                _ptr(found), _ptr(pu))
    return mask, found, pu


# ------------------------------------------------------------------ m = 128 worlds (§8 f4)
M128 = 128


def pac_hash128(keys: np.ndarray, salt: int) -> np.ndarray:
    """[n, 2] uint64: (lo = worlds 0..63, hi = worlds 64..127), exactly 64 bits set (R28)."""
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    out = np.zeros((len(keys), 2), dtype=np.uint64)
    _load().orc_pac_hash128_n(_ptr(keys), len(keys), salt & 0xFFFFFFFFFFFFFFFF, _ptr(out))
    return out


def session128(seed: int):
    js, salt = ctypes.c_int(), ctypes.c_uint64()
    P = np.zeros(M128, dtype=np.float64)
    _load().orc_session_init128(seed & 0xFFFFFFFFFFFFFFFF, ctypes.byref(js), ctypes.byref(salt), _ptr(P))
    return js.value, salt.value, P


def agg128(masks: np.ndarray, key_cols, aggs) -> dict:
    """Grouped 128-world aggregation (R29); masks [n, 2] uint64."""
    masks = np.ascontiguousarray(masks, dtype=np.uint64).reshape(-1, 2)
    n = len(masks)
    nz = np.ascontiguousarray(masks[:, 0] | masks[:, 1])
    gk = group_keys(key_cols, nz)
    G = len(gk)
    kc = _Cols(key_cols)
    kinds = np.array([k for k, _ in aggs], dtype=np.int32)
    vals = [None if v is None else np.ascontiguousarray(v) for _, v in aggs]
    world = []
    for k, _ in aggs:
        world.append(None if k == COUNT else np.zeros(G * M128, dtype=np.int64 if k == SUM_I64 else np.float64))
    vptr = (ctypes.c_void_p * max(1, len(aggs)))(*[None if v is None else v.ctypes.data for v in vals])
    wptr = (ctypes.c_void_p * max(1, len(aggs)))(*[None if w is None else w.ctypes.data for w in world])
    rows = np.zeros(G, dtype=np.int64)
    K = np.zeros(2 * G, dtype=np.uint64)
    count = np.zeros(G * M128, dtype=np.int64)
    ovf = _load().orc_agg128(_ptr(masks), n, kc.ptrs, _ptr(kc.eb), kc.n, _ptr(gk), G, _ptr(kinds), vptr, len(aggs),
                             _ptr(rows), _ptr(K), _ptr(count), wptr)
    return {"G": G, "keys": gk, "rows": rows, "K": K.reshape(G, 2), "count": count.reshape(G, M128),
            "world": [None if w is None else w.reshape(G, M128) for w in world],
            "kinds": [k for k, _ in aggs], "overflow": bool(ovf)}


def finalize128(seed: int, B: float, jstar: int, P: np.ndarray, table: dict, round_: int = 0):
    G = table["G"]
    A = len(table["kinds"])
    P = np.array(P, dtype=np.float64, copy=True)
    kinds = np.array(table["kinds"], dtype=np.int32)
    world = [None if w is None else np.ascontiguousarray(w) for w in table["world"]]
    wptr = (ctypes.c_void_p * max(1, A))(*[None if w is None else w.ctypes.data for w in world])
    release = np.zeros((G, A), dtype=np.float64)
    is_null = np.zeros((G, A), dtype=np.uint8)
    flags = np.zeros(G, dtype=np.uint8)
    delta = np.zeros((G, A), dtype=np.float64)
    K = np.ascontiguousarray(table["K"], dtype=np.uint64)
    count = np.ascontiguousarray(table["count"], dtype=np.int64)
    _load().orc_finalize128(seed & 0xFFFFFFFFFFFFFFFF, float(B), int(jstar), _ptr(P), G, A, _ptr(kinds), _ptr(K),
                            _ptr(table["rows"]), _ptr(count), wptr, int(round_), _ptr(release), _ptr(is_null),
                            _ptr(flags), _ptr(delta))
    return release, is_null, flags, delta, P


# ------------------------------------------------------------------ approximate SUM (§8 f3)
AL = 25  # levels


def approx_sum(masks: np.ndarray, values: np.ndarray, block_rows: int = 65536, two_sided: bool = True):
    """Approximate (two-sided) SUM of an ungrouped column over the 64 worlds (R35/R36).  Returns
    (counters uint16 [2, 64, 25] -- single-sided: int16 view of [0], y[64] released scale)."""
    masks = np.ascontiguousarray(masks, dtype=np.uint64)
    values = np.ascontiguousarray(values, dtype=np.int64)
    cnt = np.zeros((2, M, AL), dtype=np.uint16)
    y = np.zeros(M, dtype=np.float64)
    L = _load()
    L.orc_approx_sum.argtypes = [_P, ctypes.c_int64, _P, ctypes.c_int64, ctypes.c_int, _P, _P]
    L.orc_approx_sum(_ptr(masks), masks.shape[0], _ptr(values), int(block_rows), 1 if two_sided else 0,
                     _ptr(cnt), _ptr(y))
    return cnt, y
