"""Seeded, counter-based synthetic input columns for the PAC hot path.

This module is shared by the oracle side (tests, CPU baseline) and the CUDA side
(tests, bench).  It holds NONE of the method's arithmetic: no pac_hash, no
world accumulation, no noise.  Its mixer is MurmurHash3's fmix64 (constants
0xff51afd7ed558ccd / 0xc4ceb9fe1a85ec53), deliberately different from the
SplitMix64 finalizer the method uses for pac_hash (reading R1).

Every value is a pure function of (seed, column id, global row index), so a row's
bytes do not depend on how rows are sharded across GPUs or tiles.  The numpy
implementation here and the CUDA implementation in ``datagen/csrc/datagen.cu``
produce bit-identical integers and uniform doubles; normals go through libm
(log/cos/sqrt) and may differ in the last ulp between host and device, so parity
tests always feed both sides the same bytes (host-generated and uploaded, or
device-generated and copied back).

Workload recipes (BASELINE.json configs, restated in DESIGN.md "Input recipe"):
  C1 ungrouped COUNT+SUM, C2 low-card grouped, C3 high-card Zipf, C4 MIN/MAX,
  C5 multi-GPU sharded.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Dict, List, Optional

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_M32 = np.uint64(0xFFFFFFFF)

# ---------------------------------------------------------------- primitives

def _fmix_m3(z: np.ndarray) -> np.ndarray:
    """MurmurHash3 fmix64 (bijective) on a uint64 array (wrapping arithmetic)."""
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(33)
        z *= np.uint64(0xFF51AFD7ED558CCD)
        z ^= z >> np.uint64(33)
        z *= np.uint64(0xC4CEB9FE1A85EC53)
        z ^= z >> np.uint64(33)
    return z


def column_key(seed: int, col: int) -> int:
    """Per-(seed, column) key mixed into every row word."""
    with np.errstate(over="ignore"):
        v = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(col) * np.uint64(0xA0761D6478BD642F))
    return int(_fmix_m3(np.array([v], dtype=np.uint64))[0])


def words(seed: int, col: int, row0: int, n: int) -> np.ndarray:
    """The raw 64-bit word of column `col` for global rows row0 .. row0+n-1."""
    key = np.uint64(column_key(seed, col))
    rows = np.arange(n, dtype=np.uint64) + np.uint64(row0)
    with np.errstate(over="ignore"):
        z = rows * np.uint64(0xE7037ED1A0B428DB) + key
    return _fmix_m3(z)


def mulhi64(a: np.ndarray, b: int) -> np.ndarray:
    """floor(a * b / 2^64) for uint64 array a and scalar 0 <= b < 2^64."""
    b = np.uint64(b)
    a_lo, a_hi = a & _M32, a >> np.uint64(32)
    b_lo, b_hi = b & _M32, b >> np.uint64(32)
    with np.errstate(over="ignore"):
        p0 = a_lo * b_lo
        p1 = a_lo * b_hi
        p2 = a_hi * b_lo
        p3 = a_hi * b_hi
        mid = (p0 >> np.uint64(32)) + (p1 & _M32) + (p2 & _M32)
        return p3 + (p1 >> np.uint64(32)) + (p2 >> np.uint64(32)) + (mid >> np.uint64(32))


def scramble32(rank: np.ndarray) -> np.ndarray:
    """Bijective uint32 scramble of a rank -> int32 key (odd multiply + xorshift)."""
    with np.errstate(over="ignore"):
        x = (rank.astype(np.uint64) * np.uint64(0x9E3779B1) + np.uint64(0x7F4A7C15)) & _M32
    x ^= x >> np.uint64(15)
    return x.astype(np.uint32).view(np.int32)


def scramble64(rank: np.ndarray) -> np.ndarray:
    """Bijective uint64 scramble of a rank -> int64 key (murmur fmix64 of rank^c)."""
    return _fmix_m3(rank.astype(np.uint64) ^ np.uint64(0x6A09E667F3BCC909)).view(np.int64)


def unit_f64(w: np.ndarray) -> np.ndarray:
    """53-bit uniform in [0,1): (w >> 11) * 2^-53 (exact)."""
    return (w >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def zipf_cdf(n_distinct: int, s: float) -> np.ndarray:
    """Normalised CDF table of Zipf(s) over ranks 1..n (float64, host-built once)."""
    k = np.arange(1, n_distinct + 1, dtype=np.float64)
    w = k ** (-float(s))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return cdf


# ---------------------------------------------------------------- column specs

KIND_UNIFORM_INT = 1   # lo + mulhi(w, hi-lo+1), stored in elem_bytes
KIND_UNIFORM_KEY64 = 2  # scramble64(mulhi(w, N))
KIND_ZIPF_KEY32 = 3     # scramble32(zipf_rank(u))
KIND_ZIPF_KEY64 = 4     # scramble64(zipf_rank(u))
KIND_UNIFORM_F64 = 5    # lo + unit(w) * (hi - lo)
KIND_NORMAL_F64 = 6     # mu + sigma * BoxMuller(w(col), w(col+1))

_DTYPES = {1: np.int8, 2: np.int16, 4: np.int32, 8: np.int64}


@dataclasses.dataclass(frozen=True)
class ColSpec:
    name: str
    kind: int
    col: int              # column id mixed into the row words
    elem_bytes: int = 8
    lo: float = 0
    hi: float = 0
    n_distinct: int = 0
    zipf_s: float = 0.0

    @property
    def dtype(self):
        if self.kind in (KIND_UNIFORM_F64, KIND_NORMAL_F64):
            return np.float64
        if self.kind == KIND_ZIPF_KEY32:
            return np.int32
        if self.kind in (KIND_UNIFORM_KEY64, KIND_ZIPF_KEY64):
            return np.int64
        return _DTYPES[self.elem_bytes]


_cdf_cache: Dict[tuple, np.ndarray] = {}


def cdf_for(spec: ColSpec) -> np.ndarray:
    key = (spec.n_distinct, spec.zipf_s)
    if key not in _cdf_cache:
        _cdf_cache[key] = zipf_cdf(spec.n_distinct, spec.zipf_s)
    return _cdf_cache[key]


def gen_column(spec: ColSpec, seed: int, row0: int, n: int) -> np.ndarray:
    """Host (numpy) generation of rows row0..row0+n-1 of one column."""
    w = words(seed, spec.col, row0, n)
    if spec.kind == KIND_UNIFORM_INT:
        span = int(spec.hi) - int(spec.lo) + 1
        v = mulhi64(w, span).astype(np.int64) + int(spec.lo)
        return v.astype(_DTYPES[spec.elem_bytes])
    if spec.kind == KIND_UNIFORM_KEY64:
        return scramble64(mulhi64(w, spec.n_distinct))
    if spec.kind in (KIND_ZIPF_KEY32, KIND_ZIPF_KEY64):
        cdf = cdf_for(spec)
        u = unit_f64(w)
        rank = np.searchsorted(cdf, u, side="right")
        rank = np.minimum(rank, spec.n_distinct - 1).astype(np.uint64)
        return scramble32(rank) if spec.kind == KIND_ZIPF_KEY32 else scramble64(rank)
    if spec.kind == KIND_UNIFORM_F64:
        return float(spec.lo) + unit_f64(w) * (float(spec.hi) - float(spec.lo))
    if spec.kind == KIND_NORMAL_F64:
        w2 = words(seed, spec.col + 1, row0, n)
        u1 = ((w >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)
        u2 = ((w2 >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)
        z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
        return float(spec.lo) + float(spec.hi) * z   # lo = mu, hi = sigma
    raise ValueError(f"unknown kind {spec.kind}")


# ---------------------------------------------------------------- workloads

AGG_COUNT, AGG_SUM_I64, AGG_SUM_F64, AGG_AVG_F64, AGG_MIN_F64, AGG_MAX_F64 = range(6)


@dataclasses.dataclass(frozen=True)
class Workload:
    """One BASELINE.json config as concrete synthetic columns."""
    name: str
    n_rows: int
    seed: int
    pu: ColSpec
    keys: List[ColSpec]
    values: List[ColSpec]
    aggs: List[tuple]           # (agg kind, index into values or -1)
    budget: float = 1.0 / 128.0
    rounds: int = 1
    description: str = ""

    @property
    def in_bytes_per_row(self) -> int:
        b = 8 + sum(np.dtype(k.dtype).itemsize for k in self.keys)
        return b + sum(np.dtype(v.dtype).itemsize for v in self.values)

    def scaled(self, n_rows: int) -> "Workload":
        return dataclasses.replace(self, n_rows=int(n_rows))

    def host_columns(self, row0: int = 0, n: Optional[int] = None) -> dict:
        n = self.n_rows if n is None else n
        return {
            "pu": gen_column(self.pu, self.seed, row0, n),
            "keys": [gen_column(k, self.seed, row0, n) for k in self.keys],
            "values": [gen_column(v, self.seed, row0, n) for v in self.values],
        }


def _seed(c: int) -> int:
    return 0x5EED0000 + c


WORKLOADS: Dict[str, Workload] = {
    "C1": Workload(
        name="C1", n_rows=1_000_000, seed=_seed(1),
        pu=ColSpec("pu_key", KIND_UNIFORM_KEY64, col=0, n_distinct=100_000),
        keys=[],
        values=[ColSpec("value", KIND_UNIFORM_INT, col=1, elem_bytes=8, lo=1, hi=1_000_000)],
        aggs=[(AGG_COUNT, -1), (AGG_SUM_I64, 0)],
        description="Ungrouped PAC COUNT(*) and SUM(value): 1e6 rows; pu uniform over 1e5; "
                    "value int64 U[1,1e6]"),
    "C2": Workload(
        name="C2", n_rows=60_000_000, seed=_seed(2),
        pu=ColSpec("pu_key", KIND_UNIFORM_KEY64, col=0, n_distinct=1_500_000),
        keys=[ColSpec("g1", KIND_UNIFORM_INT, col=1, elem_bytes=1, lo=0, hi=2),
              ColSpec("g2", KIND_UNIFORM_INT, col=2, elem_bytes=1, lo=0, hi=1)],
        values=[ColSpec("cents", KIND_UNIFORM_INT, col=3, elem_bytes=8, lo=100, hi=10_000_000),
                ColSpec("disc", KIND_UNIFORM_F64, col=4, lo=0.0, hi=0.1)],
        aggs=[(AGG_SUM_I64, 0), (AGG_AVG_F64, 1), (AGG_COUNT, -1)],
        description="Low-cardinality grouped: 6e7 rows; 2 int8 keys (3x2); pu uniform over 1.5e6; "
                    "SUM int64 cents U[100,1e7], AVG f64 U[0,0.1), COUNT"),
    "C3": Workload(
        name="C3", n_rows=100_000_000, seed=_seed(3),
        pu=ColSpec("pu_key", KIND_ZIPF_KEY64, col=0, n_distinct=10_000_000, zipf_s=0.8),
        keys=[ColSpec("g", KIND_ZIPF_KEY32, col=1, n_distinct=1_000_000, zipf_s=1.1)],
        values=[ColSpec("value", KIND_UNIFORM_INT, col=2, elem_bytes=8, lo=1, hi=1_000_000)],
        aggs=[(AGG_SUM_I64, 0), (AGG_COUNT, -1)],
        description="High-cardinality grouped: 1e8 rows; int32 Zipf(1.1) over 1e6 groups; "
                    "pu Zipf(0.8) over 1e7; SUM int64 U[1,1e6], COUNT"),
    "C4": Workload(
        name="C4", n_rows=200_000_000, seed=_seed(4),
        pu=ColSpec("pu_key", KIND_UNIFORM_KEY64, col=0, n_distinct=20_000_000),
        keys=[ColSpec("g", KIND_UNIFORM_INT, col=1, elem_bytes=4, lo=0, hi=999)],
        values=[ColSpec("value", KIND_NORMAL_F64, col=2, lo=1000.0, hi=250.0)],
        aggs=[(AGG_MIN_F64, 0), (AGG_MAX_F64, 0)],
        description="PAC MIN/MAX: 2e8 rows; 1000 int32 groups; pu uniform over 2e7; "
                    "value f64 Normal(1000,250)"),
    "C5": Workload(
        name="C5", n_rows=1_200_000_000, seed=_seed(5),
        pu=ColSpec("pu_key", KIND_UNIFORM_KEY64, col=0, n_distinct=150_000_000),
        keys=[ColSpec("g", KIND_UNIFORM_INT, col=1, elem_bytes=4, lo=0, hi=99)],
        values=[ColSpec("s", KIND_UNIFORM_INT, col=2, elem_bytes=8, lo=1, hi=1_000_000),
                ColSpec("a", KIND_UNIFORM_F64, col=4, lo=0.0, hi=1.0)],
        aggs=[(AGG_SUM_I64, 0), (AGG_COUNT, -1), (AGG_AVG_F64, 1)],
        rounds=20,
        description="Multi-GPU sharded: 1.2e9 rows; 100 int32 groups; pu uniform over 1.5e8; "
                    "SUM int64 U[1,1e6], COUNT, AVG f64 U[0,1); d=20 finalize rounds"),
}


# ---------------------------------------------------------------- device side

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libdatagen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(_LIB_PATH)
        lib.dg_fill.restype = ctypes.c_int
        lib.dg_fill.argtypes = [
            ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double, ctypes.c_double,
            ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        _lib = lib
    return _lib


def device_column(spec: ColSpec, seed: int, row0: int, n: int, device="cuda", cdf_cache=None):
    """Generate the same column on the GPU (torch tensor).  Integers and uniform
    doubles are bit-identical to gen_column; normals agree to ~1 ulp."""
    import torch
    lib = _load()
    out = torch.empty(n, dtype=getattr(torch, np.dtype(spec.dtype).name), device=device)
    cdf_ptr = None
    if spec.kind in (KIND_ZIPF_KEY32, KIND_ZIPF_KEY64):
        key = (spec.n_distinct, spec.zipf_s)
        cache = cdf_cache if cdf_cache is not None else _dev_cdf_cache
        if key not in cache:
            cache[key] = torch.from_numpy(cdf_for(spec)).to(device)
        cdf_ptr = cache[key].data_ptr()
    stream = torch.cuda.current_stream(out.device).cuda_stream
    rc = lib.dg_fill(spec.kind, out.data_ptr(), spec.elem_bytes, n, row0,
                     seed & 0xFFFFFFFFFFFFFFFF, spec.col, float(spec.lo), float(spec.hi),
                     spec.n_distinct, cdf_ptr, ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"dg_fill failed rc={rc}")
    return out


_dev_cdf_cache: Dict[tuple, object] = {}


def device_columns(w: Workload, row0: int = 0, n: Optional[int] = None, device="cuda") -> dict:
    n = w.n_rows if n is None else n
    return {
        "pu": device_column(w.pu, w.seed, row0, n, device),
        "keys": [device_column(k, w.seed, row0, n, device) for k in w.keys],
        "values": [device_column(v, w.seed, row0, n, device) for v in w.values],
    }
