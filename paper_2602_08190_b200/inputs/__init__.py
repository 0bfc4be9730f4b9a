"""Seeded synthetic inputs (INPUT GENERATORS ONLY -- none of the decode method's arithmetic lives here).

Two families, both deterministic in their seed and shared by the CUDA path's tests/bench and the oracle's
tests:

* dbgen-like TPC-H lineitem / orders / partsupp columns from the native counter-based generator (tpch_gen.c);
  any row range of any column is generated independently.
* microbenchmark columns shaped like the paper's experiments: the config-1 int32 column, uniform
  w-bit columns (Fig. `bitcompVSnvcomp`), RLE group-size distributions even-X,
  random[L,R], outlier, mixed (Fig. `rleVSnvcomp`).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .. import _native

LINEITEM, ORDERS, PARTSUPP = 0, 1, 2

LINEITEM_COLS = ["l_orderkey", "l_partkey", "l_suppkey", "l_linenumber", "l_quantity", "l_extendedprice",
                 "l_discount", "l_tax", "l_returnflag", "l_linestatus", "l_shipdate", "l_commitdate",
                 "l_receiptdate", "l_shipinstruct", "l_shipmode", "l_comment"]
ORDERS_COLS = ["o_orderkey", "o_custkey", "o_orderstatus", "o_totalprice", "o_orderdate", "o_orderpriority",
               "o_clerk", "o_shippriority", "o_comment"]
PARTSUPP_COLS = ["ps_partkey", "ps_suppkey", "ps_availqty", "ps_supplycost", "ps_comment"]

# dtype tags of the CDM1 container / C-ABI: 0 I32, 1 I64, 2 F64, 3 FIXED, 4 VARBYTES
I32, I64, F64, FIXED, VARBYTES = 0, 1, 2, 3, 4

# column -> (dtype, width)  [decoded types: SURVEY §8d "Decoded types"]
COLUMN_TYPES = {
    "l_orderkey": (I64, 8), "l_partkey": (I32, 4), "l_suppkey": (I32, 4), "l_linenumber": (I32, 4),
    "l_quantity": (F64, 8), "l_extendedprice": (F64, 8), "l_discount": (F64, 8), "l_tax": (F64, 8),
    "l_returnflag": (FIXED, 1), "l_linestatus": (FIXED, 1), "l_shipdate": (I32, 4), "l_commitdate": (I32, 4),
    "l_receiptdate": (I32, 4), "l_shipinstruct": (FIXED, 25), "l_shipmode": (FIXED, 10),
    "l_comment": (VARBYTES, 1),
    "o_orderkey": (I64, 8), "o_custkey": (I32, 4), "o_orderstatus": (FIXED, 1), "o_totalprice": (F64, 8),
    "o_orderdate": (I32, 4), "o_orderpriority": (FIXED, 15), "o_clerk": (FIXED, 15),
    "o_shippriority": (I32, 4), "o_comment": (VARBYTES, 1),
    "ps_partkey": (I32, 4), "ps_suppkey": (I32, 4), "ps_availqty": (I32, 4), "ps_supplycost": (F64, 8),
    "ps_comment": (VARBYTES, 1),
}

NP_DTYPE = {I32: np.int32, I64: np.int64, F64: np.float64}

MASTER_SEED = 20260217


def _lib():
    lib = _native.load("libcdm_gen.so", _native.build_gen)
    if not getattr(lib, "_typed", False):
        lib.gen_create.restype = ctypes.c_void_p
        lib.gen_create.argtypes = [ctypes.c_double, ctypes.c_uint64]
        lib.gen_destroy.argtypes = [ctypes.c_void_p]
        lib.gen_rows.restype = ctypes.c_uint64
        lib.gen_rows.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.gen_fixed.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_void_p]
        lib.gen_varbytes.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]
        lib._typed = True
    return lib


@dataclass
class Column:
    """A plain column: data (numpy, rows*width bytes or typed), offsets (rows+1 int64) for VARBYTES."""
    name: str
    dtype: int
    width: int
    rows: int
    data: np.ndarray
    offsets: np.ndarray | None = None

    def nbytes(self) -> int:
        return int(self.data.nbytes) + (4 * (self.rows + 1) if self.offsets is not None else 0)


class TPCH:
    """dbgen-like TPC-H generator (native, counter-based).  TPCH(sf).column(name, row0, rows)."""

    def __init__(self, sf: float, seed: int = MASTER_SEED):
        self.sf = sf
        self.seed = seed
        self._lib = _lib()
        self._h = self._lib.gen_create(float(sf), int(seed))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.gen_destroy(h)
            self._h = None

    def rows(self, table: int) -> int:
        return int(self._lib.gen_rows(self._h, table))

    def column(self, name: str, row0: int = 0, rows: int | None = None) -> Column:
        if name in LINEITEM_COLS:
            table, col = LINEITEM, LINEITEM_COLS.index(name)
        elif name in ORDERS_COLS:
            table, col = ORDERS, ORDERS_COLS.index(name)
        elif name in PARTSUPP_COLS:
            table, col = PARTSUPP, PARTSUPP_COLS.index(name)
        else:
            raise KeyError(name)
        total = self.rows(table)
        if rows is None:
            rows = total - row0
        if row0 < 0 or rows < 0 or row0 + rows > total:
            raise ValueError("row range out of bounds")
        dtype, width = COLUMN_TYPES[name]
        if dtype == VARBYTES:
            offs = np.empty(rows + 1, dtype=np.int64)
            payload = ctypes.c_uint64(0)
            rc = self._lib.gen_varbytes(self._h, table, col, row0, rows, offs.ctypes.data, None, ctypes.byref(payload))
            if rc:
                raise RuntimeError("generator failed")
            data = np.empty(int(payload.value), dtype=np.uint8)
            rc = self._lib.gen_varbytes(self._h, table, col, row0, rows, offs.ctypes.data, data.ctypes.data,
                                        ctypes.byref(payload))
            if rc:
                raise RuntimeError("generator failed")
            return Column(name, dtype, width, rows, data, offs)
        if dtype in NP_DTYPE:
            data = np.empty(rows, dtype=NP_DTYPE[dtype])
        else:
            data = np.empty((rows, width), dtype=np.uint8)
        rc = self._lib.gen_fixed(self._h, table, col, row0, rows, data.ctypes.data)
        if rc:
            raise RuntimeError("generator failed")
        return Column(name, dtype, width, rows, data)


# ---------------------------------------------------------------- microbenchmark shapes (numpy, seeded)

def config1_column(n: int = 1_000_000, seed: int = 1) -> Column:
    """Config 1: int32 x = 1,000,000,007 + U[0,255], x[0] = min, x[1] = min+255 (forces w = 8)."""
    rng = np.random.default_rng(seed)
    x = (1_000_000_007 + rng.integers(0, 256, size=n, dtype=np.int64)).astype(np.int32)
    if n > 0:
        x[0] = 1_000_000_007
    if n > 1:
        x[1] = 1_000_000_007 + 255
    return Column("config1", I32, 4, n, x)


def uniform_bits_column(n: int, w: int, dtype: int = I64, seed: int = 2) -> Column:
    """Uniform w-bit values ('uniformly sampling int64 values' per bit width)."""
    rng = np.random.default_rng(seed + w)
    if w == 0:
        v = np.full(n, 12345, dtype=np.uint64)
    else:
        v = rng.integers(0, 1 << 62, size=n, dtype=np.uint64, endpoint=True) * np.uint64(4)
        v ^= rng.integers(0, 4, size=n, dtype=np.uint64)
        if w < 64:
            v &= np.uint64((1 << w) - 1)
        if n > 1:
            v[0] = 0
            v[1] = np.uint64((1 << w) - 1) if w < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    if dtype == I32:
        return Column(f"uniform{w}", I32, 4, n, v.astype(np.uint32).view(np.int32))
    return Column(f"uniform{w}", I64, 8, n, v.view(np.int64))


def rle_counts(dist: str, n: int, seed: int = 3) -> np.ndarray:
    """Group sizes summing to n for PAPER.md:384-387's distributions:
    'even-X', 'random-L-R', 'outlier-X-P' (mostly 1, fraction P% of size X), 'mixed-A+B' (concatenation)."""
    rng = np.random.default_rng(seed)
    if dist.startswith("mixed-"):
        a, b = dist[len("mixed-"):].split("+")
        half = n // 2
        return np.concatenate([rle_counts(a, half, seed + 1), rle_counts(b, n - half, seed + 2)])
    parts = dist.split("-")
    kind = parts[0]
    if kind == "even":
        x = int(parts[1])
        c = np.full(n // x, x, dtype=np.int64)
    elif kind == "random":
        lo, hi = int(parts[1]), int(parts[2])
        c = rng.integers(lo, hi + 1, size=n // max(1, (lo + hi) // 2) + 2, dtype=np.int64)
    elif kind == "outlier":
        x, pct = int(parts[1]), float(parts[2])
        m = n // 2 + 2
        c = np.where(rng.random(m) < pct / 100.0, x, 1).astype(np.int64)
    elif kind == "single":
        c = np.array([n], dtype=np.int64)
    else:
        raise ValueError(dist)
    cs = np.cumsum(c)
    k = int(np.searchsorted(cs, n, side="left"))
    c = c[: k + 1].copy() if k < len(c) else c.copy()
    tot = int(c.sum())
    if tot > n:
        c[-1] -= tot - n
    elif tot < n:
        c = np.append(c, n - tot)
    return c[c > 0]


def rle_column(dist: str, n: int, dtype: int = I64, seed: int = 4) -> Column:
    """A column whose maximal runs follow rle_counts(dist): adjacent run values always differ."""
    counts = rle_counts(dist, n, seed)
    rng = np.random.default_rng(seed + 7)
    vals = np.cumsum(rng.integers(1, 1000, size=len(counts), dtype=np.int64))  # strictly increasing => distinct
    col = np.repeat(vals, counts)
    if dtype == I32:
        return Column(f"rle:{dist}", I32, 4, n, col.astype(np.int32))
    return Column(f"rle:{dist}", I64, 8, n, col)
