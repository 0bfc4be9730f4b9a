"""Workload builder for the benchmark configurations (INPUT PRODUCTION ONLY -- no decode arithmetic here).

Generates the seeded TPC-H-like columns (inputs/) chunk by chunk and encodes every chunk (encoder/) in
parallel worker processes, straight into ONE shared host buffer that is later page-locked in place
(cudaHostRegister) -- the column store of compressed row groups the paper keeps in CPU memory
(SF=100 per PAPER.md:344 is ~21.5 GB of compressed chunks).

* Chunk c of column k holds rows [c*R, min((c+1)*R, rows)) and has the global chunk id k*10000 + c, so
  its bytes do not depend on how the chunks are split over ranks or workers (the union of
  rank outputs equals the 1-GPU output).
* Workers are forked after the generator context is built (its per-order line prefix is shared
  copy-on-write); each reserves its chunk's space in the shared buffer with an atomic bump counter.
* Phase 1 encodes chunk 0 of every column to measure compressed bytes per row; the buffer is sized from
  that (x 1.15 + alignment), phase 2 encodes the rest.
"""
from __future__ import annotations

import mmap
import multiprocessing as mp
import os
import struct
from dataclasses import dataclass, field

import numpy as np

ALIGN = 256
_G = None        # generator context (forked into the workers)
_BUF = None      # shared mmap
_CTR = None      # shared bump counter
_COLS = None     # [(name, spec)]
_ROWS = None     # chunk rows
_CAP = 0


@dataclass
class ChunkRef:
    column: int        # index into Dataset.columns
    index: int         # chunk index within the column (row order)
    chunk_id: int
    offset: int        # byte offset in Dataset.buf
    size: int          # compressed bytes (what crosses PCIe)
    rows: int
    payload: int       # decoded payload bytes
    offsets: int       # decoded offsets bytes (VARBYTES), else 0
    plain: int         # plain bytes of the rows (generator output)

    @property
    def decoded(self) -> int:
        return self.payload + self.offsets


@dataclass
class Dataset:
    buf: object                     # mmap (shared, later page-locked) or bytearray-like
    used: int
    columns: list                   # [(name, spec, dtype, width)]
    chunks: list = field(default_factory=list)
    sf: float = 0.0
    seed: int = 0
    build_s: float = 0.0
    workers: int = 1

    def array(self) -> np.ndarray:
        if isinstance(self.buf, np.ndarray):
            return self.buf[: self.used]
        return np.frombuffer(self.buf, dtype=np.uint8, count=self.used)

    def rebind(self, arr: np.ndarray) -> None:
        """Move the column store to another buffer holding the same bytes (e.g. page-locked memory); the
        shared worker mapping is released."""
        old = self.buf
        self.buf = arr
        if isinstance(old, mmap.mmap):
            try:
                old.close()
            except BufferError:  # still exported somewhere: left to the garbage collector
                pass

    def host(self, ch: ChunkRef) -> np.ndarray:
        if isinstance(self.buf, np.ndarray):
            return self.buf[ch.offset: ch.offset + ch.size]
        return np.frombuffer(self.buf, dtype=np.uint8, count=ch.size, offset=ch.offset)

    @property
    def compressed(self) -> int:
        return sum(c.size for c in self.chunks)

    @property
    def decoded(self) -> int:
        return sum(c.decoded for c in self.chunks)


def chunk_id_of(column: int, index: int) -> int:
    return column * 10000 + index


def _header(buf: np.ndarray):
    rows, payload, offsets = struct.unpack_from("<QQQ", buf, 16)
    return int(rows), int(payload), int(offsets)


def _encode(job):
    """(column index, chunk index) -> encoded chunk bytes + metadata (numpy array), in a worker."""
    from . import encoder
    k, c = job
    name, spec = _COLS[k]
    total = _row_count(_G, name)
    r0 = c * _ROWS
    r1 = min(total, r0 + _ROWS)
    if name == "config1":  # BASELINE configs[0]: the 1M-row int32 FOR + 8-bit column (one chunk)
        from .inputs import Column, config1_column
        full = config1_column()
        col = Column(full.name, full.dtype, full.width, r1 - r0, full.data[r0:r1])
    else:
        col = _G.column(name, r0, r1 - r0)
    enc = encoder.encode(spec, col, chunk_id=chunk_id_of(k, c))
    return enc, col.nbytes()


def _encode_into(job):
    enc, plain = _encode(job)
    size = int(enc.size)
    with _CTR.get_lock():
        off = _CTR.value
        _CTR.value = off + (size + ALIGN - 1) // ALIGN * ALIGN
    if off + size > _CAP:
        return job, -1, enc, plain  # overflow: the parent places it
    np.frombuffer(_BUF, dtype=np.uint8, count=size, offset=off)[:] = enc
    rows, payload, offsets = _header(enc)
    return job, off, (size, rows, payload, offsets), plain


def _row_count(g, name: str) -> int:
    if name == "config1":
        return 1_000_000
    return g.rows(0 if name.startswith("l_") else 2 if name.startswith("ps_") else 1)


def build(columns, sf: float, seed: int, chunk_rows: int = 1 << 22, select=None, workers: int | None = None,
          column_types=None) -> Dataset:
    """Generate + encode `columns` [(name, spec)] at scale factor sf.

    select: optional {column index: list of chunk indices} (a rank's shard); default every chunk.
    Returns a Dataset whose chunks are ordered by (column, chunk index)."""
    import time
    global _G, _BUF, _CTR, _COLS, _ROWS, _CAP
    from .inputs import COLUMN_TYPES, TPCH
    t0 = time.perf_counter()
    workers = max(1, workers or os.cpu_count() or 1)
    _G = TPCH(sf, seed)
    _COLS = list(columns)
    _ROWS = chunk_rows
    jobs = []
    for k, (name, _) in enumerate(_COLS):
        n = _row_count(_G, name)
        nch = max(1, -(-n // chunk_rows))
        idx = range(nch) if select is None else select.get(k, [])
        jobs += [(k, c) for c in idx]
    ctx = mp.get_context("fork")
    first = {}
    for j in jobs:
        first.setdefault(j[0], j)
    probe_jobs = list(first.values())
    # phase 1: one chunk per column (also measures bytes per row)
    with ctx.Pool(min(workers, max(1, len(probe_jobs)))) as pool:
        probe = dict(zip(probe_jobs, pool.map(_encode, probe_jobs)))
    est = 0
    for (k, c) in jobs:
        enc, _ = probe[first[k]]
        rows_probe = _header(enc)[0] or 1
        name = _COLS[k][0]
        rows = min(chunk_rows, _row_count(_G, name) - c * chunk_rows)
        est += int(enc.size / rows_probe * max(rows, 1) * 1.15) + 2 * ALIGN + 4096
    _CAP = max(est, 1 << 20)
    _BUF = mmap.mmap(-1, _CAP, flags=mmap.MAP_SHARED | mmap.MAP_ANONYMOUS)
    _CTR = ctx.Value("Q", 0)
    results = {}
    overflow = []

    def place(job, off, meta, plain):
        if off < 0:
            overflow.append((job, meta, plain))
        else:
            results[job] = (off, meta, plain)

    # probe chunks first (already encoded), then the rest in parallel, heaviest columns first
    for job in probe_jobs:
        enc, plain = probe[job]
        size = int(enc.size)
        off = _CTR.value
        _CTR.value = off + (size + ALIGN - 1) // ALIGN * ALIGN
        if off + size > _CAP:
            place(job, -1, enc, plain)
        else:
            np.frombuffer(_BUF, dtype=np.uint8, count=size, offset=off)[:] = enc
            place(job, off, (size,) + _header(enc), plain)
    rest = [j for j in jobs if j not in probe]
    weight = {k: probe[first[k]][0].size for k in first}
    rest.sort(key=lambda j: -weight[j[0]])
    if rest:
        with ctx.Pool(workers) as pool:
            for job, off, meta, plain in pool.imap_unordered(_encode_into, rest, chunksize=1):
                place(job, off, meta, plain)
    used = int(_CTR.value)
    if overflow:  # the estimate was short: grow the buffer and append (rare)
        extra = sum((int(e.size) + ALIGN - 1) // ALIGN * ALIGN for _, e, _ in overflow)
        nb = mmap.mmap(-1, min(used, _CAP) + extra + ALIGN, flags=mmap.MAP_SHARED | mmap.MAP_ANONYMOUS)
        nb[: min(used, _CAP)] = _BUF[: min(used, _CAP)]
        _BUF.close()
        _BUF = nb
        pos = min(used, _CAP)
        pos = (pos + ALIGN - 1) // ALIGN * ALIGN
        for job, enc, plain in overflow:
            size = int(enc.size)
            np.frombuffer(_BUF, dtype=np.uint8, count=size, offset=pos)[:] = enc
            results[job] = (pos, (size,) + _header(enc), plain)
            pos += (size + ALIGN - 1) // ALIGN * ALIGN
        used = pos
    else:
        used = max((off + meta[0] for off, meta, _ in results.values()), default=0)
    types = dict(column_types or COLUMN_TYPES)
    types.setdefault("config1", (0, 4))
    ds = Dataset(buf=_BUF, used=used, columns=[(n, s) + tuple(types[n]) for n, s in _COLS], sf=sf, seed=seed,
                 workers=workers)
    for (k, c) in sorted(results):
        off, (size, rows, payload, offsets), plain = results[(k, c)]
        ds.chunks.append(ChunkRef(k, c, chunk_id_of(k, c), off, size, rows, payload, offsets, plain))
    ds.build_s = time.perf_counter() - t0
    _G = None
    return ds


def sample_chunks(columns, sf: float, seed: int, chunk_rows: int = 1 << 22, per_column: int = 1):
    """The oracle's bounded sample: the first `per_column` chunks of every column, encoded exactly as in
    build() (same chunk ids), returned as [(column index, chunk index, numpy bytes)] -- cheap to produce
    without building the whole dataset (for --impl reference and the cpu_baseline)."""
    global _G, _COLS, _ROWS
    from .inputs import TPCH
    _G = TPCH(sf, seed)
    _COLS = list(columns)
    _ROWS = chunk_rows
    jobs = []
    for k, (name, _) in enumerate(_COLS):
        nch = max(1, -(-_row_count(_G, name) // chunk_rows))
        jobs += [(k, c) for c in range(min(per_column, nch))]
    with mp.get_context("fork").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        encs = pool.map(_encode, jobs)
    _G = None
    return [(k, c, e) for (k, c), (e, _) in zip(jobs, encs)]
