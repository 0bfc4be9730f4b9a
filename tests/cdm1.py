"""Test-local CDM1 container reader/writer (independent of the encoder, the oracle and the CUDA runtime).

Used to (a) hand-assemble chunks from golden stream bytes so the oracle and the GPU path can be pinned
without going through the encoder, and (b) inspect the encoder's streams.  Layout: DESIGN.md
"CDM1 chunk container".
"""
from __future__ import annotations

import struct

import numpy as np

RAW, BITPACK, DICT, FLOAT2INT, DELTA, RLE, LZ4, STR, ANS, DSTRIDE, STRDICT = range(11)
I32, I64, F64, FIXED, VARBYTES = range(5)


def pack_bits(fields, w: int) -> bytes:
    """LSB-first contiguous bit packing by big-integer arithmetic (the plain definition)."""
    acc = 0
    for i, f in enumerate(fields):
        assert 0 <= int(f) < (1 << w) or (w == 0 and int(f) == 0)
        acc |= int(f) << (i * w)
    nbytes = (len(fields) * w + 7) // 8
    return acc.to_bytes(nbytes, "little") if nbytes else b""


class Node:
    def __init__(self, codec, n, children=(), stream=None, eb=0, w=0, base=0, entries=0, E=0, d=0, nruns=0,
                 maxrun=0, nsub=0, sub=0, tl=0, il=0, stride=0):
        self.codec, self.n, self.children, self.stream, self.eb = codec, n, list(children), stream, eb
        self.w, self.base, self.entries, self.E, self.d = w, base, entries, E, d
        self.nruns, self.maxrun, self.nsub, self.sub = nruns, maxrun, nsub, sub
        self.tl, self.il, self.stride = tl, il, stride

    def params(self) -> bytes:
        p = bytearray(16)
        if self.codec == BITPACK:
            p[0] = self.w
            p[8:16] = struct.pack("<Q", self.base & ((1 << 64) - 1))
        elif self.codec == DICT:
            p[0:8] = struct.pack("<II", self.entries, self.E)
        elif self.codec == STRDICT:
            p[0:12] = struct.pack("<III", self.entries, self.E, 32)  # entries, token bytes, max token
        elif self.codec == FLOAT2INT:
            p[0] = self.d
        elif self.codec == DELTA:
            p[8:16] = struct.pack("<Q", self.base & ((1 << 64) - 1))
        elif self.codec in (RLE, DSTRIDE):
            p[0:8] = struct.pack("<II", self.nruns, self.maxrun)
            if self.codec == DSTRIDE:
                p[8:16] = struct.pack("<Q", self.stride & ((1 << 64) - 1))
        elif self.codec in (LZ4, ANS):
            p[0:8] = struct.pack("<II", self.nsub, self.sub)
            if self.codec == ANS:
                p[8] = self.tl
                p[9] = self.il
        return bytes(p)


def raw(data: bytes, eb: int = 1) -> Node:
    assert len(data) % eb == 0
    return Node(RAW, len(data) // eb, stream=bytes(data), eb=eb)


def bitpack(values, w: int, base: int) -> Node:
    fields = [(int(v) - base) & ((1 << 64) - 1) for v in values]
    return Node(BITPACK, len(fields), [raw(pack_bits(fields, w))], w=w, base=base)


def build(root: Node, dtype: int, width: int, rows: int, payload: int | None = None, chunk_id: int = 0,
          cascade_hash: int = 0) -> np.ndarray:
    nodes, streams = [], []

    def walk(nd):
        sid = 0xFFFF
        if nd.codec == RAW:
            sid = len(streams)
            streams.append(nd.stream)
        nodes.append(struct.pack("<BBHIQ", nd.codec, len(nd.children), sid, nd.eb if nd.codec == RAW else 0, nd.n)
                     + nd.params())
        for ch in nd.children:
            walk(ch)

    walk(root)
    if payload is None:
        payload = rows * width
    offs_bytes = 4 * (rows + 1) if dtype == VARBYTES else 0
    hdr = 64 + 32 * len(nodes) + 16 * len(streams)
    hdr = (hdr + 15) & ~15
    pos = hdr
    table = b""
    body = b""
    for s in streams:
        table += struct.pack("<QQ", pos, len(s))
        padded = s + b"\0" * (((len(s) + 15) & ~15) - len(s) + 16)
        body += padded
        pos += len(padded)
    total = pos
    head = struct.pack("<IHHHBBIQQQQQQ", 0x314D4443, 1, len(nodes), len(streams), dtype, 0, width, rows, payload,
                       offs_bytes, total, cascade_hash, chunk_id)
    blob = head + b"".join(nodes) + table
    blob += b"\0" * (hdr - len(blob))
    blob += body
    assert len(blob) == total
    return np.frombuffer(blob, dtype=np.uint8).copy()


def parse(chunk: np.ndarray):
    """Return (header dict, list of node dicts in preorder, list of stream bytes)."""
    b = chunk.tobytes()
    (magic, ver, nn, ns, dtype, _r, width, rows, payload, offs_bytes, total, h, cid) = struct.unpack_from(
        "<IHHHBBIQQQQQQ", b, 0)
    header = dict(magic=magic, version=ver, n_nodes=nn, n_streams=ns, dtype=dtype, width=width, rows=rows,
                  payload=payload, offsets_bytes=offs_bytes, total=total, hash=h, chunk_id=cid)
    nodes = []
    for i in range(nn):
        codec, nch, sid, eb, n = struct.unpack_from("<BBHIQ", b, 64 + 32 * i)
        p = b[64 + 32 * i + 16: 64 + 32 * i + 32]
        nodes.append(dict(codec=codec, nch=nch, stream=sid, eb=eb, n=n, w=p[0],
                          base=struct.unpack_from("<q", p, 8)[0], u32=struct.unpack_from("<II", p, 0), d=p[0]))
    streams = []
    for i in range(ns):
        off, ln = struct.unpack_from("<QQ", b, 64 + 32 * nn + 16 * i)
        streams.append(b[off:off + ln])
    return header, nodes, streams
