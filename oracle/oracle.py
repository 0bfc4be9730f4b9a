"""ctypes binding of the plain-C oracle decoder (cdm_oracle.c).  TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libcdm_oracle.so")
SRC = os.path.join(HERE, "cdm_oracle.c")
_lock = threading.Lock()
_lib = None


class OracleResult(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_uint64), ("payload_bytes", ctypes.c_uint64), ("offsets_bytes", ctypes.c_uint64),
                ("chunk_id", ctypes.c_uint64), ("status", ctypes.c_int32), ("detail", ctypes.c_char * 200)]


class OracleError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"oracle status {status}: {detail}")
        self.status = status
        self.detail = detail


def build(force: bool = False) -> str:
    """gcc -O2 the oracle (plain scalar C, no SIMD intrinsics) into oracle/_build/."""
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or not os.path.exists(LIB) or os.path.getmtime(SRC) > os.path.getmtime(LIB):
        r = subprocess.run(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fvisibility=hidden", "-o", LIB, SRC,
                            "-lpthread"], capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stdout + r.stderr)
    return LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            try:
                build()
            except (OSError, RuntimeError):
                if not os.path.exists(LIB):
                    raise
            lib = ctypes.CDLL(LIB)
            lib.oracle_decode_chunk.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                                ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(OracleResult)]
            lib.oracle_decode_many.argtypes = [ctypes.c_void_p] * 7 + [ctypes.c_size_t, ctypes.c_int]
            lib.oracle_checksum.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64]
            lib.oracle_checksum.restype = ctypes.c_uint64
            _lib = lib
        return _lib


def _header(chunk: np.ndarray):
    h = chunk[:64].tobytes()
    dtype = h[10]
    width = int.from_bytes(h[12:16], "little")
    rows = int.from_bytes(h[16:24], "little")
    payload = int.from_bytes(h[24:32], "little")
    return dtype, width, rows, payload


def decode_chunk(chunk: np.ndarray):
    """Decode one chunk.  Returns (payload uint8 array, offsets int32 array or None).  Raises OracleError."""
    lib = _load()
    chunk = np.ascontiguousarray(chunk, dtype=np.uint8)
    if chunk.size < 64:
        res = OracleResult()
        rc = lib.oracle_decode_chunk(chunk.ctypes.data if chunk.size else None, chunk.size, None, 0, None, 0,
                                     ctypes.byref(res))
        raise OracleError(rc, res.detail.decode(errors="replace"))
    dtype, width, rows, payload = _header(chunk)
    cap = payload if payload < (1 << 31) else 0
    out = np.empty(max(cap, 1), dtype=np.uint8)
    offs = np.empty(rows + 1 if dtype == 4 and rows < (1 << 27) else 1, dtype=np.int32)
    res = OracleResult()
    rc = lib.oracle_decode_chunk(chunk.ctypes.data, chunk.size, out.ctypes.data, cap, offs.ctypes.data, offs.size,
                                 ctypes.byref(res))
    if rc:
        raise OracleError(rc, res.detail.decode(errors="replace"))
    return out[:payload], (offs if dtype == 4 else None)


def decode_many(chunks: list[np.ndarray], nthreads: int = 1):
    """Chunk-parallel oracle (each chunk decoded by the plain routine).  Returns list of (payload, offsets)."""
    lib = _load()
    n = len(chunks)
    chunks = [np.ascontiguousarray(c, dtype=np.uint8) for c in chunks]
    outs, offs = [], []
    for c in chunks:
        dtype, width, rows, payload = _header(c)
        outs.append(np.empty(max(payload, 1), dtype=np.uint8))
        offs.append(np.empty(rows + 1 if dtype == 4 else 1, dtype=np.int32))
    P = ctypes.c_void_p * n
    S = ctypes.c_size_t * n
    res = (OracleResult * n)()
    rc = lib.oracle_decode_many(P(*[c.ctypes.data for c in chunks]), S(*[c.size for c in chunks]),
                                P(*[o.ctypes.data for o in outs]), S(*[o.size for o in outs]),
                                P(*[o.ctypes.data for o in offs]), S(*[o.size for o in offs]), res, n, nthreads)
    if rc:
        bad = next(i for i in range(n) if res[i].status)
        raise OracleError(res[bad].status, f"chunk {bad}: " + res[bad].detail.decode(errors="replace"))
    result = []
    for i, c in enumerate(chunks):
        dtype, width, rows, payload = _header(c)
        result.append((outs[i][:payload], offs[i] if dtype == 4 else None))
    return result


def checksum(data: np.ndarray, chunk_id: int) -> int:
    """SURVEY Sec. 8a H9 positional checksum of a decoded buffer (see cdm_oracle.c)."""
    lib = _load()
    data = np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    return int(lib.oracle_checksum(data.ctypes.data if data.size else None, data.size, chunk_id))
