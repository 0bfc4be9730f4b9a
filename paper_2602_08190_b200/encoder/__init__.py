"""CPU cascade encoder (native, cdm_encode.c): plain columns -> self-contained CDM1 chunks.

The paper's offline CPU compression side.  An input producer for the decode hot
path; it shares no code with the CUDA kernels or the oracle.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .. import _native
from ..inputs import Column, VARBYTES


def _lib():
    lib = _native.load("libcdm_enc.so", _native.build_enc)
    if not getattr(lib, "_typed", False):
        lib.cdm_encode.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p),
                                   ctypes.POINTER(ctypes.c_size_t)]
        lib.cdm_encode_error.restype = ctypes.c_char_p
        lib.cdm_encode_free.argtypes = [ctypes.c_void_p]
        lib.cdm_encode_canonical.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t]
        lib._typed = True
    return lib


class EncodeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"encode error {code}: {msg}")
        self.code = code


def canonical(cascade: str) -> str:
    lib = _lib()
    buf = ctypes.create_string_buffer(1024)
    rc = lib.cdm_encode_canonical(cascade.encode(), buf, 1024)
    if rc:
        raise EncodeError(rc, lib.cdm_encode_error().decode())
    return buf.value.decode()


def encode_raw(cascade: str, dtype: int, width: int, data: np.ndarray, rows: int,
               offsets: np.ndarray | None = None, chunk_id: int = 0) -> np.ndarray:
    lib = _lib()
    data = np.ascontiguousarray(data)
    if offsets is not None:
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    buf = ctypes.c_void_p()
    ln = ctypes.c_size_t()
    rc = lib.cdm_encode(cascade.encode(), dtype, width, data.ctypes.data if data.size else None,
                        offsets.ctypes.data if offsets is not None else None, rows, chunk_id,
                        ctypes.byref(buf), ctypes.byref(ln))
    if rc:
        raise EncodeError(rc, lib.cdm_encode_error().decode())
    try:
        out = np.empty(ln.value, dtype=np.uint8)
        ctypes.memmove(out.ctypes.data, buf.value, ln.value)
    finally:
        lib.cdm_encode_free(buf)
    return out


def encode(cascade: str, col: Column, chunk_id: int = 0) -> np.ndarray:
    """Encode a whole Column into one chunk (uint8 numpy array)."""
    return encode_raw(cascade, col.dtype, col.width, col.data, col.rows, col.offsets, chunk_id)


def encode_chunks(cascade: str, col: Column, rows_per_chunk: int, first_chunk_id: int = 0) -> list[np.ndarray]:
    """Split a column into row groups of rows_per_chunk rows (last one ragged), one self-contained chunk each."""
    chunks = []
    n = col.rows
    k = 0
    for r0 in range(0, max(n, 1), rows_per_chunk):
        r1 = min(n, r0 + rows_per_chunk)
        if col.dtype == VARBYTES:
            offs = col.offsets[r0:r1 + 1]
            data = col.data
            chunks.append(encode_raw(cascade, col.dtype, col.width, data, r1 - r0, offs, first_chunk_id + k))
        else:
            chunks.append(encode_raw(cascade, col.dtype, col.width, col.data[r0:r1], r1 - r0, None,
                                     first_chunk_id + k))
        k += 1
    return chunks
