"""Thin Python binding of libcdm (include/cdm.h): argument marshalling only.

Every step of the decode path runs in libcdm's sm_100a kernels; this module converts numpy / torch
buffers to pointers and C structs.  PyTorch supplies device memory and streams.  There is no fallback:
if libcdm.so is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native

I32, I64, F64, FIXED, VARBYTES = 0, 1, 2, 3, 4
STATUS = {0: "CDM_OK", 1: "CDM_E_INVALID_ARG", 2: "CDM_E_PARSE", 3: "CDM_E_UNSUPPORTED", 4: "CDM_E_CORRUPT",
          5: "CDM_E_CAPACITY", 6: "CDM_E_CUDA", 7: "CDM_E_OOM", 8: "CDM_E_BUSY"}
ERR_DICT_INDEX, ERR_RUN_SUM, ERR_LZ4, ERR_LENGTHS, ERR_WIDTH = 0x1, 0x2, 0x4, 0x8, 0x10
FAMILIES = ["fp", "scan", "rle", "lz4", "copy"]
KERNELS = ["fp_kernel", "scan_kernel", "rle_sums_kernel", "rle_kernel(level0)", "rle_kernel", "rle_big_kernel",
           "lz4_kernel", "device_copy", "ans_kernel", "strdict_kernel", "fp_kernel(char)"]
# cdm_batch_kernel_times slots (include/cdm.h): the ANS slot times ans_warp_kernel (il = 32) and ans_kernel
# (il = 1); "rle_kernel" carries the algorithmic bytes of the whole RLE chain

SYMBOLS = ["cdm_status_str", "cdm_last_error", "cdm_version", "cdm_cascade_create", "cdm_cascade_destroy",
           "cdm_cascade_describe", "cdm_chunk_info", "cdm_chunk_check", "cdm_engine_create", "cdm_engine_destroy", "cdm_submit",
           "cdm_submit_batch", "cdm_wait", "cdm_ticket_event", "cdm_engine_launches", "cdm_engine_set_ingest", "cdm_synchronize", "cdm_johnson_order", "cdm_batch_create", "cdm_batch_launch",
           "cdm_batch_results", "cdm_batch_destroy", "cdm_batch_set_timing", "cdm_batch_kernel_ms",
           "cdm_batch_set_graph", "cdm_batch_collect_timing", "cdm_batch_kernel_times", "cdm_batch_kernel_bytes",
           "cdm_pipeline_create", "cdm_pipeline_launch", "cdm_pipeline_results", "cdm_pipeline_destroy",
           "cdm_tune_set", "cdm_tune_get", "cdm_checksum", "cdm_pipeline_info", "cdm_host_register",
           "cdm_host_unregister", "cdm_host_alloc", "cdm_host_free"]


class EngineOpts(ctypes.Structure):
    _fields_ = [("n_slots", ctypes.c_uint32), ("slot_bytes", ctypes.c_uint64), ("copy_stream", ctypes.c_void_p),
                ("decode_stream", ctypes.c_void_p), ("pcie_gbps", ctypes.c_double), ("decode_gbps", ctypes.c_double),
                ("order_policy", ctypes.c_uint32), ("flags", ctypes.c_uint32)]


ENGINE_CHECKSUM = 0x1  # cdm_engine_opts.flags: H9 checksum of every submitted chunk in cdm_result.checksum


class Result(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_uint64), ("payload_bytes", ctypes.c_uint64), ("offsets_bytes", ctypes.c_uint64),
                ("compressed_bytes", ctypes.c_uint64), ("chunk_id", ctypes.c_uint64), ("error_bits", ctypes.c_uint32),
                ("status", ctypes.c_uint32), ("checksum", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Job(ctypes.Structure):
    _fields_ = [("cascade", ctypes.c_void_p), ("host_chunk", ctypes.c_void_p), ("dev_chunk", ctypes.c_void_p),
                ("chunk_bytes", ctypes.c_size_t), ("dev_out", ctypes.c_void_p), ("dev_out_bytes", ctypes.c_size_t),
                ("dev_offsets", ctypes.c_void_p), ("dev_offsets_bytes", ctypes.c_size_t)]


class CdmError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status
        self.detail = detail


_lib = None


def lib():
    """Load libcdm.so (building it if missing/stale; the build is a CPU-only nvcc cross-compile)."""
    global _lib
    if _lib is not None:
        return _lib
    L = _native.load("libcdm.so", _native.build_cdm)
    vp, sz, u32, u64, st = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    L.cdm_status_str.restype = ctypes.c_char_p
    L.cdm_last_error.restype = ctypes.c_char_p
    L.cdm_version.restype = ctypes.c_char_p
    sig = {
        "cdm_cascade_create": [ctypes.c_char_p, st, u32, ctypes.POINTER(vp)],
        "cdm_cascade_destroy": [vp],
        "cdm_cascade_describe": [vp, ctypes.c_char_p, sz],
        "cdm_chunk_info": [vp, sz, ctypes.POINTER(Result)],
        "cdm_chunk_check": [vp, vp, sz],
        "cdm_engine_create": [st, ctypes.POINTER(EngineOpts), ctypes.POINTER(vp)],
        "cdm_engine_destroy": [vp],
        "cdm_submit": [vp, ctypes.POINTER(Job), ctypes.POINTER(u64)],
        "cdm_submit_batch": [vp, ctypes.POINTER(Job), sz, ctypes.POINTER(u64)],
        "cdm_wait": [vp, u64, ctypes.POINTER(Result)],
        "cdm_synchronize": [vp],
        "cdm_ticket_event": [vp, u64, ctypes.POINTER(vp)],
        "cdm_engine_launches": [vp, ctypes.POINTER(u64)],
        "cdm_engine_set_ingest": [vp, ctypes.POINTER(ctypes.c_int), sz],
        "cdm_johnson_order": [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), sz,
                              ctypes.POINTER(sz)],
        "cdm_batch_create": [vp, ctypes.POINTER(Job), sz, ctypes.POINTER(vp)],
        "cdm_batch_launch": [vp, vp, ctypes.POINTER(u32)],
        "cdm_batch_results": [vp, vp, ctypes.POINTER(Result)],
        "cdm_batch_destroy": [vp],
        "cdm_batch_set_timing": [vp, st],
        "cdm_batch_kernel_ms": [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(u64)],
        "cdm_batch_set_graph": [vp, st],
        "cdm_batch_collect_timing": [vp],
        "cdm_batch_kernel_times": [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(u64)],
        "cdm_batch_kernel_bytes": [vp, ctypes.POINTER(u64)],
        "cdm_pipeline_create": [vp, ctypes.POINTER(Job), sz, ctypes.POINTER(vp)],
        "cdm_pipeline_launch": [vp, vp],
        "cdm_pipeline_results": [vp, ctypes.POINTER(Result)],
        "cdm_pipeline_destroy": [vp],
        "cdm_pipeline_info": [vp, ctypes.POINTER(u32), ctypes.POINTER(u32), ctypes.POINTER(u32)],
        "cdm_host_register": [vp, sz],
        "cdm_host_unregister": [vp],
        "cdm_host_alloc": [sz, ctypes.POINTER(vp)],
        "cdm_host_free": [vp],
        "cdm_tune_set": [ctypes.c_char_p, ctypes.c_int],
        "cdm_tune_get": [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int)],
        "cdm_checksum": [vp, ctypes.c_uint64, ctypes.c_uint64, vp, ctypes.POINTER(ctypes.c_uint64)],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = st
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc:
        raise CdmError(rc, lib().cdm_last_error().decode(errors="replace"))


def version() -> str:
    return lib().cdm_version().decode()


def _ptr(x) -> int:
    """Pointer of a numpy array or torch tensor (host or device)."""
    if x is None:
        return 0
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _nbytes(x) -> int:
    if x is None:
        return 0
    if isinstance(x, np.ndarray):
        return x.nbytes
    return x.numel() * x.element_size()


class Cascade:
    """cdm_cascade_create: a column's encoding cascade in Table 2 notation, compiled to a fused plan."""

    def __init__(self, spec: str, dtype: int, width: int = 0):
        h = ctypes.c_void_p()
        _check(lib().cdm_cascade_create(spec.encode(), dtype, width, ctypes.byref(h)))
        self.h = h
        self.spec, self.dtype, self.width = spec, dtype, width

    def describe(self) -> str:
        buf = ctypes.create_string_buffer(1024)
        _check(lib().cdm_cascade_describe(self.h, buf, 1024))
        return buf.value.decode()

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.cdm_cascade_destroy(self.h)
            self.h = None


def checksum(dev_buf, chunk_id: int, stream=None) -> int:
    """H9 positional checksum of a decoded device buffer (include/cdm.h cdm_checksum)."""
    v = ctypes.c_uint64()
    _check(lib().cdm_checksum(_ptr(dev_buf), _nbytes(dev_buf), int(chunk_id), _stream_ptr(stream), ctypes.byref(v)))
    return v.value


def tune_set(knob: str, value: int) -> None:
    """NEXT-3 launch-parameter knob (include/cdm.h: "fp_ctas_per_sm", "lz4_lanes", "lz4_split", "lz4_split_g",
    "lz4_spec", "gp_ctas_per_sm", "scan_mode")."""
    _check(lib().cdm_tune_set(knob.encode(), int(value)))


def tune_get(knob: str) -> int:
    v = ctypes.c_int()
    _check(lib().cdm_tune_get(knob.encode(), ctypes.byref(v)))
    return v.value


def chunk_info(host_chunk) -> dict:
    r = Result()
    _check(lib().cdm_chunk_info(_ptr(host_chunk), _nbytes(host_chunk), ctypes.byref(r)))
    return r.as_dict()


def chunk_check(cascade: Cascade, host_chunk) -> None:
    """Host-only validation of a chunk against a cascade (raises CdmError)."""
    _check(lib().cdm_chunk_check(cascade.h, _ptr(host_chunk), _nbytes(host_chunk)))


def johnson_order(t: list[float], d: list[float]) -> list[int]:
    """cdm_johnson_order: the H3 issue order."""
    n = len(t)
    T = (ctypes.c_double * max(n, 1))(*t)
    D = (ctypes.c_double * max(n, 1))(*d)
    O = (ctypes.c_size_t * max(n, 1))()
    _check(lib().cdm_johnson_order(T, D, n, O))
    return [O[i] for i in range(n)]


@dataclass
class Decode:
    """One chunk to decode: the host bytes (pinned for submit), optional device copy, outputs (torch)."""
    cascade: Cascade
    host_chunk: object
    dev_out: object
    dev_offsets: object = None
    dev_chunk: object = None

    def cjob(self) -> Job:
        # the buffers are held by this object, so their addresses are fixed: marshal once
        key = (self.cascade.h.value, id(self.host_chunk), id(self.dev_chunk), id(self.dev_out), id(self.dev_offsets))
        cj = self.__dict__.get("_cj")
        if cj is None or cj[0] != key:
            cj = (key, Job(self.cascade.h.value, _ptr(self.host_chunk), _ptr(self.dev_chunk), _nbytes(self.host_chunk),
                           _ptr(self.dev_out), _nbytes(self.dev_out), _ptr(self.dev_offsets),
                           _nbytes(self.dev_offsets)))
            self.__dict__["_cj"] = cj
        return cj[1]


class Engine:
    """cdm_engine_create: staging ring + copy/decode streams on one device."""

    def __init__(self, device: int = 0, n_slots: int = 4, slot_bytes: int = 64 << 20, copy_stream=None,
                 decode_stream=None, order_policy: int = 1, pcie_gbps: float = 55.0, decode_gbps: float = 5000.0,
                 checksum: bool = False):
        o = EngineOpts(n_slots, slot_bytes, _stream_ptr(copy_stream), _stream_ptr(decode_stream), pcie_gbps,
                       decode_gbps, order_policy, ENGINE_CHECKSUM if checksum else 0)
        h = ctypes.c_void_p()
        _check(lib().cdm_engine_create(device, ctypes.byref(o), ctypes.byref(h)))
        self.h = h
        self._keep = []
        self._arrays = {}

    def submit(self, d: Decode) -> int:
        t = ctypes.c_uint64()
        j = d.cjob()
        _check(lib().cdm_submit(self.h, ctypes.byref(j), ctypes.byref(t)))
        return t.value

    def submit_batch(self, ds: list[Decode]) -> list[int]:
        n = len(ds)
        cjs = [d.cjob() for d in ds]
        key = tuple(id(j) for j in cjs)
        cached = self._arrays.get(key)
        if cached is None:  # the same list resubmitted (a scan loop) reuses its marshalled job array
            cached = ((Job * n)(*cjs), (ctypes.c_uint64 * n)(), cjs)
            if len(self._arrays) > 64:
                self._arrays.clear()
            self._arrays[key] = cached
        jobs, tickets, _ = cached
        _check(lib().cdm_submit_batch(self.h, jobs, n, tickets))
        return list(tickets)

    def wait(self, ticket: int, raise_on_error: bool = True) -> dict:
        r = Result()
        rc = lib().cdm_wait(self.h, ticket, ctypes.byref(r))
        if rc and (raise_on_error or rc != 4):
            _check(rc)
        return r.as_dict()

    def ticket_event(self, ticket: int) -> int:
        """cdm_ticket_event: the cudaEvent_t (as an int handle) completing with the ticket's decode."""
        ev = ctypes.c_void_p()
        _check(lib().cdm_ticket_event(self.h, ticket, ctypes.byref(ev)))
        return ev.value or 0

    def set_ingest(self, devices: list[int]) -> None:
        """cdm_engine_set_ingest (NEXT-4): copy over these devices' PCIe links, then NVLink into this engine."""
        arr = (ctypes.c_int * max(len(devices), 1))(*devices)
        _check(lib().cdm_engine_set_ingest(self.h, arr, len(devices)))

    def launches(self) -> int:
        """cdm_engine_launches: kernels enqueued through cdm_submit* so far."""
        n = ctypes.c_uint64()
        _check(lib().cdm_engine_launches(self.h, ctypes.byref(n)))
        return n.value

    def synchronize(self) -> None:
        _check(lib().cdm_synchronize(self.h))

    def close(self) -> None:
        if getattr(self, "h", None) and _lib is not None:
            _lib.cdm_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


class Batch:
    """cdm_batch_create/launch/results: decode of chunks already resident in device memory."""

    def __init__(self, engine: Engine, ds: list[Decode]):
        n = len(ds)
        self.n = n
        self._ds = ds
        jobs = (Job * max(n, 1))(*[d.cjob() for d in ds])
        h = ctypes.c_void_p()
        _check(lib().cdm_batch_create(engine.h, jobs, n, ctypes.byref(h)))
        self.h = h

    def launch(self, stream=None) -> int:
        nl = ctypes.c_uint32()
        _check(lib().cdm_batch_launch(self.h, _stream_ptr(stream), ctypes.byref(nl)))
        return nl.value

    def results(self, stream=None, raise_on_error: bool = True) -> list[dict]:
        res = (Result * max(self.n, 1))()
        rc = lib().cdm_batch_results(self.h, _stream_ptr(stream), res)
        if rc and (raise_on_error or rc != 4):
            _check(rc)
        return [res[i].as_dict() for i in range(self.n)]

    def set_timing(self, on) -> None:
        """False/0 off, True/1 per kernel family, 2 per kernel launch."""
        _check(lib().cdm_batch_set_timing(self.h, int(on)))

    def set_graph(self, on: bool) -> None:
        _check(lib().cdm_batch_set_graph(self.h, 1 if on else 0))

    def collect_timing(self) -> None:
        _check(lib().cdm_batch_collect_timing(self.h))

    def kernel_ms(self) -> dict:
        ms = (ctypes.c_double * 5)()
        nl = (ctypes.c_uint64 * 5)()
        _check(lib().cdm_batch_kernel_ms(self.h, ms, nl))
        return {FAMILIES[i]: (ms[i], nl[i]) for i in range(5)}

    def kernel_times(self) -> dict:
        ms = (ctypes.c_double * len(KERNELS))()
        nl = (ctypes.c_uint64 * len(KERNELS))()
        _check(lib().cdm_batch_kernel_times(self.h, ms, nl))
        return {KERNELS[i]: (ms[i], nl[i]) for i in range(len(KERNELS))}

    def kernel_bytes(self) -> dict:
        """Algorithmic bytes (Eq. 1) one launch of the batch moves, per kernel kind."""
        b = (ctypes.c_uint64 * len(KERNELS))()
        _check(lib().cdm_batch_kernel_bytes(self.h, b))
        return {KERNELS[i]: int(b[i]) for i in range(len(KERNELS))}

    def close(self) -> None:
        if getattr(self, "h", None) and _lib is not None:
            _lib.cdm_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


class Pipeline:
    """cdm_pipeline_create/launch/results: the H2D + decode schedule of a fixed job set from PINNED host
    memory, captured once into a CUDA graph; each launch re-copies and re-decodes every job."""

    def __init__(self, engine: Engine, ds: list[Decode]):
        n = len(ds)
        self.n = n
        self._ds = ds
        jobs = (Job * max(n, 1))(*[d.cjob() for d in ds])
        h = ctypes.c_void_p()
        _check(lib().cdm_pipeline_create(engine.h, jobs, n, ctypes.byref(h)))
        self.h = h
        self._res = (Result * max(n, 1))()

    def launch(self, stream=None) -> None:
        _check(lib().cdm_pipeline_launch(self.h, _stream_ptr(stream)))

    def results(self, raise_on_error: bool = True) -> list[dict]:
        rc = lib().cdm_pipeline_results(self.h, self._res)
        if rc and (raise_on_error or rc != 4):
            _check(rc)
        return [self._res[i].as_dict() for i in range(self.n)]

    def info(self) -> dict:
        a, b, c = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        _check(lib().cdm_pipeline_info(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return {"kernel_launches": a.value, "groups": b.value, "h2d_copies": c.value}

    def close(self) -> None:
        if getattr(self, "h", None) and _lib is not None:
            _lib.cdm_pipeline_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def _stream_ptr(s) -> int | None:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream  # torch.cuda.Stream


# --------------------------------------------------------------------------- torch helpers
def output_buffers(host_chunk: np.ndarray, device="cuda"):
    """Allocate (dev_out, dev_offsets) torch buffers for a chunk from its header (16-byte aligned)."""
    import torch
    info = chunk_info(host_chunk)
    out = torch.empty(max(16, (info["payload_bytes"] + 15) // 16 * 16), dtype=torch.uint8, device=device)
    offs = None
    if info["offsets_bytes"]:
        offs = torch.empty(info["offsets_bytes"] // 4, dtype=torch.int32, device=device)
    return out, offs


def host_register(ptr: int, nbytes: int) -> None:
    """cdm_host_register: page-lock a caller-owned host range in place."""
    _check(lib().cdm_host_register(ptr, nbytes))


def host_unregister(ptr: int) -> None:
    _check(lib().cdm_host_unregister(ptr))


class PinnedBuffer:
    """cdm_host_alloc: `nbytes` of page-locked host memory (no size rounding), viewed as a numpy uint8 array."""

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        _check(lib().cdm_host_alloc(max(int(nbytes), 1), ctypes.byref(p)))
        self.ptr = p.value
        self.nbytes = int(nbytes)
        self.array = np.ctypeslib.as_array((ctypes.c_uint8 * max(self.nbytes, 1)).from_address(self.ptr))[: self.nbytes]

    def close(self) -> None:
        if getattr(self, "ptr", None) and _lib is not None:
            self.array = None
            _lib.cdm_host_free(ctypes.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        self.close()


def pinned(a: np.ndarray):
    """A pinned host copy of a numpy byte array (torch pin_memory)."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    return t
