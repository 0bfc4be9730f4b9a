"""Build + load helpers for the in-tree native libraries of the product path.

Everything is compiled IN-TREE (the .so files travel to the GPU box with the gpurun snapshot):
  paper_2602_08190_b200/_lib/libcdm.so       CUDA decode runtime + kernels, C-ABI in include/cdm.h
  paper_2602_08190_b200/_lib/libcdm_gen.so   seeded TPC-H-shaped input generator (inputs/)
  paper_2602_08190_b200/_lib/libcdm_enc.so   CPU cascade encoder (encoder/), links liblz4
The CPU oracle (oracle/, test infrastructure) is built by oracle.build() (oracle/oracle.py), never from here.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIBDIR = os.path.join(PKG, "_lib")
NVCC = os.environ.get("CDM_NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

_lock = threading.Lock()


def _newer(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)


def _csrc(*names: str) -> list[str]:
    return [os.path.join(PKG, "csrc", n) for n in names]


CUDA_SOURCES = ["runtime.cpp", "kernels_fp.cu", "kernels_fpc.cu", "kernels_scan.cu", "kernels_rle.cu", "kernels_lz4.cu", "kernels_ans.cu", "kernels_strdict.cu",
                "kernels_util.cu"]
CUDA_HEADERS = ["format.h", "plan.h", "kernels.h", "device_util.cuh"]


def build_cdm(force: bool = False) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 ... -> _lib/libcdm.so"""
    os.makedirs(LIBDIR, exist_ok=True)
    out = os.path.join(LIBDIR, "libcdm.so")
    srcs = _csrc(*CUDA_SOURCES)
    deps = srcs + _csrc(*CUDA_HEADERS) + [os.path.join(ROOT, "include", "cdm.h")]
    if not force and not _newer(out, deps):
        return out
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        objs.append(o)
        cmd = [NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden",
               "-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc"),
               "-Xptxas", "-warn-spills", "-c", s, "-o", o]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for cmd, p in procs:
        txt = p.communicate()[0]
        if p.returncode != 0:
            raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + txt)
    _run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-lpthread"])
    return out


def build_gen(force: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    out = os.path.join(LIBDIR, "libcdm_gen.so")
    src = os.path.join(PKG, "inputs", "tpch_gen.c")
    if force or _newer(out, [src]):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fvisibility=hidden", "-o", out, src, "-lm"])
    return out


def build_enc(force: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    out = os.path.join(LIBDIR, "libcdm_enc.so")
    src = os.path.join(PKG, "encoder", "cdm_encode.c")
    if force or _newer(out, [src]):
        _run(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fvisibility=hidden", "-o", out, src,
              "-l:liblz4.so.1", "-lm"])
    return out


def build_all(force: bool = False) -> None:
    with _lock:
        build_gen(force)
        build_enc(force)
        build_cdm(force)


_loaded: dict[str, ctypes.CDLL] = {}


def load(name: str, builder=None) -> ctypes.CDLL:
    """Load an in-tree library, building it first if it is missing or stale (CPU-only build step)."""
    with _lock:
        if name in _loaded:
            return _loaded[name]
        path = os.path.join(LIBDIR, name)
        if builder is not None:
            try:
                builder()
            except (OSError, RuntimeError):
                if not os.path.exists(path):
                    raise
        if not os.path.exists(path):
            raise RuntimeError(f"native library {path} is missing; run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        _loaded[name] = lib
        return lib
