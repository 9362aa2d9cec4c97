"""Locating, building and loading the two native libraries.

* ``libhmx_host.so``  - C++ host builder (csrc/hbuild.cpp): meshes, cluster
  tree, partition, ACA, scheme preparation.  Untimed host code.
* ``libhmx_gpu.so``   - the product: sm_100a CUDA kernels behind the C-ABI
  declared in ``include/hmx_gpu.h``.

Both are built in-tree into ``paper_1911_00093_b200/lib`` so they travel to
the GPU box with the repo snapshot.  The GPU library is never replaced by a
CPU fallback: if it is missing or no CUDA device is present, loading fails
with an exception.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
LIB_DIR = PKG_DIR / "lib"
REPO_ROOT = PKG_DIR.parent
INCLUDE_DIR = REPO_ROOT / "include"

HOST_LIB = LIB_DIR / "libhmx_host.so"
GPU_LIB = LIB_DIR / "libhmx_gpu.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = "-gencode=arch=compute_100a,code=sm_100a"

GPU_SOURCES = ["hmx_plan.cu", "hmx_kernels.cu", "hmx_solver.cu", "hmx_prepare.cu", "hmx_build.cu"]

_lock = threading.Lock()
_host = None
_gpu = None


def _run(cmd):
    proc = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if proc.returncode != 0:
        raise RuntimeError("native build failed:\n" + " ".join(cmd) + "\n" + proc.stdout)
    return proc.stdout


def build_host(force: bool = False) -> Path:
    """Compile the host C++ library (cluster tree, partition, ACA) in-tree with g++."""
    src = CSRC / "hbuild.cpp"
    if not force and HOST_LIB.exists() and HOST_LIB.stat().st_mtime >= src.stat().st_mtime:
        return HOST_LIB
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    tmp = HOST_LIB.with_suffix(".so.tmp%d" % os.getpid())
    _run(["g++", "-O3", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
          "-Wall", "-o", str(tmp), str(src)])
    os.replace(tmp, HOST_LIB)
    return HOST_LIB


def gpu_sources():
    """CUDA sources of the GPU library, in link order."""
    return [CSRC / s for s in GPU_SOURCES]


def build_gpu(force: bool = False, verbose: bool = False) -> Path:
    """Compile the GPU library in-tree for sm_100a with nvcc (`-gencode arch=compute_100a,code=sm_100a -lineinfo`)."""
    srcs = gpu_sources()
    deps = srcs + list(CSRC.glob("*.cuh")) + [INCLUDE_DIR / "hmx_gpu.h"]
    if (not force and GPU_LIB.exists()
            and all(GPU_LIB.stat().st_mtime >= p.stat().st_mtime for p in deps if p.exists())):
        return GPU_LIB
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    objs = []
    for s in srcs:
        o = LIB_DIR / (s.stem + ".o")
        cmd = [NVCC, GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-ffp-contract=off", "--fmad=true",
               "-I", str(INCLUDE_DIR), "-I", str(CSRC), "-c", str(s), "-o", str(o)]
        cmd[1:1] = os.environ.get("HMX_NVCC_EXTRA", "").split()  # A/B builds (tools/ab_build.sh)
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        out = _run(cmd)
        if verbose and out:
            print(out)
        objs.append(str(o))
    tmp = GPU_LIB.with_suffix(".so.tmp%d" % os.getpid())
    _run([NVCC, GENCODE, "-shared", "-o", str(tmp)] + objs + ["-lcudart", "-ldl"])
    os.replace(tmp, GPU_LIB)
    return GPU_LIB


# --------------------------------------------------------------------------
# host library

c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_f64p = ctypes.POINTER(ctypes.c_double)
c_f32p = ctypes.POINTER(ctypes.c_float)
c_i8p = ctypes.POINTER(ctypes.c_int8)


class HbNode(ctypes.Structure):
    """ctypes mirror of one cluster-tree node of the host library (index range, bounding box, children)."""
    _fields_ = [("start", ctypes.c_int64), ("end", ctypes.c_int64),
                ("bmin", ctypes.c_double * 3), ("bmax", ctypes.c_double * 3),
                ("left", ctypes.c_int64), ("right", ctypes.c_int64)]


def host():
    """The host-builder library (built on first use if absent)."""
    global _host
    with _lock:
        if _host is None:
            lib = ctypes.CDLL(str(build_host()))
            lib.hb_icosphere_nverts.restype = ctypes.c_int64
            lib.hb_icosphere_nfaces.restype = ctypes.c_int64
            lib.hb_icosphere.argtypes = [ctypes.c_int, c_f64p, c_i64p]
            lib.hb_normalize_rows3.argtypes = [c_f64p, ctypes.c_int64]
            lib.hb_normalize_rows3.restype = None
            lib.hb_cluster_tree.argtypes = [c_f64p, ctypes.c_int64, ctypes.c_int64, c_i64p,
                                            ctypes.c_void_p, ctypes.c_int64, c_i64p]
            lib.hb_partition.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                         c_i64p, ctypes.c_int64]
            lib.hb_partition.restype = ctypes.c_int64
            lib.hb_is_admissible.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double]
            lib.hb_build.argtypes = [c_f64p, c_f64p, ctypes.c_int64, c_i64p, ctypes.c_int64,
                                     ctypes.c_double, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_char_p, ctypes.c_int]
            lib.hb_build.restype = ctypes.c_void_p
            lib.hb_build_fallbacks.argtypes = [ctypes.c_void_p]
            lib.hb_build_fallbacks.restype = ctypes.c_int64
            lib.hb_build_layout.argtypes = [ctypes.c_void_p, c_i32p, c_i64p, c_i64p]
            lib.hb_build_layout.restype = ctypes.c_int64
            lib.hb_build_export.argtypes = [ctypes.c_void_p, c_f64p, c_i64p, ctypes.c_int]
            lib.hb_build_free.argtypes = [ctypes.c_void_p]
            lib.hb_build_free.restype = None
            lib.hb_scale_diag.argtypes = [c_f64p, ctypes.c_int64, c_i32p, c_i64p, c_i64p, c_i64p,
                                          c_i64p, c_i64p, ctypes.c_double, ctypes.c_int, c_f64p,
                                          c_i8p, c_i64p, ctypes.c_int]
            lib.hb_scale_fill.argtypes = [c_f64p, ctypes.c_int64, c_i32p, c_i64p, c_i64p, c_i64p,
                                          c_i64p, c_i64p, c_i8p, c_i64p, c_i64p, c_f64p, c_f32p,
                                          c_f64p, c_f64p, c_i64p, ctypes.c_int]
            lib.hb_cast_f32.argtypes = [c_f64p, ctypes.c_int64, c_f32p, c_i64p, ctypes.c_int]
            lib.hb_cast_f32.restype = ctypes.c_int64
            lib.hb_copy_f64.argtypes = [c_f64p, c_f64p, ctypes.c_int64, ctypes.c_int]
            lib.hb_copy_f64.restype = None
            _host = lib
    return _host


def ptr(arr, ctype):
    """ctypes pointer to a numpy array's data (None for None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(ctype)


def host_threads() -> int:
    """Thread count of the host builder (HMX_HOST_THREADS, else the CPU count)."""
    env = os.environ.get("HMX_HOST_THREADS")
    if env:
        return max(1, int(env))
    return max(1, os.cpu_count() or 1)
