"""ctypes binding of the C ABI in include/hmx_gpu.h (libhmx_gpu.so).

There is deliberately no CPU fallback: every public entry point of this
package that computes a matvec or a solve goes through these bindings and
raises if the library cannot be loaded or no CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _native

HMX_OK, HMX_ERR_ARG, HMX_ERR_CUDA, HMX_ERR_NONFINITE, HMX_ERR_SHAPE, HMX_ERR_OVERFLOW = 0, 1, 2, 3, 4, 5
HMX_ERR_COMM = 6
HMX_DEVICE_PTRS, HMX_PERMUTED = 1, 2

SCHEME_CODES = {"m1-double": 0, "m1-single": 1, "m1-mixed": 2, "m2-double": 3,
                "m2-single": 4, "m2-mixed": 5}

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)


class MatrixDesc(ctypes.Structure):
    """ctypes mirror of `hmx_matrix_desc` (include/hmx_gpu.h:72-93): the packed H-matrix handed to `hmx_plan_create`."""
    _fields_ = [("n", ctypes.c_int64), ("n_blocks", ctypes.c_int64),
                ("scheme", ctypes.c_int32), ("a32", ctypes.c_int32), ("hi32", ctypes.c_int32),
                ("reserved", ctypes.c_int32),
                ("perm", _i64p), ("table", _i64p), ("kind", _i32p),
                ("a_off", _i64p), ("hi_off", _i64p), ("khi", _i64p), ("dhi_off", _i64p),
                ("lo_off", _i64p), ("klo", _i64p), ("dlo_off", _i64p),
                ("buf64", ctypes.POINTER(ctypes.c_double)), ("n64", ctypes.c_int64),
                ("buf32", ctypes.POINTER(ctypes.c_float)), ("n32", ctypes.c_int64)]


class PlanOptions(ctypes.Structure):
    """ctypes mirror of `hmx_plan_options` (include/hmx_gpu.h:97-102)."""
    _fields_ = [("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("s1_chunk_bytes", ctypes.c_int32), ("flags", ctypes.c_int32)]


HMX_PLAN_LOCAL_FIRST = 1
HMX_PLAN_FP32_CHAIN = 2


def fp32_order_flags() -> int:
    """Plan flags of the FP32 accumulation order: HMX_FP32_ORDER=sgemv (the
    default: OpenBLAS SGEMV-T's own order, bitwise the reference's FP32
    products) or chain (one sequential FP32 chain per (row, block): faster,
    the round-1 order)."""
    import os
    order = os.environ.get("HMX_FP32_ORDER", "sgemv").lower()
    if order not in ("sgemv", "chain"):
        raise ValueError(f"HMX_FP32_ORDER must be 'sgemv' or 'chain', not {order!r}")
    return HMX_PLAN_FP32_CHAIN if order == "chain" else 0


class PlanInfo(ctypes.Structure):
    """ctypes mirror of `hmx_plan_info` (include/hmx_gpu.h:112-121): bytes streamed per matvec and the launch shape."""
    _fields_ = [("n", ctypes.c_int64), ("payload_bytes", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("s1_segments", ctypes.c_int64),
                ("s1_tasks", ctypes.c_int64), ("s2_segments", ctypes.c_int64),
                ("s2_runs", ctypes.c_int64), ("z_len", ctypes.c_int64),
                ("stage1_bytes", ctypes.c_int64), ("stage2_bytes", ctypes.c_int64),
                ("s1_grid", ctypes.c_int32), ("s1_block", ctypes.c_int32),
                ("s2_grid", ctypes.c_int32), ("s2_block", ctypes.c_int32)]


class SolveReport(ctypes.Structure):
    """ctypes mirror of `hmx_solve_report` (include/hmx_gpu.h:156-168)."""
    _fields_ = [("converged", ctypes.c_int32), ("iterations", ctypes.c_int32),
                ("has_true_residual", ctypes.c_int32), ("breakdown", ctypes.c_int32),
                ("true_residual", ctypes.c_double), ("breakdown_value", ctypes.c_double),
                ("breakdown_iteration", ctypes.c_int32), ("history_len", ctypes.c_int32),
                ("matvecs", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("device_ms", ctypes.c_double)]


class MasterDesc(ctypes.Structure):
    """ctypes mirror of `hmx_master_desc` (include/hmx_gpu.h:130-140): the FP64 master copy kept on the device."""
    _fields_ = [("n", ctypes.c_int64), ("n_blocks", ctypes.c_int64),
                ("perm", _i64p), ("table", _i64p), ("kind", _i32p), ("offset", _i64p),
                ("rank", _i64p), ("data", ctypes.POINTER(ctypes.c_double)),
                ("n_data", ctypes.c_int64)]


class BuildDesc(ctypes.Structure):
    """ctypes mirror of `hmx_build_desc` (include/hmx_gpu.h:217-228): inputs of the on-device ACA compression."""
    _fields_ = [("n", ctypes.c_int64), ("n_blocks", ctypes.c_int64),
                ("pcent", ctypes.POINTER(ctypes.c_double)), ("parea", ctypes.POINTER(ctypes.c_double)),
                ("perm", _i64p), ("table", _i64p), ("tol", ctypes.c_double),
                ("max_rank", ctypes.c_int64), ("row_lo", ctypes.c_int64), ("row_hi", ctypes.c_int64)]


class PrepareInfo(ctypes.Structure):
    """ctypes mirror of `hmx_prepare_info` (include/hmx_gpu.h:145-150)."""
    _fields_ = [("payload_bytes", ctypes.c_int64), ("underflow_count", ctypes.c_int64),
                ("overflow_block", ctypes.c_int64), ("fp32_ranks", ctypes.c_int64)]


# every exported symbol of include/hmx_gpu.h with its ctypes signature
SIGNATURES = {
    "hmx_last_error": (ctypes.c_char_p, []),
    "hmx_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "hmx_plan_create": (ctypes.c_int, [ctypes.POINTER(MatrixDesc), ctypes.c_int,
                                       ctypes.POINTER(PlanOptions),
                                       ctypes.POINTER(ctypes.c_void_p)]),
    "hmx_plan_destroy": (None, [ctypes.c_void_p]),
    "hmx_plan_get_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PlanInfo)]),
    "hmx_matvec": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_int]),
    "hmx_nonfinite_block": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "hmx_true_residual": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.POINTER(ctypes.c_double)]),
    "hmx_bicgstab": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_double, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.POINTER(SolveReport)]),
    "hmx_bench_matvec": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int64, ctypes.POINTER(ctypes.c_double)]),
    "hmx_apply_local": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_uint64]),
    "hmx_master_create": (ctypes.c_int, [ctypes.POINTER(MasterDesc), ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_void_p)]),
    "hmx_master_destroy": (None, [ctypes.c_void_p]),
    "hmx_master_build": (ctypes.c_int, [ctypes.POINTER(BuildDesc), ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_void_p), _i32p, _i64p, _i64p,
                                        _i64p, _i64p]),
    "hmx_master_download": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "hmx_plan_create_prepared": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_double,
                                                ctypes.POINTER(PlanOptions),
                                                ctypes.POINTER(ctypes.c_void_p),
                                                ctypes.POINTER(PrepareInfo)]),
    "hmx_host_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    "hmx_comm_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "hmx_comm_create": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       _i64p, ctypes.POINTER(ctypes.c_void_p)]),
    "hmx_comm_destroy": (None, [ctypes.c_void_p]),
    "hmx_dist_matvec": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64]),
    "hmx_bicgstab_dist": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_double, ctypes.c_int,
                                         ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.POINTER(SolveReport)]),
    "hmx_host_free": (None, [ctypes.c_void_p]),
}

_lib = None
_lock = threading.Lock()


def load_library(build: bool = False):
    """Load libhmx_gpu.so (building it first if asked).  Raises if absent."""
    global _lib
    with _lock:
        if _lib is None:
            path = _native.GPU_LIB
            if os.environ.get("HMX_GPU_LIB"):  # A/B experiments with another build
                from pathlib import Path
                path = Path(os.environ["HMX_GPU_LIB"])
            elif build or os.environ.get("HMX_BUILD_ON_IMPORT") == "1":
                path = _native.build_gpu()
            if not path.exists():
                raise RuntimeError(
                    f"{path} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                    "There is no CPU fallback for the H-matvec.")
            lib = ctypes.CDLL(str(path))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    """Message of the last failed `hmx_*` call on this thread."""
    msg = load_library().hmx_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str):
    """Raise the Python exception matching an `hmx_status` code (include/hmx_gpu.h:38-46); no-op on HMX_OK."""
    if rc == HMX_OK:
        return
    msg = f"{what} failed: {last_error()}"
    if rc == HMX_ERR_SHAPE:
        raise ValueError(msg)
    if rc == HMX_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(msg)


def device_count() -> int:
    """Number of CUDA devices the native library sees."""
    lib = load_library()
    c = ctypes.c_int(0)
    lib.hmx_device_count(ctypes.byref(c))
    return c.value


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


class Plan:
    """A device-resident flattened H-matrix for one scheme (owns a C plan)."""

    def __init__(self, packed, table, perm, scheme_label: str, n: int, device: int = 0,
                 row_range=None, s1_chunk_bytes: int = 0, local_first: bool = False):
        lib = load_library()
        code = SCHEME_CODES.get(scheme_label, 6 if scheme_label.startswith("m3") else None)
        if code is None:
            raise ValueError(f"unsupported scheme {scheme_label!r}")
        self._keep = []

        def keep(a, dtype):
            a = np.ascontiguousarray(a, dtype=dtype)
            self._keep.append(a)
            return a

        t = keep(table, np.int64)
        d = MatrixDesc()
        d.n = n
        d.n_blocks = t.shape[0]
        d.scheme = code
        d.a32 = int(bool(packed.a32))
        d.hi32 = int(bool(packed.hi32))
        d.perm = _p(keep(perm, np.int64), ctypes.c_int64)
        d.table = _p(t, ctypes.c_int64)
        d.kind = _p(keep(packed.kind, np.int32), ctypes.c_int32)
        for name in ("a_off", "hi_off", "khi", "dhi_off", "lo_off", "klo", "dlo_off"):
            setattr(d, name, _p(keep(getattr(packed, name), np.int64), ctypes.c_int64))
        b64 = keep(packed.buf64 if packed.buf64.size else np.zeros(1), np.float64)
        b32 = keep(packed.buf32 if packed.buf32.size else np.zeros(1, np.float32), np.float32)
        d.buf64 = _p(b64, ctypes.c_double)
        d.n64 = int(packed.buf64.size)
        d.buf32 = _p(b32, ctypes.c_float)
        d.n32 = int(packed.buf32.size)
        opt = PlanOptions()
        if row_range is not None:
            opt.row_begin, opt.row_end = int(row_range[0]), int(row_range[1])
        opt.s1_chunk_bytes = int(s1_chunk_bytes)
        opt.flags = (HMX_PLAN_LOCAL_FIRST if local_first else 0) | fp32_order_flags()
        h = ctypes.c_void_p()
        rc = lib.hmx_plan_create(ctypes.byref(d), int(device), ctypes.byref(opt), ctypes.byref(h))
        self._keep = []  # the plan holds device copies; host arrays may go
        check(rc, "hmx_plan_create")
        self.handle = h
        self.n = n
        self.scheme = scheme_label
        self.device = device
        self._lib = lib

    @classmethod
    def prepared(cls, master: "Master", scheme_label: str, split_factor: float = 0.0,
                 row_range=None) -> tuple["Plan", dict]:
        """prepare_scheme + plan on the device from resident masters
        (hmx_plan_create_prepared).  Raises OverflowError like the reference's
        _cast_fp32 (precision.py:241-253); the message is completed by the
        caller, which knows the block geometry."""
        lib = load_library()
        code = SCHEME_CODES.get(scheme_label, 6 if scheme_label.startswith("m3") else None)
        if code is None:
            raise ValueError(f"unsupported scheme {scheme_label!r}")
        opt = PlanOptions()
        if row_range is not None:
            opt.row_begin, opt.row_end = int(row_range[0]), int(row_range[1])
        opt.flags = fp32_order_flags()
        h = ctypes.c_void_p()
        info = PrepareInfo()
        rc = lib.hmx_plan_create_prepared(master.handle, code, float(split_factor),
                                          ctypes.byref(opt), ctypes.byref(h), ctypes.byref(info))
        out = {f: getattr(info, f) for f, _ in PrepareInfo._fields_}
        if rc == HMX_ERR_OVERFLOW:
            raise OverflowError(f"block {out['overflow_block']}")
        check(rc, "hmx_plan_create_prepared")
        self = cls.__new__(cls)
        self._keep = []
        self.handle = h
        self.n = master.n
        self.scheme = scheme_label
        self.device = master.device
        self._lib = lib
        return self, out

    def info(self) -> dict:
        i = PlanInfo()
        check(self._lib.hmx_plan_get_info(self.handle, ctypes.byref(i)), "hmx_plan_get_info")
        return {f: getattr(i, f) for f, _ in PlanInfo._fields_}

    def matvec(self, x: np.ndarray, permuted: bool = False) -> tuple[np.ndarray, int]:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = result_array(self.n)
        rc = self._lib.hmx_matvec(self.handle, x.ctypes.data, y.ctypes.data,
                                  HMX_PERMUTED if permuted else 0)
        if rc not in (HMX_OK, HMX_ERR_NONFINITE):
            check(rc, "hmx_matvec")
        return y, rc

    def matvec_device(self, x_ptr: int, y_ptr: int, permuted: bool = True) -> int:
        rc = self._lib.hmx_matvec(self.handle, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr),
                                  HMX_DEVICE_PTRS | (HMX_PERMUTED if permuted else 0))
        if rc not in (HMX_OK, HMX_ERR_NONFINITE):
            check(rc, "hmx_matvec")
        return rc

    def apply_local(self, xp_ptr: int, y_ptr: int, w1_ptr: int = 0, yy: bool = False,
                    dots_ptr: int = 0, nonfinite_ptr: int = 0, stream: int | None = None) -> None:
        """Enqueue the local rows of y = A xp (device pointers) on `stream`
        (a cudaStream_t handle such as torch's `cuda_stream`; None = the
        plan's own stream)."""
        stream = (1 << 64) - 1 if stream is None else stream
        rc = self._lib.hmx_apply_local(self.handle, ctypes.c_void_p(xp_ptr), ctypes.c_void_p(y_ptr),
                                       ctypes.c_void_p(w1_ptr or None), int(bool(yy)),
                                       ctypes.c_void_p(dots_ptr or None),
                                       ctypes.c_void_p(nonfinite_ptr or None), int(stream))
        check(rc, "hmx_apply_local")

    def nonfinite_block(self) -> int:
        b = ctypes.c_int64(-1)
        check(self._lib.hmx_nonfinite_block(self.handle, ctypes.byref(b)), "hmx_nonfinite_block")
        return b.value

    def bench(self, warmup: int, iters: int, flush_l2: int = 0) -> dict:
        out = (ctypes.c_double * 4)()
        check(self._lib.hmx_bench_matvec(self.handle, warmup, iters, flush_l2, out),
              "hmx_bench_matvec")
        return {"ms": out[0], "stage1_ms": out[1], "stage2_ms": out[2], "min_ms": out[3]}

    @property
    def closed(self) -> bool:
        return not getattr(self, "handle", None)

    def close(self):
        if getattr(self, "handle", None):
            self._lib.hmx_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _PinnedLease:
    """Owner of one pooled page-locked buffer; numpy arrays made from it keep
    it alive (ndarray.base) and it returns to the pool when the last one dies."""

    __slots__ = ("ptr", "nbytes", "__array_interface__")

    def __init__(self, ptr: int, nbytes: int):
        self.ptr = ptr
        self.nbytes = nbytes
        self.__array_interface__ = {"shape": (nbytes // 8,), "typestr": "<f8",
                                    "data": (ptr, False), "version": 3}

    def __del__(self):
        try:
            _host_pool.release(self.ptr, self.nbytes)
        except Exception:
            pass


class _HostPool:
    """Page-locked buffers for matvec results.  The reference returns a fresh
    array per call (matvec.py:145-147); so does this pool - each buffer backs
    at most one live array - but the device->host copy into it is one DMA
    instead of the driver's staged pageable copy.  Live plus cached pinned
    bytes are capped (HMX_PINNED_POOL_MB, default 1024); past the cap,
    results are ordinary pageable arrays."""

    def __init__(self):
        self.lock = threading.Lock()
        self.free: dict[int, list[int]] = {}
        self.held = 0
        self.cap = int(os.environ.get("HMX_PINNED_POOL_MB", "1024")) << 20

    def array(self, n: int):
        nbytes = 8 * int(n)
        with self.lock:
            bucket = self.free.get(nbytes)
            ptr = bucket.pop() if bucket else None
            if ptr is None:
                if self.held + nbytes > self.cap:
                    return None
                out = ctypes.c_void_p()
                if load_library().hmx_host_alloc(nbytes, ctypes.byref(out)) != HMX_OK:
                    return None
                ptr = out.value
                self.held += nbytes
        return np.asarray(_PinnedLease(ptr, nbytes))

    def release(self, ptr: int, nbytes: int) -> None:
        with self.lock:
            self.free.setdefault(nbytes, []).append(ptr)


_host_pool = _HostPool()


def result_array(n: int) -> np.ndarray:
    """A fresh, uninitialised float64 array of length n for a matvec result
    (page-locked when the pool allows)."""
    if n > 0:
        y = _host_pool.array(n)
        if y is not None:
            return y
    return np.empty(n, dtype=np.float64)


def _nccl_first():
    """Load torch (and with it torch's NCCL) before libhmx_gpu resolves NCCL
    at run time, so the process holds one NCCL: libhmx_gpu's dlopen of
    libnccl.so.2 then returns torch's copy."""
    import torch  # noqa: F401


class Comm:
    """This rank's NCCL communicator and multi-GPU solver workspace
    (hmx_comm_create).  `cuts` are the world + 1 row-slice boundaries of the
    permuted index space; `uid` is Comm.unique_id() made on rank 0 and
    passed to every rank."""

    def __init__(self, uid: bytes, world: int, rank: int, device: int, cuts):
        _nccl_first()
        lib = load_library()
        self._cuts = np.ascontiguousarray(cuts, dtype=np.int64)
        if self._cuts.shape != (world + 1,):
            raise ValueError("cuts must have world + 1 entries")
        h = ctypes.c_void_p()
        check(lib.hmx_comm_create(bytes(uid), int(world), int(rank), int(device),
                                  _p(self._cuts, ctypes.c_int64), ctypes.byref(h)),
              "hmx_comm_create")
        self.handle = h
        self.world, self.rank, self.device = int(world), int(rank), int(device)
        self.r0, self.r1 = int(self._cuts[rank]), int(self._cuts[rank + 1])
        self._lib = lib

    @staticmethod
    def unique_id() -> bytes:
        _nccl_first()
        buf = ctypes.create_string_buffer(128)
        check(load_library().hmx_comm_unique_id(buf), "hmx_comm_unique_id")
        return buf.raw

    def matvec(self, plan: "Plan", x_local_ptr: int, y_local_ptr: int, nonfinite_ptr: int = 0,
               stream: int | None = None) -> None:
        """Enqueue y_local = (A x)[r0:r1] (device pointers, permuted order):
        allgather of the x slices, then the local product."""
        stream = (1 << 64) - 1 if stream is None else stream
        check(self._lib.hmx_dist_matvec(plan.handle, self.handle, ctypes.c_void_p(x_local_ptr),
                                        ctypes.c_void_p(y_local_ptr),
                                        ctypes.c_void_p(nonfinite_ptr or None), int(stream)),
              "hmx_dist_matvec")

    def bicgstab(self, plan: "Plan", plan64: "Plan", b_local, tol: float, max_iter: int):
        """BiCG-STAB on this rank's rows: returns (x_local, SolveReport,
        history array, rc)."""
        b = np.ascontiguousarray(b_local, dtype=np.float64)
        if b.shape != (self.r1 - self.r0,):
            raise ValueError(f"local right-hand side shape {b.shape} != ({self.r1 - self.r0},)")
        x = np.zeros_like(b)
        hist = np.zeros(int(max_iter) + 2, dtype=np.float64)
        rep = SolveReport()
        rc = self._lib.hmx_bicgstab_dist(plan.handle, plan64.handle if plan64 else None,
                                         self.handle, b.ctypes.data, float(tol), int(max_iter),
                                         x.ctypes.data, hist.ctypes.data, ctypes.byref(rep))
        if rc not in (HMX_OK, HMX_ERR_NONFINITE):
            check(rc, "hmx_bicgstab_dist")
        return x, rep, hist, rc

    @property
    def closed(self) -> bool:
        return not getattr(self, "handle", None)

    def close(self):
        if getattr(self, "handle", None):
            self._lib.hmx_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Master:
    """FP64 masters of one H-matrix resident on a device (hmx_master_create);
    schemes are then prepared on the device with Plan.prepared."""

    def __init__(self, packed_master, table, perm, n: int, device: int = 0):
        lib = load_library()
        keep = [np.ascontiguousarray(perm, dtype=np.int64),
                np.ascontiguousarray(table, dtype=np.int64),
                np.ascontiguousarray(packed_master.kinds, dtype=np.int32),
                np.ascontiguousarray(packed_master.offsets, dtype=np.int64),
                np.ascontiguousarray(packed_master.ranks, dtype=np.int64),
                np.ascontiguousarray(packed_master.data, dtype=np.float64)]
        d = MasterDesc()
        d.n = int(n)
        d.n_blocks = keep[1].shape[0]
        d.perm = _p(keep[0], ctypes.c_int64)
        d.table = _p(keep[1], ctypes.c_int64)
        d.kind = _p(keep[2], ctypes.c_int32)
        d.offset = _p(keep[3], ctypes.c_int64)
        d.rank = _p(keep[4], ctypes.c_int64)
        d.data = _p(keep[5] if keep[5].size else np.zeros(1), ctypes.c_double)
        d.n_data = int(keep[5].size)
        h = ctypes.c_void_p()
        check(lib.hmx_master_create(ctypes.byref(d), int(device), ctypes.byref(h)),
              "hmx_master_create")
        self.handle = h
        self.n = int(n)
        self.device = int(device)
        self._lib = lib

    @classmethod
    def build(cls, pcent, parea, perm, table, tol: float, max_rank: int = 0, rows=None,
              device: int = 0):
        """Build the masters on the device (hmx_master_build): returns
        (Master, kinds, ranks, offsets, n_data, fallbacks)."""
        lib = load_library()
        keep = [np.ascontiguousarray(pcent, dtype=np.float64),
                np.ascontiguousarray(parea, dtype=np.float64),
                np.ascontiguousarray(perm, dtype=np.int64),
                np.ascontiguousarray(table, dtype=np.int64)]
        nb = keep[3].shape[0]
        d = BuildDesc()
        d.n = keep[1].shape[0]
        d.n_blocks = nb
        d.pcent = _p(keep[0], ctypes.c_double)
        d.parea = _p(keep[1], ctypes.c_double)
        d.perm = _p(keep[2], ctypes.c_int64)
        d.table = _p(keep[3], ctypes.c_int64)
        d.tol = float(tol)
        d.max_rank = int(max_rank or 0)
        d.row_lo, d.row_hi = (int(rows[0]), int(rows[1])) if rows else (0, 0)
        kinds = np.empty(nb, dtype=np.int32)
        ranks = np.empty(nb, dtype=np.int64)
        offsets = np.empty(nb, dtype=np.int64)
        n_data, fallbacks = ctypes.c_int64(0), ctypes.c_int64(0)
        h = ctypes.c_void_p()
        check(lib.hmx_master_build(ctypes.byref(d), int(device), ctypes.byref(h),
                                   _p(kinds, ctypes.c_int32), _p(ranks, ctypes.c_int64),
                                   _p(offsets, ctypes.c_int64), ctypes.byref(n_data),
                                   ctypes.byref(fallbacks)), "hmx_master_build")
        self = cls.__new__(cls)
        self.handle = h
        self.n = int(d.n)
        self.device = int(device)
        self._lib = lib
        return self, kinds, ranks, offsets, int(n_data.value), int(fallbacks.value)

    def download(self, n_data: int) -> np.ndarray:
        """The packed master data (float64) on the host."""
        out = np.empty(n_data, dtype=np.float64)
        check(self._lib.hmx_master_download(self.handle, out.ctypes.data), "hmx_master_download")
        return out

    @property
    def closed(self) -> bool:
        return not getattr(self, "handle", None)

    def close(self):
        if getattr(self, "handle", None):
            self._lib.hmx_master_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
