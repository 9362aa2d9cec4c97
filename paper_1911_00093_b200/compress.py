"""FP64 master H-matrix: containers and the (native, parallel) ACA build.

Interface of reference pkg/src/hmx/compress.py:25-33.  The build restates
`build_hmatrix` (compress.py:285-342) in csrc/hbuild.cpp and fans the
per-block ACA out over host threads; blocks are independent, so the result
does not depend on the thread count.

Storage is packed: one float64 buffer holds every block (dense m x n values,
or U m x r followed by Vt r x n, all row-major), described by per-block
kind/rank/offset arrays.  `payloads` materialises reference-style per-block
objects (numpy views, no copies) on first access.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .partition import (
    DEFAULT_ETA,
    DEFAULT_LEAF_SIZE,
    BlockPartition,
    build_block_partition,
    build_cluster_tree,
)

__all__ = [
    "DenseBlockF64",
    "LowRankBlockF64",
    "BuildReport",
    "HMatrixF64",
    "PackedMaster",
    "build_hmatrix",
    "densify",
]

DEFAULT_ACA_TOL = 1e-8   # reference compress.py:35
DENSIFY_CAP = 4096       # reference compress.py:36


@dataclass
class DenseBlockF64:
    """A dense (inadmissible) block stored in FP64 (reference compress.py:42-50)."""
    values: np.ndarray

    def __post_init__(self):
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)


@dataclass
class LowRankBlockF64:
    """`u` rows x r, `vt` r x cols (reference compress.py:52-77)."""

    u: np.ndarray
    vt: np.ndarray
    fallback: bool = False

    def __post_init__(self):
        self.u = np.ascontiguousarray(self.u, dtype=np.float64)
        self.vt = np.ascontiguousarray(self.vt, dtype=np.float64)
        if self.u.ndim != 2 or self.vt.ndim != 2 or self.u.shape[1] != self.vt.shape[0]:
            raise ValueError(f"inconsistent factor shapes {self.u.shape} x {self.vt.shape}")
        if self.rank > min(self.u.shape[0], self.vt.shape[1]):
            raise ValueError("rank exceeds min(rows, cols)")

    @property
    def rank(self) -> int:
        return int(self.u.shape[1])


@dataclass
class BuildReport:
    """Statistics of one H-matrix build (reference compress.py:211-233)."""
    n: int
    dense_blocks: int
    lowrank_blocks: int
    fallback_blocks: int
    rank_histogram: dict
    stored_scalars: int
    compression_ratio: float
    aca_tol: float

    def to_dict(self) -> dict:
        return {
            "n": self.n, "dense_blocks": self.dense_blocks,
            "lowrank_blocks": self.lowrank_blocks, "fallback_blocks": self.fallback_blocks,
            "rank_histogram": {str(k): v for k, v in sorted(self.rank_histogram.items())},
            "stored_scalars": self.stored_scalars, "compression_ratio": self.compression_ratio,
            "aca_tol": self.aca_tol,
        }


@dataclass
class PackedMaster:
    """Packed FP64 masters: kinds (0 dense / 1 low rank), ranks, offsets into
    `data` (float64 elements)."""

    data: np.ndarray
    kinds: np.ndarray
    ranks: np.ndarray
    offsets: np.ndarray

    @classmethod
    def from_payloads(cls, table: np.ndarray, payloads) -> "PackedMaster":
        nb = table.shape[0]
        kinds = np.zeros(nb, dtype=np.int32)
        ranks = np.zeros(nb, dtype=np.int64)
        sizes = np.zeros(nb, dtype=np.int64)
        for k, p in enumerate(payloads):
            if isinstance(p, DenseBlockF64) or hasattr(p, "values"):
                sizes[k] = p.values.size
            else:
                kinds[k] = 1
                ranks[k] = p.u.shape[1]
                sizes[k] = p.u.size + p.vt.size
        offsets = np.zeros(nb, dtype=np.int64)
        if nb:
            offsets[1:] = np.cumsum(sizes)[:-1]
        data = np.empty(int(sizes.sum()), dtype=np.float64)
        for k, p in enumerate(payloads):
            o = offsets[k]
            if kinds[k] == 0:
                data[o:o + sizes[k]] = np.asarray(p.values, dtype=np.float64).ravel()
            else:
                nu = p.u.size
                data[o:o + nu] = np.asarray(p.u, dtype=np.float64).ravel()
                data[o + nu:o + sizes[k]] = np.asarray(p.vt, dtype=np.float64).ravel()
        return cls(data, kinds, ranks, offsets)

    def payload(self, table_row, k: int):
        rs, re, cs, ce = (int(v) for v in table_row[:4])
        m, n, o = re - rs, ce - cs, int(self.offsets[k])
        if self.kinds[k] == 2:
            return None  # not built (row-restricted build)
        if self.kinds[k] == 0:
            return DenseBlockF64(self.data[o:o + m * n].reshape(m, n))
        r = int(self.ranks[k])
        return LowRankBlockF64(self.data[o:o + m * r].reshape(m, r),
                               self.data[o + m * r:o + r * (m + n)].reshape(r, n))


class DevicePackedMaster(PackedMaster):
    """Packed masters built on a device (hmx_master_build): `kinds`, `ranks`,
    `offsets` on the host, `data` copied from the device on first use (the
    device-side consumers -- prepare_scheme_device, device plans -- never
    need it)."""

    def __init__(self, master, n_data: int, kinds, ranks, offsets):
        self._master = master
        self._n_data = int(n_data)
        self._data = None
        self.kinds = kinds
        self.ranks = ranks
        self.offsets = offsets

    @property
    def data(self) -> np.ndarray:
        if self._data is None:
            self._data = self._master.download(self._n_data)
        return self._data


class HMatrixF64:
    """FP64 master H-matrix: partition plus one payload per block."""

    def __init__(self, partition: BlockPartition, payloads=None, report=None,
                 packed: PackedMaster | None = None):
        self.partition = partition
        self.report = report
        self._payloads = list(payloads) if payloads is not None else None
        self._packed = packed
        if self._payloads is None and packed is None:
            raise ValueError("HMatrixF64 needs payloads or packed storage")

    @property
    def payloads(self) -> list:
        if self._payloads is None:
            t = self.partition.table
            self._payloads = [self._packed.payload(t[k], k) for k in range(t.shape[0])]
        return self._payloads

    @property
    def packed(self) -> PackedMaster:
        if self._packed is None:
            self._packed = PackedMaster.from_payloads(self.partition.table, self._payloads)
        return self._packed

    @property
    def n(self) -> int:
        return self.partition.n

    @property
    def permutation(self) -> np.ndarray:
        return self.partition.tree.permutation

    def items(self):
        return zip(self.partition.blocks, self.payloads)


def build_hmatrix(mesh, partition: BlockPartition | None = None,
                  aca_tol: float = DEFAULT_ACA_TOL, max_rank: int | None = None,
                  leaf_size: int = DEFAULT_LEAF_SIZE, eta: float = DEFAULT_ETA,
                  threads: int | None = None, rows: tuple | None = None,
                  device: int | None = None) -> HMatrixF64:
    """Compress the kernel matrix of `mesh` (reference compress.py:285-342).

    `rows=(lo, hi)` (permuted indices) builds only the blocks whose rows meet
    [lo, hi); the others are kept as kind 2 (not built, no payload).  Used by
    the multi-GPU mode, where each rank owns a row slice.

    `device=k` compresses on CUDA device k (hmx_master_build: GPU ACA and
    kernel-entry assembly, bit-identical to the host build); the masters stay
    resident there for prepare_scheme_device / device plans, and a host copy
    backs the returned object like a host build's.
    """
    if partition is None:
        tree = build_cluster_tree(mesh, leaf_size=leaf_size)
        partition = build_block_partition(tree, eta=eta)
    if aca_tol <= 0.0:
        raise ValueError("tol must be positive")
    if max_rank is not None and max_rank < 1:
        raise ValueError("max_rank must be >= 1")
    perm = partition.tree.permutation
    pcent = np.ascontiguousarray(np.asarray(mesh.centroids)[perm], dtype=np.float64)
    parea = np.ascontiguousarray(np.asarray(mesh.areas)[perm], dtype=np.float64)
    order = np.lexsort(pcent.T)
    if np.any(np.all(pcent[order[1:]] == pcent[order[:-1]], axis=1)):
        raise ValueError("mesh has coincident panel centroids")

    table = partition.table
    nb = table.shape[0]
    if device is not None:
        return _build_on_device(partition, pcent, parea, table, aca_tol, max_rank, rows, device)
    lib = _native.host()
    nthreads = threads or _native.host_threads()
    err = ctypes.create_string_buffer(256)
    handle = lib.hb_build(_native.ptr(pcent, _native.c_f64p), _native.ptr(parea, _native.c_f64p),
                          pcent.shape[0], _native.ptr(table, _native.c_i64p), nb, float(aca_tol),
                          int(max_rank or 0), int(nthreads),
                          int(rows[0]) if rows else 0, int(rows[1]) if rows else partition.n,
                          err, 256)
    if not handle:
        raise ValueError(err.value.decode() or "H-matrix build failed")
    try:
        kinds = np.empty(nb, dtype=np.int32)
        ranks = np.empty(nb, dtype=np.int64)
        offsets = np.empty(nb, dtype=np.int64)
        total = int(lib.hb_build_layout(handle, _native.ptr(kinds, _native.c_i32p),
                                        _native.ptr(ranks, _native.c_i64p),
                                        _native.ptr(offsets, _native.c_i64p)))
        data = np.empty(total, dtype=np.float64)
        lib.hb_build_export(handle, _native.ptr(data, _native.c_f64p),
                            _native.ptr(offsets, _native.c_i64p), int(nthreads))
        fallbacks = int(lib.hb_build_fallbacks(handle))
    finally:
        lib.hb_build_free(handle)

    low = kinds == 1
    hist_r, hist_c = np.unique(ranks[low], return_counts=True)
    n = partition.n
    report = BuildReport(
        n=n, dense_blocks=int(np.count_nonzero(kinds == 0)), lowrank_blocks=int(np.count_nonzero(low)),
        fallback_blocks=fallbacks,
        rank_histogram={int(r): int(c) for r, c in zip(hist_r, hist_c)},
        stored_scalars=total, compression_ratio=float(total) / float(n * n), aca_tol=aca_tol)
    return HMatrixF64(partition, report=report,
                      packed=PackedMaster(data, kinds, ranks, offsets))


def _report(n, kinds, ranks, total, fallbacks, aca_tol) -> BuildReport:
    low = kinds == 1
    hist_r, hist_c = np.unique(ranks[low], return_counts=True)
    return BuildReport(
        n=n, dense_blocks=int(np.count_nonzero(kinds == 0)), lowrank_blocks=int(np.count_nonzero(low)),
        fallback_blocks=fallbacks,
        rank_histogram={int(r): int(c) for r, c in zip(hist_r, hist_c)},
        stored_scalars=total, compression_ratio=float(total) / float(n * n), aca_tol=aca_tol)


def _build_on_device(partition, pcent, parea, table, aca_tol, max_rank, rows, device) -> HMatrixF64:
    from . import _gpu

    master, kinds, ranks, offsets, total, fallbacks = _gpu.Master.build(
        pcent, parea, partition.tree.permutation, table, aca_tol, max_rank or 0, rows,
        device=int(device))
    h = HMatrixF64(partition, report=_report(partition.n, kinds, ranks, total, fallbacks, aca_tol),
                   packed=DevicePackedMaster(master, total, kinds, ranks, offsets))
    object.__setattr__(h, "_hmx_gpu_master", master)  # device_prepare.get_master reuses it
    return h


def densify(h: HMatrixF64, cap: int = DENSIFY_CAP) -> np.ndarray:
    """Dense FP64 matrix in original index order (reference compress.py:345-357)."""
    n = h.n
    if n > cap:
        raise ValueError(f"densify of N={n} exceeds the cap of {cap}")
    out = np.zeros((n, n), dtype=np.float64)
    for blk, pay in h.items():
        vals = pay.values if hasattr(pay, "values") else pay.u @ pay.vt
        out[blk.row_start:blk.row_end, blk.col_start:blk.col_end] = vals
    perm = h.permutation
    result = np.empty_like(out)
    result[np.ix_(perm, perm)] = out
    return result
