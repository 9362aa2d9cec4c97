"""Reference-shaped objects for the drop-in tests (test infrastructure).

The classes below have the names, fields and methods of the reference's
hmx.precision payloads and containers (reference precision.py:52-104,
:169-234; compress.py:42-77; partition.py:63-71, :108-139) -- not this
repo's classes.  `scheme_hmatrix(name)` rebuilds the reference's own
SchemeHMatrix of the ref240_aca4 fixture from the arrays the reference
produced (tests/golden/make_refpayloads.py), so the GPU path can be driven
exactly as the reference's callers drive it, on a box without the reference.
"""
from __future__ import annotations

import types
from dataclasses import dataclass, field

import numpy as np

from golden_util import GOLDEN, load


@dataclass(frozen=True)
class PrecisionScheme:
    method: int
    variant: str | None = None
    c: int | None = None

    @property
    def label(self) -> str:
        if self.method == 3:
            return f"m3:c={self.c}"
        return f"m{self.method}-{self.variant}"

    @property
    def reads_fp32_source(self) -> bool:
        return self.variant == "single"

    @property
    def casts_dense_fp32(self) -> bool:
        return self.method in (1, 2) and self.variant != "double"


def parse_scheme(name: str) -> PrecisionScheme:
    if name.startswith("m3:c="):
        return PrecisionScheme(3, None, int(name[5:]))
    m, v = name.split("-")
    return PrecisionScheme(int(m[1]), v)


@dataclass(slots=True)
class DensePayload:
    values: np.ndarray


@dataclass(slots=True)
class FactorPayload:
    u: np.ndarray
    vt: np.ndarray


@dataclass(slots=True)
class ScaledPayload:
    u: np.ndarray
    vt: np.ndarray
    diag: np.ndarray


@dataclass(slots=True)
class SplitLowRank:
    idx_fp64: np.ndarray
    idx_fp32: np.ndarray
    u_hi: np.ndarray
    vt_hi: np.ndarray
    diag_hi: np.ndarray
    u_lo: np.ndarray
    vt_lo: np.ndarray
    diag_lo: np.ndarray


@dataclass
class DenseBlockF64:
    values: np.ndarray


@dataclass
class LowRankBlockF64:
    u: np.ndarray
    vt: np.ndarray

    @property
    def rank(self) -> int:
        return int(self.u.shape[1])


@dataclass(frozen=True)
class Block:
    row_start: int
    row_end: int
    col_start: int
    col_end: int
    admissible: bool


@dataclass
class BlockPartition:
    blocks: list
    n: int


@dataclass
class HMatrixF64:
    partition: BlockPartition
    payloads: list
    permutation: np.ndarray

    @property
    def n(self) -> int:
        return self.partition.n


@dataclass
class SchemeHMatrix:
    base: HMatrixF64
    scheme: PrecisionScheme
    payloads: list
    payload_bytes: int
    underflow_count: int = 0
    _blocks: list = field(default=None, repr=False)

    def __post_init__(self):
        if self._blocks is None:
            self._blocks = self.base.partition.blocks

    @property
    def n(self) -> int:
        return self.base.n

    def items(self):
        return zip(self._blocks, self.payloads)


_KIND = {0: (DensePayload, ("values",)), 1: (FactorPayload, ("u", "vt")),
         2: (ScaledPayload, ("u", "vt", "diag")),
         3: (SplitLowRank, ("idx_fp64", "idx_fp32", "u_hi", "vt_hi", "diag_hi", "u_lo", "vt_lo",
                            "diag_lo"))}


def hmatrix():
    """The reference's FP64 masters of the ref240_aca4 fixture, reference-shaped."""
    arr, meta = load("ref240_aca4")
    table, kinds, ranks, data = arr["table"], arr["kinds"], arr["ranks"], arr["data"]
    blocks = [Block(int(r[0]), int(r[1]), int(r[2]), int(r[3]), bool(r[4])) for r in table]
    pays, off = [], 0
    for b, kd, rk in zip(blocks, kinds, ranks):
        m, n = b.row_end - b.row_start, b.col_end - b.col_start
        if kd == 0:
            pays.append(DenseBlockF64(data[off:off + m * n].reshape(m, n)))
            off += m * n
        else:
            u = data[off:off + m * rk].reshape(m, rk)
            vt = data[off + m * rk:off + rk * (m + n)].reshape(rk, n)
            pays.append(LowRankBlockF64(u, vt))
            off += rk * (m + n)
    part = BlockPartition(blocks, int(arr["perm"].shape[0]))
    return HMatrixF64(part, pays, arr["perm"]), arr, meta


def scheme_hmatrix(h, name: str) -> SchemeHMatrix:
    """The reference's own prepare_scheme(h, name) result, rebuilt from its arrays."""
    f = np.load(GOLDEN / "ref240_aca4_payloads.npz")
    kinds = f[f"{name}/kind"]
    pays = []
    for k, kd in enumerate(kinds):
        cls, fields = _KIND[int(kd)]
        pays.append(cls(*[f[f"{name}/{k}/{fl}"] for fl in fields]))
    return SchemeHMatrix(h, parse_scheme(name), pays, int(f[f"{name}/payload_bytes"]),
                         int(f[f"{name}/underflow_count"]))


def fake_reference_package(name: str = "hmx_refshape"):
    """A module tree with the reference package's layout (hmx, hmx.matvec,
    hmx.solver, hmx.bench) holding placeholder operator names, for
    drop_in.install to rebind."""
    import sys

    def placeholder(*_a, **_k):
        raise AssertionError("the reference's CPU operator was called")

    root = types.ModuleType(name)
    root.__path__ = []
    for sub in ("matvec", "solver", "bench"):
        m = types.ModuleType(f"{name}.{sub}")
        for attr in ("matvec", "matvec_threaded", "bicgstab", "true_residual"):
            setattr(m, attr, placeholder)
        setattr(root, sub, m)
        sys.modules[f"{name}.{sub}"] = m
    for attr in ("matvec", "matvec_threaded", "bicgstab", "true_residual"):
        setattr(root, attr, placeholder)
    root.SolverConfig = None
    sys.modules[name] = root
    return root
