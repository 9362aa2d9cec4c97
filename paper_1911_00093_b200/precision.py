"""Precision schemes and per-scheme payload preparation (host, untimed).

Same names, arguments, payload dtypes and error behaviour as the reference's
``hmx.precision`` (reference pkg/src/hmx/precision.py:26-41):

* Method 1 casts the stored factors/blocks (``double``/``single``/``mixed``).
* Method 2 stores unit-scaled factors U', Vt' plus an FP64 diagonal d.
* Method 3 splits every low-rank block's rank columns into an FP64 class
  and an FP32 class by the exponent distance ``c``; dense blocks stay FP64.

Preparation works on the packed master (compress.PackedMaster) and yields a
`PackedScheme`: two flat buffers (float64 / float32) plus per-block offsets.
That is the form the GPU flattener consumes; reference-style per-block
payload objects are numpy views into it, materialised on demand.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native

__all__ = [
    "PrecisionScheme", "parse_scheme", "ScaledLowRank", "SplitLowRank", "DensePayload",
    "FactorPayload", "ScaledPayload", "SchemeHMatrix", "PackedScheme", "scale_decompose",
    "split_indices", "prepare_scheme", "payload_bytes", "storage_table", "SCHEME_NAMES",
]

_VARIANTS = ("double", "single", "mixed")
SCHEME_NAMES = ("m1-double", "m1-single", "m1-mixed", "m2-double", "m2-single", "m2-mixed")


@dataclass(frozen=True)
class PrecisionScheme:
    """(method, variant) for methods 1-2; (3, c) for method 3 (precision.py:52-87)."""

    method: int
    variant: str | None = None
    c: int | None = None

    def __post_init__(self):
        if self.method in (1, 2):
            if self.variant not in _VARIANTS or self.c is not None:
                raise ValueError(f"method {self.method} needs a variant and no c")
        elif self.method == 3:
            if self.variant is not None or not isinstance(self.c, int):
                raise ValueError("method 3 needs an integer c and no variant")
        else:
            raise ValueError(f"unknown method {self.method!r}")

    @property
    def label(self) -> str:
        return f"m3:c={self.c}" if self.method == 3 else f"m{self.method}-{self.variant}"

    @property
    def reads_fp32_source(self) -> bool:
        return self.variant == "single"

    @property
    def casts_dense_fp32(self) -> bool:
        return self.method in (1, 2) and self.variant != "double"


def parse_scheme(name: str) -> PrecisionScheme:
    """'m2-mixed', 'm3:c=-1', ... (precision.py:90-104)."""
    key = name.strip().lower()
    if key in SCHEME_NAMES:
        return PrecisionScheme(int(key[1]), key.split("-", 1)[1])
    if key.startswith("m3:c="):
        try:
            return PrecisionScheme(3, c=int(key[5:]))
        except ValueError:
            raise ValueError(f"bad split parameter in scheme name {name!r}") from None
    raise ValueError(f"unknown scheme {name!r}; expected one of {', '.join(SCHEME_NAMES)} "
                     f"or m3:c=<int>")


def _as_scheme(scheme) -> PrecisionScheme:
    return parse_scheme(scheme) if isinstance(scheme, str) else scheme


@dataclass
class ScaledLowRank:
    """Low-rank factors with per-column scales (reference precision.py:107-119)."""
    u_unit: np.ndarray
    vt_unit: np.ndarray
    diag: np.ndarray


def scale_decompose(u, vt) -> ScaledLowRank:
    """U = U' diag(d) Vt' with unit max-abs columns/rows (precision.py:121-141)."""
    u = np.asarray(u, dtype=np.float64)
    vt = np.asarray(vt, dtype=np.float64)
    if u.ndim != 2 or vt.ndim != 2 or u.shape[1] != vt.shape[0]:
        raise ValueError(f"inconsistent factor shapes {u.shape} x {vt.shape}")
    cmag = np.abs(u).max(axis=0) if u.shape[0] else np.zeros(u.shape[1])
    rmag = np.abs(vt).max(axis=1) if vt.shape[1] else np.zeros(vt.shape[0])
    u_unit = u / np.where(cmag == 0.0, 1.0, cmag)
    vt_unit = vt / np.where(rmag == 0.0, 1.0, rmag)[:, None]
    return ScaledLowRank(np.ascontiguousarray(u_unit), np.ascontiguousarray(vt_unit), cmag * rmag)


def _split_factor(c: int) -> float:
    # evaluated exactly as the reference does (Python float power; raises
    # OverflowError for c <= -309 like the reference)
    return 10.0 ** (-c)


def split_indices(diag, c: int):
    """(idx_fp64, idx_fp32): FP32 iff d_i < max(d) * 10**(-c) (precision.py:144-162)."""
    d = np.asarray(diag, dtype=np.float64)
    if d.ndim != 1:
        raise ValueError("diagonal must be one-dimensional")
    if d.size and np.any(d < 0.0):
        raise ValueError("diagonal entries must be non-negative")
    if d.size == 0:
        none = np.empty(0, dtype=np.intp)
        return none, none
    lo = d < float(np.max(d)) * _split_factor(c)
    return np.flatnonzero(~lo), np.flatnonzero(lo)


@dataclass(slots=True)
class DensePayload:
    """Dense block payload of a prepared scheme (reference precision.py:169-172)."""
    values: np.ndarray


@dataclass(slots=True)
class FactorPayload:
    """Low-rank factors stored in one dtype (reference precision.py:174-180)."""
    u: np.ndarray
    vt: np.ndarray


@dataclass(slots=True)
class ScaledPayload:
    """Scaled low-rank factors (reference precision.py:182-189)."""
    u: np.ndarray
    vt: np.ndarray
    diag: np.ndarray


@dataclass(slots=True)
class SplitLowRank:
    """Method 3 block: leading `c` ranks in FP64, the rest in FP32 (reference precision.py:191-207)."""
    idx_fp64: np.ndarray
    idx_fp32: np.ndarray
    u_hi: np.ndarray
    vt_hi: np.ndarray
    diag_hi: np.ndarray
    u_lo: np.ndarray
    vt_lo: np.ndarray
    diag_lo: np.ndarray


# ---------------------------------------------------------------------------
# packed scheme storage


@dataclass
class PackedScheme:
    """Flat payload storage for one scheme.

    Per block k (`table` row k = rs, re, cs, ce, adm):
      kind[k]   0 dense / 1 low rank
      a_off[k]  dense values (m x n row-major) in buf32 if `a32` else buf64
      hi_off[k] U_hi (m x khi) then Vt_hi (khi x n), in buf32 if `hi32` else buf64
      dhi_off[k] d_hi (khi, buf64) or -1 when the method has no diagonal
      lo_off[k] U_lo (m x klo) then Vt_lo (klo x n) in buf32 (method 3 only)
      dlo_off[k] d_lo (klo, buf64) or -1
      lo_cls    int8 per rank (original order) at roff[k]: 1 = FP32 class (method 3)
    """

    method: int
    a32: bool
    hi32: bool
    buf64: np.ndarray
    buf32: np.ndarray
    kind: np.ndarray
    a_off: np.ndarray
    hi_off: np.ndarray
    khi: np.ndarray
    dhi_off: np.ndarray
    lo_off: np.ndarray
    klo: np.ndarray
    dlo_off: np.ndarray
    roff: np.ndarray
    lo_cls: np.ndarray

    def payload(self, row, k: int):
        m, n = int(row[1] - row[0]), int(row[3] - row[2])
        if self.kind[k] == 2:
            return None  # not built (row-restricted build)
        if self.kind[k] == 0:
            buf = self.buf32 if self.a32 else self.buf64
            o = int(self.a_off[k])
            return DensePayload(buf[o:o + m * n].reshape(m, n))
        hb = self.buf32 if self.hi32 else self.buf64
        kh, o = int(self.khi[k]), int(self.hi_off[k])
        u_hi = hb[o:o + m * kh].reshape(m, kh)
        vt_hi = hb[o + m * kh:o + kh * (m + n)].reshape(kh, n)
        if self.method == 1:
            return FactorPayload(u_hi, vt_hi)
        dh = int(self.dhi_off[k])
        d_hi = self.buf64[dh:dh + kh]
        if self.method == 2:
            return ScaledPayload(u_hi, vt_hi, d_hi)
        kl, lo, dl = int(self.klo[k]), int(self.lo_off[k]), int(self.dlo_off[k])
        cls = self.lo_cls[int(self.roff[k]):int(self.roff[k]) + kh + kl].astype(bool)
        return SplitLowRank(
            idx_fp64=np.flatnonzero(~cls), idx_fp32=np.flatnonzero(cls),
            u_hi=u_hi, vt_hi=vt_hi, diag_hi=d_hi,
            u_lo=self.buf32[lo:lo + m * kl].reshape(m, kl),
            vt_lo=self.buf32[lo + m * kl:lo + kl * (m + n)].reshape(kl, n),
            diag_lo=self.buf64[dl:dl + kl])

    @classmethod
    def from_payloads(cls, scheme, table: np.ndarray, payloads) -> "PackedScheme":
        """Pack reference-style per-block payloads (e.g. from hmx.precision)."""
        scheme = _as_scheme(scheme)
        nb = table.shape[0]
        f64, f32 = [], []
        n64 = n32 = 0

        def put(arr):
            nonlocal n64, n32
            a = np.ascontiguousarray(arr)
            if a.dtype == np.float32:
                f32.append(a.ravel())
                n32 += a.size
                return n32 - a.size, True
            a = a.astype(np.float64, copy=False)
            f64.append(a.ravel())
            n64 += a.size
            return n64 - a.size, False

        z = np.zeros(nb, dtype=np.int64)
        kind, a_off, hi_off, khi = z.astype(np.int32), z.copy(), z.copy(), z.copy()
        dhi_off, lo_off, klo, dlo_off = z - 1, z.copy(), z.copy(), z - 1
        roff, cls_parts, a32, hi32 = z.copy(), [], None, None
        rtot = 0
        for k, p in enumerate(payloads):
            roff[k] = rtot
            if hasattr(p, "values"):
                a_off[k], is32 = put(p.values)
                a32 = is32 if a32 is None else a32
                if a32 != is32:
                    raise TypeError("dense payloads must share one dtype")
                continue
            kind[k] = 1
            if hasattr(p, "u_hi"):
                uh, vh, dh = p.u_hi, p.vt_hi, p.diag_hi
            else:
                uh, vh, dh = p.u, p.vt, getattr(p, "diag", None)
            if uh.dtype != vh.dtype:
                raise TypeError("low-rank factors must share one dtype")
            khi[k] = uh.shape[1]
            o1, is32 = put(uh)
            put(vh)
            hi_off[k] = o1
            hi32 = is32 if hi32 is None else hi32
            if hi32 != is32:
                raise TypeError("low-rank payloads must share one dtype")
            if dh is not None:
                dhi_off[k], _ = put(np.asarray(dh, dtype=np.float64))
            c = np.zeros(khi[k], dtype=np.int8)
            if hasattr(p, "u_lo"):
                klo[k] = p.u_lo.shape[1]
                if klo[k]:
                    lo_off[k], _ = put(np.asarray(p.u_lo, dtype=np.float32))
                    put(np.asarray(p.vt_lo, dtype=np.float32))
                dlo_off[k], _ = put(np.asarray(p.diag_lo, dtype=np.float64))
                c = np.zeros(khi[k] + klo[k], dtype=np.int8)
                c[np.asarray(p.idx_fp32, dtype=np.intp)] = 1
            cls_parts.append(c)
            rtot += c.size
        buf64 = np.concatenate(f64) if f64 else np.zeros(0)
        buf32 = np.concatenate(f32) if f32 else np.zeros(0, dtype=np.float32)
        lo_cls = np.concatenate(cls_parts) if cls_parts else np.zeros(0, dtype=np.int8)
        default32 = scheme.casts_dense_fp32
        return cls(scheme.method, bool(default32 if a32 is None else a32),
                   bool((scheme.variant not in ("double", None)) if hi32 is None else hi32),
                   buf64, buf32, kind, a_off, hi_off, khi, dhi_off, lo_off, klo, dlo_off,
                   roff, lo_cls)


class SchemeHMatrix:
    """An H-matrix prepared for one scheme (precision.py:209-234)."""

    def __init__(self, base, scheme, payloads=None, payload_bytes: int = 0,
                 underflow_count: int = 0, packed: PackedScheme | None = None):
        self.base = base
        self.scheme = _as_scheme(scheme)
        self._payloads = list(payloads) if payloads is not None else None
        self.payload_bytes = int(payload_bytes)
        self.underflow_count = int(underflow_count)
        self._packed = packed
        if payloads is None and packed is None:
            raise ValueError("SchemeHMatrix needs payloads or packed storage")

    @property
    def n(self) -> int:
        return self.base.n

    @property
    def payloads(self) -> list:
        if self._payloads is None:
            t = self.base.partition.table
            self._payloads = [self._packed.payload(t[k], k) for k in range(t.shape[0])]
        return self._payloads

    @property
    def packed(self) -> PackedScheme:
        if self._packed is None:
            self._packed = PackedScheme.from_payloads(self.scheme, _block_table(self.base),
                                                      self._payloads)
        return self._packed

    def items(self):
        return zip(self.base.partition.blocks, self.payloads)


def _block_table(h) -> np.ndarray:
    part = h.partition
    if hasattr(part, "table"):
        return part.table
    return np.array([[b.row_start, b.row_end, b.col_start, b.col_end, int(b.admissible)]
                     for b in part.blocks], dtype=np.int64).reshape(-1, 5)


_F32_TINY = float(np.finfo(np.float32).tiny)
_F32_MAX = float(np.finfo(np.float32).max)


def _where(table, k) -> str:
    r = table[k]
    return f"block {k} rows [{r[0]},{r[1]}) cols [{r[2]},{r[3]})"


def _cast_checked(src64: np.ndarray, table, offsets, kinds, ranks, scheme_name=""):
    """Round-to-nearest FP32 copy of the packed buffer; FP32 overflow raises
    OverflowError naming the first offending block/array, underflow is counted
    (precision.py:241-253)."""
    src64 = np.ascontiguousarray(src64, dtype=np.float64)
    out = np.empty(src64.size, dtype=np.float32)
    lost = ctypes.c_int64(0)
    first = int(_native.host().hb_cast_f32(_native.ptr(src64, _native.c_f64p), src64.size,
                                           _native.ptr(out, _native.c_f32p), ctypes.byref(lost),
                                           _native.host_threads()))
    if first >= 0:
        k = int(np.searchsorted(offsets, first, side="right") - 1)
        m, n = int(table[k, 1] - table[k, 0]), int(table[k, 3] - table[k, 2])
        o = int(offsets[k])
        if kinds[k] == 0:
            arr = src64[o:o + m * n]
        else:
            r = int(ranks[k])
            arr = src64[o:o + m * r] if first < o + m * r else src64[o + m * r:o + r * (m + n)]
        peak = float(np.max(np.abs(arr)))
        raise OverflowError(f"FP32 overflow while casting {_where(table, k)}: |value| up to "
                            f"{peak:.6g} exceeds {_F32_MAX:.6g}")
    return out, int(lost.value)


def prepare_scheme(h, scheme) -> SchemeHMatrix:
    """Build the scheme's payloads once, up front (precision.py:256-329)."""
    scheme = _as_scheme(scheme)
    pm = h.packed if hasattr(h, "packed") else _pack_foreign(h)
    table = _block_table(h)
    nb = table.shape[0]
    m = table[:, 1] - table[:, 0]
    n = table[:, 3] - table[:, 2]
    low = pm.kinds == 1
    r = np.where(low, pm.ranks, 0)
    roff = np.zeros(nb, dtype=np.int64)
    if nb:
        roff[1:] = np.cumsum(r)[:-1]
    rtot = int(r.sum())
    none = np.full(nb, -1, dtype=np.int64)
    zeros = np.zeros(nb, dtype=np.int64)
    lib = _native.host()
    th = _native.host_threads()
    P = _native.ptr
    c_i64, c_i32, c_f64, c_f32, c_i8 = (_native.c_i64p, _native.c_i32p, _native.c_f64p,
                                        _native.c_f32p, _native.c_i8p)
    dense_elems = int(np.sum(np.where(pm.kinds == 0, m * n, 0)))  # kind 2: not built
    lr_elems = int(np.sum(r * (m + n)))
    underflow = 0

    if scheme.method == 1:
        if scheme.variant == "double":
            packed = PackedScheme(1, False, False, pm.data, np.zeros(0, np.float32), pm.kinds,
                                  pm.offsets, pm.offsets, r, none, zeros, zeros, none, roff,
                                  np.zeros(rtot, np.int8))
            nbytes = 8 * (dense_elems + lr_elems)
        else:
            buf32, underflow = _cast_checked(pm.data, table, pm.offsets, pm.kinds, pm.ranks)
            packed = PackedScheme(1, True, True, np.zeros(0), buf32, pm.kinds, pm.offsets,
                                  pm.offsets, r, none, zeros, zeros, none, roff,
                                  np.zeros(rtot, np.int8))
            nbytes = 4 * (dense_elems + lr_elems)
        return SchemeHMatrix(h, scheme, payload_bytes=nbytes, underflow_count=underflow,
                             packed=packed)

    # methods 2 and 3: magnitudes and (for 3) classes
    split = scheme.method == 3
    factor = _split_factor(scheme.c) if split and rtot else 0.0
    diag = np.zeros(rtot, dtype=np.float64)
    cls = np.zeros(rtot, dtype=np.int8)
    nlo = np.zeros(nb, dtype=np.int64)
    m64 = np.ascontiguousarray(m, dtype=np.int64)
    n64 = np.ascontiguousarray(n, dtype=np.int64)
    lib.hb_scale_diag(P(pm.data, c_f64), nb, P(pm.kinds, c_i32), P(pm.ranks, c_i64),
                      P(m64, c_i64), P(n64, c_i64), P(pm.offsets, c_i64), P(roff, c_i64),
                      float(factor), int(split), P(diag, c_f64), P(cls, c_i8), P(nlo, c_i64), th)
    khi = r - nlo
    klo = nlo
    lo_sizes = klo * (m + n)
    lo_off = np.zeros(nb, dtype=np.int64)
    if nb:
        lo_off[1:] = np.cumsum(lo_sizes)[:-1]
    # unit factors written into a copy of the master: U_hi/Vt_hi fit in the
    # block's original slot; the diagonal (reordered hi|lo) is appended
    work = np.empty(pm.data.size + rtot, dtype=np.float64)
    lib.hb_copy_f64(P(pm.data, c_f64), P(work, c_f64), pm.data.size, th)
    dpos = pm.data.size
    buf32_lo = np.zeros(int(lo_sizes.sum()), dtype=np.float32)
    lost = np.zeros(nb, dtype=np.int64)
    lib.hb_scale_fill(P(pm.data, c_f64), nb, P(pm.kinds, c_i32), P(pm.ranks, c_i64),
                      P(m64, c_i64), P(n64, c_i64), P(pm.offsets, c_i64), P(roff, c_i64),
                      P(cls, c_i8), P(pm.offsets, c_i64), P(lo_off, c_i64), P(work, c_f64),
                      P(buf32_lo, c_f32), P(diag, c_f64),
                      P(work[dpos:], c_f64), P(lost, c_i64), th)
    dhi_off = np.where(low, dpos + roff, -1)
    dlo_off = np.where(low, dpos + roff + khi, -1)
    diag_bytes = 8 * rtot

    if scheme.method == 2:
        if scheme.variant == "double":
            packed = PackedScheme(2, False, False, work, np.zeros(0, np.float32), pm.kinds,
                                  pm.offsets, pm.offsets, r, dhi_off, zeros, zeros, none, roff,
                                  cls)
            nbytes = 8 * (dense_elems + lr_elems) + diag_bytes
        else:
            body = work[:dpos]
            buf32, underflow = _cast_checked(body, table, pm.offsets, pm.kinds, pm.ranks)
            packed = PackedScheme(2, True, True, work[dpos:], buf32, pm.kinds, pm.offsets,
                                  pm.offsets, r, dhi_off - dpos, zeros, zeros, none, roff, cls)
            packed.dhi_off = np.where(low, roff, -1)
            nbytes = 4 * (dense_elems + lr_elems) + diag_bytes
        return SchemeHMatrix(h, scheme, payload_bytes=nbytes, underflow_count=underflow,
                             packed=packed)

    # method 3: dense FP64 masters, FP64 class in `work`, FP32 class in buf32_lo
    packed = PackedScheme(3, False, False, work, buf32_lo, pm.kinds, pm.offsets, pm.offsets,
                          khi, dhi_off, lo_off, klo, dlo_off, roff, cls)
    hi_elems = int(np.sum(khi * (m + n)))
    nbytes = 8 * (dense_elems + hi_elems) + 4 * int(lo_sizes.sum()) + diag_bytes
    return SchemeHMatrix(h, scheme, payload_bytes=nbytes, underflow_count=int(lost.sum()),
                         packed=packed)


def _pack_foreign(h):
    """Pack an H-matrix object from another implementation (duck typed)."""
    from .compress import PackedMaster
    return PackedMaster.from_payloads(_block_table(h), h.payloads)


def payload_bytes(sh) -> int:
    """Matrix bytes one matvec traverses under this scheme (precision.py:332-334)."""
    return sh.payload_bytes


def _dense_columns(variant: str) -> dict:
    return {"target": "fp64", "matrix": "fp64" if variant == "double" else "fp32",
            "source": "fp32" if variant == "single" else "fp64"}


def _lowrank_columns(method: int, variant: str) -> dict:
    low = variant != "double"
    return {"intermediate": "fp32" if (method == 1 and low) else "fp64",
            "right_factor": "fp32" if low else "fp64",
            "source": "fp32" if variant == "single" else "fp64",
            "scale": "fp64" if method == 2 else None,
            "target": "fp64",
            "left_factor": "fp32" if low else "fp64"}


def storage_table(scheme) -> dict:
    """Storage precision of every symbol the scheme touches (precision.py:357-381)."""
    scheme = _as_scheme(scheme)
    if scheme.method == 3:
        return {"dense": _dense_columns("double"),
                "lowrank": {"fp64_class": _lowrank_columns(2, "double"),
                            "fp32_class": _lowrank_columns(2, "mixed")},
                "result": "fp64"}
    return {"dense": _dense_columns(scheme.variant),
            "lowrank": _lowrank_columns(scheme.method, scheme.variant), "result": "fp64"}
