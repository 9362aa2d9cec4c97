"""prepare_scheme on the GPU.

`prepare_scheme_device(h, scheme)` has the contract of
`prepare_scheme(h, scheme)` (reference precision.py:256-329) but runs the
scaling (scale_decompose, :121-141), the Method-3 split (split_indices,
:144-162) and the FP32 casts (_cast_fp32, :241-253) on the device, from FP64
masters uploaded once per H-matrix (`get_master`).  Sweeping schemes or
Method-3 cut-offs c therefore moves no payload over the host link: each
scheme costs the device pack plus the host flattener's layout pass.

The device plan is bit-identical to the plan of the host-prepared payloads
(tests/test_gpu_prepare.py), so every matvec/solver result is too.  Host
payload arrays are produced lazily (by the host preparation) only if a caller
asks for `payloads`/`packed`.
"""

from __future__ import annotations

import threading

import numpy as np

from . import _gpu
from .matvec import default_device
from .precision import (_F32_MAX, SchemeHMatrix, _as_scheme, _block_table, _pack_foreign,
                        _split_factor, _where, prepare_scheme)

__all__ = ["get_master", "prepare_scheme_device", "DeviceSchemeHMatrix"]

_lock = threading.Lock()


def get_master(h, device: int | None = None) -> _gpu.Master:
    """Device-resident FP64 masters of `h`, uploaded on first use and cached."""
    dev = default_device() if device is None else device
    m = getattr(h, "_hmx_gpu_master", None)
    if m is not None and m.device == dev and not m.closed:
        return m
    with _lock:
        m = getattr(h, "_hmx_gpu_master", None)
        if m is None or m.device != dev or m.closed:
            pm = h.packed if hasattr(h, "packed") else _pack_foreign(h)
            m = _gpu.Master(pm, _block_table(h), np.asarray(h.permutation), int(h.n), device=dev)
            try:
                object.__setattr__(h, "_hmx_gpu_master", m)
            except Exception:
                pass
    return m


class DeviceSchemeHMatrix(SchemeHMatrix):
    """SchemeHMatrix whose payloads live only on the device; host payloads are
    prepared on demand."""

    def __init__(self, base, scheme, payload_bytes: int, underflow_count: int, fp32_ranks: int):
        self.base = base
        self.scheme = _as_scheme(scheme)
        self._payloads = None
        self._packed = None
        self.payload_bytes = int(payload_bytes)
        self.underflow_count = int(underflow_count)
        self.fp32_ranks = int(fp32_ranks)

    @property
    def packed(self):
        if self._packed is None:
            self._packed = prepare_scheme(self.base, self.scheme).packed
        return self._packed

    @property
    def payloads(self) -> list:
        if self._payloads is None:
            t = self.base.partition.table
            self._payloads = [self.packed.payload(t[k], k) for k in range(t.shape[0])]
        return self._payloads


def _overflow_message(h, k: int) -> str:
    """The reference's OverflowError text for block k (precision.py:246-250):
    the first array cast (dense values, else U, else Vt) that overflows."""
    pm = h.packed if hasattr(h, "packed") else _pack_foreign(h)
    t = _block_table(h)
    m, n = int(t[k, 1] - t[k, 0]), int(t[k, 3] - t[k, 2])
    o = int(pm.offsets[k])
    if pm.kinds[k] == 0:
        arrays = [pm.data[o:o + m * n]]
    else:
        r = int(pm.ranks[k])
        arrays = [pm.data[o:o + m * r], pm.data[o + m * r:o + r * (m + n)]]
    arr = next((a for a in arrays if np.any(np.abs(a) > _F32_MAX)), arrays[-1])
    peak = float(np.max(np.abs(arr)))
    return f"FP32 overflow while casting {_where(t, k)}: |value| up to {peak:.6g} exceeds {_F32_MAX:.6g}"


def prepare_scheme_device(h, scheme, device: int | None = None) -> DeviceSchemeHMatrix:
    """prepare_scheme(h, scheme) computed on the device; the returned object's
    device plan is ready (matvec/bicgstab use it directly)."""
    scheme = _as_scheme(scheme)
    dev = default_device() if device is None else device
    master = get_master(h, dev)
    factor = _split_factor(scheme.c) if scheme.method == 3 else 0.0
    try:
        plan, info = _gpu.Plan.prepared(master, scheme.label, factor)
    except OverflowError as e:
        k = int(str(e).split()[-1])
        raise OverflowError(_overflow_message(h, k)) from None
    sh = DeviceSchemeHMatrix(h, scheme, info["payload_bytes"], info["underflow_count"],
                             info["fp32_ranks"])
    # cache the plan where get_plan looks for it (m1-double plans are shared
    # with the true-residual operator on the masters)
    if scheme.label == "m1-double":
        prev = getattr(h, "_hmx_gpu_plan64", None)
        if prev is not None and prev.device == dev and not prev.closed:
            plan.close()
            plan = prev
        else:
            object.__setattr__(h, "_hmx_gpu_plan64", plan)
    else:
        sh._hmx_gpu_plan = plan
    return sh
