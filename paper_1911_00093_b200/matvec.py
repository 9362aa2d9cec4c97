"""Drop-in H-matrix vector product on the B200 (reference pkg/src/hmx/matvec.py).

`matvec(sh, x)` and `matvec_threaded(sh, x, threads)` keep the reference's
signatures, argument meaning and error behaviour:

* `x` is a `SourceVector` or anything `np.asarray(x, float64)` accepts;
  a wrong length raises ValueError (matvec.py:115-116);
* the result is a new float64 array in the original panel order
  (matvec.py:145-147);
* a non-finite result raises FloatingPointError naming the first block
  whose own contribution is non-finite (matvec.py:123-135).

The product runs in libhmx_gpu.so (include/hmx_gpu.h).  `sh` may be this
package's SchemeHMatrix or the reference's (duck typed); the flattened
device plan is built once and cached on the object.
"""

from __future__ import annotations

import os
import threading

import numpy as np

from . import _gpu
from .precision import PackedScheme, parse_scheme, prepare_scheme

__all__ = ["SourceVector", "matvec", "matvec_threaded", "get_plan", "get_plan64",
           "default_device"]

_plan_lock = threading.Lock()


class SourceVector:
    """FP64 source vector with a lazily built FP32 shadow (matvec.py:31-52)."""

    def __init__(self, values):
        master = np.ascontiguousarray(values, dtype=np.float64)
        if master.ndim != 1:
            raise ValueError("source vector must be one-dimensional")
        self.master = master
        self._shadow = None

    @property
    def shadow(self) -> np.ndarray:
        if self._shadow is None:
            self._shadow = self.master.astype(np.float32)
        return self._shadow

    def __len__(self):
        return self.master.shape[0]


def default_device() -> int:
    """CUDA device the matvec path uses (HMX_DEVICE, default 0)."""
    return int(os.environ.get("HMX_DEVICE", "0"))


def _table(h) -> np.ndarray:
    part = h.partition
    if hasattr(part, "table"):
        return part.table
    return np.array([[b.row_start, b.row_end, b.col_start, b.col_end, int(b.admissible)]
                     for b in part.blocks], dtype=np.int64).reshape(-1, 5)


def _packed_of(sh) -> PackedScheme:
    if isinstance(getattr(sh, "_packed", None), PackedScheme) or hasattr(type(sh), "packed"):
        return sh.packed
    return PackedScheme.from_payloads(sh.scheme, _table(sh.base), sh.payloads)


def get_plan(sh, device: int | None = None) -> "_gpu.Plan":
    """Device plan of a prepared scheme, created on first use and cached."""
    dev = default_device() if device is None else device
    scheme = sh.scheme if not isinstance(sh.scheme, str) else parse_scheme(sh.scheme)
    # every m1-double scheme of one H-matrix is the FP64 masters: one device
    # copy, shared with the true-residual operator (get_plan64)
    owner, attr = sh, "_hmx_gpu_plan"
    if scheme.label == "m1-double" and getattr(sh, "base", None) is not None:
        owner, attr = sh.base, "_hmx_gpu_plan64"
    plan = getattr(owner, attr, None)
    if plan is not None and plan.device == dev and not plan.closed:
        return plan
    with _plan_lock:
        plan = getattr(owner, attr, None)
        if plan is None or plan.device != dev or plan.closed:
            plan = _gpu.Plan(_packed_of(sh), _table(sh.base), np.asarray(sh.base.permutation),
                             scheme.label, int(sh.n), device=dev)
            try:
                object.__setattr__(owner, attr, plan)
            except Exception:
                pass
    return plan


def get_plan64(h64, device: int | None = None) -> "_gpu.Plan":
    """m1-double plan of the FP64 masters (true-residual operator)."""
    cached = getattr(h64, "_hmx_gpu_sh64", None)
    if cached is None:
        cached = prepare_scheme(h64, "m1-double")
        try:
            object.__setattr__(h64, "_hmx_gpu_sh64", cached)
        except Exception:
            pass
    return get_plan(cached, device)


def _source(sh, x) -> np.ndarray:
    src = x.master if isinstance(x, SourceVector) else np.asarray(x, dtype=np.float64)
    if src.shape != (sh.n,):
        raise ValueError(f"vector shape {src.shape} does not match matrix size {sh.n}")
    return src


def raise_nonfinite(plan, h) -> None:
    """Raise the reference's FloatingPointError naming the first block with a non-finite contribution (reference matvec.py:123-135)."""
    k = plan.nonfinite_block()
    if k >= 0:
        r = _table(h)[k]
        raise FloatingPointError(
            f"non-finite matvec contribution from block {k} rows "
            f"[{r[0]},{r[1]}) cols [{r[2]},{r[3]})")
    raise FloatingPointError("non-finite matvec result after summation")


def _is_cuda_tensor(x) -> bool:
    t = type(x)
    return t.__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _matvec_cuda_tensor(sh, x):
    """x a CUDA torch tensor: zero-copy in and out, y a new
    float64 CUDA tensor in original order on x's device."""
    import torch
    if x.dim() != 1 or x.shape[0] != sh.n:
        raise ValueError(f"vector shape {tuple(x.shape)} does not match matrix size {sh.n}")
    x = x.to(torch.float64).contiguous()
    plan = get_plan(sh, x.device.index)
    y = torch.empty_like(x)
    torch.cuda.current_stream(x.device).synchronize()  # x complete before the plan's stream reads it
    rc = plan.matvec_device(x.data_ptr(), y.data_ptr(), permuted=False)  # synchronous
    if rc == _gpu.HMX_ERR_NONFINITE:
        raise_nonfinite(plan, sh.base)
    return y


def matvec(sh, x) -> np.ndarray:
    """Multiply the prepared H-matrix by x on the GPU; FP64 result (a numpy
    array, or a CUDA tensor when x is one)."""
    if _is_cuda_tensor(x):
        return _matvec_cuda_tensor(sh, x)
    src = _source(sh, x)
    plan = get_plan(sh)
    y, rc = plan.matvec(src)
    if rc == _gpu.HMX_ERR_NONFINITE:
        raise_nonfinite(plan, sh.base)
    return y


def matvec_threaded(sh, x, threads: int = 1) -> np.ndarray:
    """Same contract as matvec_threaded (matvec.py:161-197).  The device
    product is deterministic and independent of `threads`, so every thread
    count returns the bit-identical vector."""
    if threads < 1:
        raise ValueError("threads must be >= 1")
    return matvec(sh, x)
