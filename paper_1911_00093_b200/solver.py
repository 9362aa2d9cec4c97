"""Drop-in BiCG-STAB on the B200 (reference pkg/src/hmx/solver.py).

Same signatures, dataclasses and semantics as the reference:
`bicgstab(sh, h64, b, cfg)` solves from x0 = 0 with the scheme's operator,
declares convergence only when the recurrence residual is below `tol` AND an
FP64 true residual (m1-double operator of `h64`) confirms it, stops without
further iterations when the confirmation fails, and reports breakdowns in
`SolverReport.breakdown` instead of raising.  The iteration runs entirely in
libhmx_gpu.so (hmx_bicgstab).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _gpu
from .matvec import get_plan, get_plan64, raise_nonfinite

__all__ = ["SolverConfig", "SolverReport", "bicgstab", "true_residual"]


@dataclass
class SolverConfig:
    """BiCG-STAB stopping rule and iteration cap (reference solver.py:30-43)."""
    tol: float = 1e-6
    max_iter: int = 1000
    threads: int = 1

    def __post_init__(self):
        if not (self.tol > 0.0):
            raise ValueError("tol must be positive")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")


@dataclass
class SolverReport:
    """Outcome of one solve (reference solver.py:45-54) plus device timings."""
    scheme: str
    converged: bool
    iterations: int
    residual_history: list = field(default_factory=list)
    true_residual: float | None = None
    wall_time_s: float = 0.0
    breakdown: str | None = None
    device_time_s: float = 0.0
    matvecs: int = 0


def true_residual(h64, x, b) -> float:
    """||b - A x|| / ||b|| with the FP64 operator (solver.py:56-65)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = h64.n
    # the reference raises here too: matvec's shape check (matvec.py:115-116),
    # then numpy broadcasting of b - A x
    if x.shape != (n,):
        raise ValueError(f"vector shape {x.shape} does not match matrix size {n}")
    if b.shape in ((), (1,)):
        # numpy broadcasts a scalar-like b in `b - A x`, while ||b|| stays the
        # norm of the scalar: ||b_full|| = sqrt(n) |b|
        return true_residual(h64, x, np.full(n, float(b.reshape(-1)[0]))) * float(np.sqrt(n))
    if b.shape != (n,):
        raise ValueError(f"operands could not be broadcast together with shapes {b.shape} ({n},)")
    plan = get_plan64(h64)
    out = ctypes.c_double(0.0)
    rc = plan._lib.hmx_true_residual(plan.handle, x.ctypes.data, b.ctypes.data,
                                     ctypes.byref(out))
    if rc == _gpu.HMX_ERR_NONFINITE:
        raise_nonfinite(plan, h64)
    _gpu.check(rc, "hmx_true_residual")
    return float(out.value)


def _breakdown_message(code: int, value: float, it: int) -> str | None:
    if code == 1:
        return f"rho vanished ({value:.3e}) at iteration {it}"
    if code == 2:
        return f"shadow projection vanished ({value:.3e}) at iteration {it}"
    if code == 3:
        return f"stabilization direction vanished at iteration {it}"
    if code == 4:
        return f"omega vanished ({value:.3e}) at iteration {it}"
    return None


def bicgstab(sh, h64, b, cfg: SolverConfig | None = None):
    """Solve A x = b; returns (x, SolverReport) (solver.py:68-168)."""
    if cfg is None:
        cfg = SolverConfig()
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = sh.n
    if b.shape != (n,):
        raise ValueError(f"right-hand side shape {b.shape} does not match {n}")
    plan = get_plan(sh)
    plan64 = get_plan64(h64, plan.device)
    x = np.empty(n, dtype=np.float64)
    hist = np.zeros(cfg.max_iter + 2, dtype=np.float64)
    rep = _gpu.SolveReport()
    t0 = time.perf_counter()
    rc = plan._lib.hmx_bicgstab(plan.handle, plan64.handle, b.ctypes.data, float(cfg.tol),
                                int(cfg.max_iter), x.ctypes.data, hist.ctypes.data,
                                ctypes.byref(rep))
    wall = time.perf_counter() - t0
    if rc == _gpu.HMX_ERR_NONFINITE:
        if plan.nonfinite_block() >= 0 or plan64 is plan:
            raise_nonfinite(plan, sh.base)
        raise_nonfinite(plan64, h64)
    _gpu.check(rc, "hmx_bicgstab")
    label = sh.scheme.label if not isinstance(sh.scheme, str) else sh.scheme
    return x, SolverReport(
        scheme=label,
        converged=bool(rep.converged),
        iterations=int(rep.iterations),
        residual_history=[float(v) for v in hist[:rep.history_len]],
        true_residual=float(rep.true_residual) if rep.has_true_residual else None,
        wall_time_s=wall,
        breakdown=_breakdown_message(rep.breakdown, rep.breakdown_value,
                                     rep.breakdown_iteration),
        device_time_s=rep.device_ms / 1e3,
        matvecs=int(rep.matvecs),
    )
