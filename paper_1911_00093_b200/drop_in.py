"""Install the B200 path into the reference package `hmx`.

The reference binds its operator names by import (solver.py:21,
bench.py:30, __init__.py:20, :53), so a drop-in rebinds them in every
module that holds a copy:

    import hmx
    from paper_1911_00093_b200 import drop_in
    saved = drop_in.install(hmx)       # hmx.matvec / bicgstab / ... now run on the GPU
    ...
    drop_in.uninstall(saved)

The reference keeps building its own H-matrices and SchemeHMatrix objects;
the GPU functions accept them (duck-typed payload lists are packed once and
the device plan is cached on the object) and return what the reference's
functions return.  The per-block helpers `block_mul_dense/lowrank` are not
rebound (they are numpy utilities the reference's tests pin).
"""

from __future__ import annotations

import importlib

# (the package attribute `matvec` is the function; take the modules)
_gm = importlib.import_module(__package__ + ".matvec")
_gs = importlib.import_module(__package__ + ".solver")

# (module, attribute) -> replacement, for every copy of an operator name
_BINDINGS = (
    ("hmx.matvec", "matvec", _gm.matvec),
    ("hmx.matvec", "matvec_threaded", _gm.matvec_threaded),
    ("hmx.solver", "matvec", _gm.matvec),
    ("hmx.solver", "matvec_threaded", _gm.matvec_threaded),
    ("hmx.solver", "bicgstab", _gs.bicgstab),
    ("hmx.solver", "true_residual", _gs.true_residual),
    ("hmx.bench", "matvec", _gm.matvec),
    ("hmx.bench", "matvec_threaded", _gm.matvec_threaded),
    ("hmx", "matvec", _gm.matvec),
    ("hmx", "matvec_threaded", _gm.matvec_threaded),
    ("hmx", "bicgstab", _gs.bicgstab),
    ("hmx", "true_residual", _gs.true_residual),
)


def install(pkg=None) -> list:
    """Rebind the reference's operator names to the GPU path; returns what
    `uninstall` needs to restore them.  `pkg` is the imported `hmx` package
    (imported by name when omitted)."""
    root = pkg.__name__ if pkg is not None else "hmx"
    saved = []
    for mod_name, attr, fn in _BINDINGS:
        mod = importlib.import_module(mod_name.replace("hmx", root, 1))
        saved.append((mod, attr, getattr(mod, attr)))
        setattr(mod, attr, fn)
    return saved


def uninstall(saved: list) -> None:
    """Restore the bindings `install` replaced."""
    for mod, attr, fn in reversed(saved):
        setattr(mod, attr, fn)
