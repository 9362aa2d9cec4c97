"""The drop-in installer (paper_1911_00093_b200/drop_in.py) against the
reference package itself (imported from /root/reference in the build
container; skipped where it is absent, e.g. on the GPU box): every copy of
the operator names is rebound, calls through the reference's own modules
reach the device path (here: no GPU, so they fail loudly instead of
falling back to the CPU), and uninstall restores the reference."""

import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")


@pytest.fixture()
def hmx():
    if not REF.exists():
        pytest.skip("reference package not present")
    sys.path.insert(0, str(REF))
    try:
        import hmx as ref
        yield ref
    finally:
        sys.path.remove(str(REF))


def _cuda():
    from paper_1911_00093_b200 import _gpu
    try:
        return _gpu.device_count() > 0
    except Exception:
        return False


def _mods():
    import importlib
    # (`hmx.matvec` as an attribute is the function: take the modules)
    return [importlib.import_module(m) for m in ("hmx.matvec", "hmx.solver", "hmx.bench", "hmx")]


def test_install_rebinds_every_copy_and_uninstall_restores(hmx):
    import importlib

    from paper_1911_00093_b200 import drop_in
    gm = importlib.import_module("paper_1911_00093_b200.matvec")
    gs = importlib.import_module("paper_1911_00093_b200.solver")

    mods = _mods()
    names = ("matvec", "matvec_threaded", "bicgstab", "true_residual")
    before = [(m, a, getattr(m, a)) for m in mods for a in names if hasattr(m, a)]
    saved = drop_in.install(hmx)
    try:
        for mod in mods:
            assert mod.matvec is gm.matvec and mod.matvec_threaded is gm.matvec_threaded
        assert hmx.bicgstab is gs.bicgstab and mods[1].bicgstab is gs.bicgstab
        assert hmx.true_residual is gs.true_residual and mods[1].true_residual is gs.true_residual
    finally:
        drop_in.uninstall(saved)
    for m, a, f in before:
        assert getattr(m, a) is f


@pytest.mark.skipif(_cuda(), reason="checks the no-GPU behaviour")
def test_reference_objects_reach_the_device_path(hmx):
    """A reference-built SchemeHMatrix through the reference's own module
    reaches the GPU path: without a GPU it raises, it never computes on the
    CPU; shape errors keep the reference's ValueError."""
    from paper_1911_00093_b200 import drop_in
    ref_matvec = _mods()[0]

    mesh = hmx.build_sphere_mesh(hmx.axis_centers(1, 3.0), refinement=0)
    h = hmx.build_hmatrix(mesh)
    sh = hmx.prepare_scheme(h, "m1-double")
    saved = drop_in.install(hmx)
    try:
        with pytest.raises(RuntimeError, match="CUDA"):
            ref_matvec.matvec(sh, np.ones(mesh.n))
        with pytest.raises(RuntimeError, match="CUDA"):
            hmx.bicgstab(sh, h, np.ones(mesh.n))
        with pytest.raises(ValueError):
            ref_matvec.matvec(sh, np.ones(mesh.n + 1))
    finally:
        drop_in.uninstall(saved)
    y = ref_matvec.matvec(sh, np.ones(mesh.n))   # the reference again
    assert y.shape == (mesh.n,)
