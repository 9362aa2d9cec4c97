"""GPU vs oracle parity through the public API / C ABI (needs a B200)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCHEMES = ["m1-double", "m1-single", "m1-mixed", "m2-double", "m2-single", "m2-mixed",
           "m3:c=-1", "m3:c=1", "m3:c=3", "m3:c=5", "m3:c=7"]
TIGHT = {"m1-double", "m2-double"}   # all-FP64 payloads


@pytest.fixture(scope="module")
def prob240(hx):
    mesh = hx.build_sphere_mesh(hx.axis_centers(3, 3.0), refinement=1)
    h = hx.build_hmatrix(mesh)
    x = np.random.default_rng(17).uniform(-1.0, 1.0, mesh.n)
    return mesh, h, x


@pytest.fixture(scope="module")
def cfg1(hx):
    mesh = hx.jittered_sphere_mesh(3, seed=42)
    h = hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32, eta=2.0)
    x = np.random.default_rng(42).uniform(-1.0, 1.0, mesh.n)
    return mesh, h, x


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.mark.parametrize("name", SCHEMES)
def test_matvec_vs_oracle_240(hx, orc, prob240, name):
    _, h, x = prob240
    sh = hx.prepare_scheme(h, name)
    y = hx.matvec(sh, x)
    ref = orc.matvec(sh, x)
    tol = 1e-12 if name in TIGHT or name in ("m3:c=7",) else 1e-5
    assert rel(y, ref) <= tol


@pytest.mark.parametrize("name", SCHEMES)
def test_matvec_vs_oracle_config1(hx, orc, cfg1, name):
    _, h, x = cfg1
    sh = hx.prepare_scheme(h, name)
    y = hx.matvec(sh, x)
    ref = orc.matvec(sh, x)
    tol = 1e-12 if name in TIGHT else 1e-5
    assert rel(y, ref) <= tol


def test_solver_config1_m1_double(hx, orc, cfg1):
    mesh, h, _ = cfg1
    b = mesh.centroids[:, 2].copy()
    sh = hx.prepare_scheme(h, "m1-double")
    x, rep = hx.bicgstab(sh, h, b, hx.SolverConfig(tol=1e-8))
    xr, ref = orc.bicgstab(sh, sh, b, tol=1e-8)
    assert rep.converged == ref["converged"]
    assert abs(rep.iterations - ref["iterations"]) <= max(1, ref["iterations"] // 20)
    assert rel(x, xr) <= 1e-6
