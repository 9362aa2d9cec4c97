"""The reference's end-to-end acceptance criteria (reference
pkg/tests/test_acceptance.py, criteria 05-11), rerun on the GPU path through
this package's public API, on the same problems (three spheres on the x axis,
refinement 1 / 2, ACA 1e-8) with the same bounds:

  05  every scheme vs the dense matvec oracle: <= 1e-6 (FP64 payloads) / 1e-4
  06  threaded matvec vs sequential: <= 1e-12 (the device result is bitwise)
  07  all eleven schemes converge at N=960 (tol 1e-6): true residual < 1e-6,
      <= 200 iterations
  08  the reference's iteration-count orderings
  09  payload byte identities
  10  FP32 storage faster than FP64 at N=10,240 (soft in the reference: a
      warning; here the device result is asserted)
  11  the m1-double iterative solution vs dense LU: <= 1e-5
"""

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ALL_SCHEMES = ["m1-double", "m1-single", "m1-mixed",
               "m2-double", "m2-single", "m2-mixed",
               "m3:c=-1", "m3:c=1", "m3:c=3", "m3:c=5", "m3:c=7"]


def _pure_fp64(sh) -> bool:
    pk = sh.packed
    return pk.buf32.size == 0


@pytest.fixture(scope="module")
def problem240(hx):
    mesh = hx.build_sphere_mesh(hx.axis_centers(3, 3.0), refinement=1)
    h = hx.build_hmatrix(mesh, aca_tol=1e-8)
    return mesh, h, hx.assemble_dense(mesh)


@pytest.fixture(scope="module")
def problem960(hx):
    mesh = hx.build_sphere_mesh(hx.axis_centers(3, 3.0), refinement=2)
    h = hx.build_hmatrix(mesh, aca_tol=1e-8)
    return mesh, h, hx.right_hand_side(mesh)


@pytest.fixture(scope="module")
def reports960(hx, problem960):
    _, h, b = problem960
    cfg = hx.SolverConfig(tol=1e-6, max_iter=200)
    return {name: hx.bicgstab(hx.prepare_scheme(h, name), h, b, cfg)[1] for name in ALL_SCHEMES}


def test_criterion_05_matvec_oracle(hx, problem240):
    _, h, a = problem240
    x = np.random.default_rng(42).uniform(-1.0, 1.0, h.n)
    ref = a @ x
    scale = np.max(np.abs(ref))
    for name in ALL_SCHEMES:
        sh = hx.prepare_scheme(h, name)
        err = np.max(np.abs(hx.matvec(sh, x) - ref)) / scale
        bound = 1e-6 if _pure_fp64(sh) else 1e-4
        assert err <= bound, f"{name}: {err:.3e} > {bound:.0e}"


def test_criterion_06_thread_equivalence(hx, problem240):
    _, h, _ = problem240
    x = np.random.default_rng(43).uniform(-1.0, 1.0, h.n)
    for name in ALL_SCHEMES:
        sh = hx.prepare_scheme(h, name)
        y1 = hx.matvec_threaded(sh, x, threads=1)
        for threads in (2, 4, 8):
            assert np.array_equal(hx.matvec_threaded(sh, x, threads=threads), y1), name


def test_criterion_07_solver_convergence(reports960):
    for name, rep in reports960.items():
        assert rep.converged, f"{name} did not converge"
        assert rep.true_residual < 1e-6, f"{name}: {rep.true_residual:.3e}"
        assert rep.iterations <= 200


def test_criterion_08_iteration_orderings(reports960):
    it = {name: rep.iterations for name, rep in reports960.items()}
    assert it["m1-double"] <= it["m1-mixed"] + 2
    assert it["m1-mixed"] + 2 <= it["m1-single"] + 4
    assert it["m2-double"] <= it["m1-double"] + 2
    assert it["m2-mixed"] <= it["m1-single"]
    assert it["m3:c=7"] <= it["m3:c=1"] + 2


def test_criterion_09_storage_identities(hx, problem960):
    _, h, _ = problem960
    m1d = hx.payload_bytes(hx.prepare_scheme(h, "m1-double"))
    m1s = hx.payload_bytes(hx.prepare_scheme(h, "m1-single"))
    m2d = hx.payload_bytes(hx.prepare_scheme(h, "m2-double"))
    assert m1s * 2 == m1d
    assert m2d - m1d == 8 * int(h.packed.ranks[h.packed.kinds == 1].sum())


def test_criterion_10_fp32_storage_is_faster(hx, monkeypatch):
    """Reference: N = 2 x 20 x 4^4, m1-single should take <= 0.95 of
    m1-double's time (soft there).  On the device the product is
    bandwidth-bound, so halving the stored bytes must show -- with the FP32
    products as one chain per (row, block) (HMX_FP32_ORDER=chain).  The
    default order, SGEMV's own (bitwise the reference's FP32 products), reads
    each 4096-column block of a row as two sequential FMA chains and is
    latency-bound at this size; its time is reported, not asserted
    (FP32 accumulation order)."""
    from paper_1911_00093_b200.matvec import get_plan

    mesh = hx.build_sphere_mesh(hx.axis_centers(2, 3.0), refinement=4)
    h = hx.build_hmatrix(mesh, leaf_size=64)
    t = {"m1-single (sgemv order)": get_plan(hx.prepare_scheme(h, "m1-single")).bench(5, 50)["ms"]}
    monkeypatch.setenv("HMX_FP32_ORDER", "chain")
    for name in ("m1-double", "m1-single"):
        plan = get_plan(hx.prepare_scheme(h, name))
        t[name] = plan.bench(5, 50)["ms"]
    assert t["m1-single"] <= 0.95 * t["m1-double"], t


def test_criterion_11_solver_oracle(hx, problem960):
    mesh, h, b = problem960
    x_lu = np.linalg.solve(hx.assemble_dense(mesh), b)
    x_it, rep = hx.bicgstab(hx.prepare_scheme(h, "m1-double"), h, b,
                            hx.SolverConfig(tol=1e-8, max_iter=200))
    assert rep.converged
    assert np.linalg.norm(x_it - x_lu) / np.linalg.norm(x_lu) <= 1e-5
