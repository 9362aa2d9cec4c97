"""The reference's matvec and solver unit tests (reference
pkg/tests/test_matvec.py and test_solver.py) that concern the operator and
the solver, rerun on the GPU path through this package's API with the same
problems and bounds.  (The reference's per-block numpy helpers
block_mul_dense/lowrank and its host-only checks are covered by the CPU
tests; the golden-fixture and bitwise-invariant tests live in
test_gpu_parity.py.)"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def dense_as_hmatrix(hx, values):
    """One dense block covering the whole matrix (the reference tests'
    dense_as_hmatrix / identity_hmatrix)."""
    from paper_1911_00093_b200.partition import ClusterNode, ClusterTree
    values = np.asarray(values, dtype=np.float64)
    n = values.shape[0]
    node = ClusterNode(0, n, np.zeros(3), np.zeros(3))
    tree = ClusterTree(root=node, permutation=np.arange(n), leaf_size=n)
    part = hx.BlockPartition(blocks=[hx.Block(0, n, 0, n, False)], n=n, tree=tree)
    return hx.HMatrixF64(partition=part, payloads=[hx.DenseBlockF64(values)])


@pytest.fixture(scope="module")
def problem(hx):
    """test_solver.py / test_matvec.py `problem`: three spheres, refinement 1."""
    mesh = hx.build_sphere_mesh(hx.axis_centers(3, 3.0), refinement=1)
    h = hx.build_hmatrix(mesh)
    return mesh, h, hx.right_hand_side(mesh), np.random.default_rng(41).uniform(-1, 1, mesh.n)


# ---------------------------------------------------------------- solver (test_solver.py)

def test_identity_converges_immediately(hx):
    h = dense_as_hmatrix(hx, np.eye(8))
    b = np.arange(1.0, 9.0)
    x, report = hx.bicgstab(hx.prepare_scheme(h, "m1-double"), h, b)
    assert report.converged and report.iterations <= 1
    assert np.allclose(x, b, rtol=1e-12)
    assert report.residual_history[0] == 1.0
    assert report.true_residual < 1e-12


def test_small_dense_system(hx):
    rng = np.random.default_rng(51)
    a = rng.normal(size=(20, 20)) + 20.0 * np.eye(20)
    h = dense_as_hmatrix(hx, a)
    b = rng.normal(size=20)
    x, report = hx.bicgstab(hx.prepare_scheme(h, "m1-double"), h, b, hx.SolverConfig(tol=1e-10))
    assert report.converged
    assert np.linalg.norm(a @ x - b) / np.linalg.norm(b) < 1e-10


def test_bem_problem_converges(hx, problem):
    _, h, b, _ = problem
    _, report = hx.bicgstab(hx.prepare_scheme(h, "m2-mixed"), h, b)
    assert report.converged and report.true_residual < 1e-6
    assert report.breakdown is None and report.scheme == "m2-mixed"
    assert len(report.residual_history) == report.iterations + 1


def test_threaded_solve_converges_same_problem(hx, problem):
    _, h, b, _ = problem
    sh = hx.prepare_scheme(h, "m1-single")
    x1, r1 = hx.bicgstab(sh, h, b, hx.SolverConfig(threads=1))
    x2, r2 = hx.bicgstab(sh, h, b, hx.SolverConfig(threads=2))
    assert r1.converged and r2.converged
    # the device product does not depend on `threads`: here even bitwise
    assert np.array_equal(x1, x2)


def test_solution_matches_dense_factorization(hx, problem):
    mesh, h, b, _ = problem
    x_ref = np.linalg.solve(hx.assemble_dense(mesh), b)
    x, report = hx.bicgstab(hx.prepare_scheme(h, "m1-double"), h, b,
                            hx.SolverConfig(tol=1e-8, max_iter=200))
    assert report.converged
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-5


def test_lower_precision_never_speeds_convergence(hx, problem):
    _, h, b, _ = problem
    _, rep64 = hx.bicgstab(hx.prepare_scheme(h, "m1-double"), h, b)
    _, rep32 = hx.bicgstab(hx.prepare_scheme(h, "m1-single"), h, b)
    assert rep64.converged and rep32.converged
    assert rep32.iterations >= rep64.iterations


def test_true_residual_at_exact_solution_hits_compression_floor(hx, problem):
    mesh, h, b, _ = problem
    x_ref = np.linalg.solve(hx.assemble_dense(mesh), b)
    assert hx.true_residual(h, x_ref, b) <= 1e-6


def test_true_residual_from_zero_guess_is_one(hx, problem):
    _, h, b, _ = problem
    assert hx.true_residual(h, np.zeros(b.shape[0]), b) == 1.0


def test_true_residual_zero_rhs(hx):
    h = dense_as_hmatrix(hx, np.eye(3))
    assert hx.true_residual(h, np.zeros(3), np.zeros(3)) == 0.0


# ---------------------------------------------------------------- matvec (test_matvec.py)

def test_m3_all_fp32_class_matches_m2_mixed_closely(hx, problem):
    _, h, _, x = problem
    y_mixed = hx.matvec(hx.prepare_scheme(h, "m2-mixed"), x)
    y_m3 = hx.matvec(hx.prepare_scheme(h, "m3:c=-1"), x)
    assert np.max(np.abs(y_mixed - y_m3)) <= 1e-4 * np.max(np.abs(y_mixed))


def test_single_and_mixed_differ_in_accumulation(hx, problem):
    _, h, _, x = problem
    y_single = hx.matvec(hx.prepare_scheme(h, "m1-single"), x)
    y_mixed = hx.matvec(hx.prepare_scheme(h, "m1-mixed"), x)
    diff = np.max(np.abs(y_single - y_mixed))
    assert 0.0 < diff <= 1e-4 * np.max(np.abs(y_mixed))


def test_fullsize_matvec_against_densified_matrix(hx, problem):
    _, h, _, x = problem
    exact = hx.densify(h) @ x
    y = hx.matvec(hx.prepare_scheme(h, "m1-double"), x)
    assert np.max(np.abs(y - exact)) <= 1e-12 * np.max(np.abs(exact))


def test_single_precision_error_is_bounded_and_visible(hx, problem):
    _, h, _, x = problem
    y64 = hx.matvec(hx.prepare_scheme(h, "m1-double"), x)
    y32 = hx.matvec(hx.prepare_scheme(h, "m1-single"), x)
    rel = np.max(np.abs(y32 - y64)) / np.max(np.abs(y64))
    assert 1e-9 < rel <= 1e-5


def test_matvec_accepts_source_vector_and_checks_shape(hx, problem):
    _, h, _, x = problem
    sh = hx.prepare_scheme(h, "m1-single")
    assert np.array_equal(hx.matvec(sh, hx.SourceVector(x)), hx.matvec(sh, x))
    with pytest.raises(ValueError):
        hx.matvec(sh, x[:-1])
    with pytest.raises(ValueError):
        hx.matvec_threaded(sh, x, 0)
