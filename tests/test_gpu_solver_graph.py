"""The graph-resident BiCG-STAB loop (one CUDA graph launch per solve: a
WHILE conditional node around one captured iteration) against the batched
stream path (HMX_SOLVER_NO_GRAPH=1): same kernels, so bit-identical results,
including breakdown and max_iter outcomes."""

import os

import numpy as np
import pytest

from golden_util import config1_hmatrix

pytestmark = pytest.mark.gpu


def _solve(hx, sh, h, b, cfg, graph):
    if graph:
        os.environ.pop("HMX_SOLVER_NO_GRAPH", None)
    else:
        os.environ["HMX_SOLVER_NO_GRAPH"] = "1"
    try:
        return hx.bicgstab(sh, h, b, cfg)
    finally:
        os.environ.pop("HMX_SOLVER_NO_GRAPH", None)


@pytest.mark.parametrize("scheme", ["m1-double", "m1-mixed", "m2-single", "m3:c=3"])
@pytest.mark.parametrize("max_iter", [1, 7, 1000])
def test_graph_loop_matches_batched_path(hx, scheme, max_iter):
    _, h = config1_hmatrix()
    b = np.random.default_rng(11).uniform(-1.0, 1.0, h.n)
    sh = hx.prepare_scheme(h, scheme)
    cfg = hx.SolverConfig(tol=1e-8, max_iter=max_iter)
    xg, rg = _solve(hx, sh, h, b, cfg, True)
    xb, rb = _solve(hx, sh, h, b, cfg, False)
    assert np.array_equal(xg, xb)
    assert rg.iterations == rb.iterations and rg.converged == rb.converged
    assert rg.residual_history == rb.residual_history
    assert rg.breakdown == rb.breakdown and rg.matvecs == rb.matvecs
    if max_iter < 10:
        assert rg.iterations == max_iter and not rg.converged


def test_graph_loop_reused_across_solves_and_tolerances(hx):
    _, h = config1_hmatrix()
    sh = hx.prepare_scheme(h, "m2-mixed")
    b = np.random.default_rng(2).uniform(-1.0, 1.0, h.n)
    for tol in (1e-4, 1e-8, 1e-6):
        xg, rg = _solve(hx, sh, h, b, hx.SolverConfig(tol=tol), True)
        xb, rb = _solve(hx, sh, h, b, hx.SolverConfig(tol=tol), False)
        assert rg.iterations == rb.iterations and np.array_equal(xg, xb)


def test_graph_loop_one_step_exit(hx):
    # identity operator: exact after one step, the loop stops on the early
    # |s| exit inside its first iteration
    from paper_1911_00093_b200.compress import HMatrixF64, PackedMaster
    from paper_1911_00093_b200.partition import BlockPartition, ClusterNode, ClusterTree
    n = 8
    perm = np.arange(n, dtype=np.int64)
    perm.setflags(write=False)
    tree = ClusterTree(root=ClusterNode(0, n, np.zeros(3), np.zeros(3)), permutation=perm, leaf_size=n)
    table = np.array([[0, n, 0, n, 0]], dtype=np.int64)
    part = BlockPartition(n=n, tree=tree, table=table)
    h = HMatrixF64(part, packed=PackedMaster(np.eye(n).ravel(), np.array([0], np.int32),
                                            np.array([0], np.int64), np.array([0], np.int64)))
    b = np.arange(1.0, n + 1)
    sh = hx.prepare_scheme(h, "m1-double")
    xg, rg = _solve(hx, sh, h, b, hx.SolverConfig(tol=1e-8), True)
    xb, rb = _solve(hx, sh, h, b, hx.SolverConfig(tol=1e-8), False)
    assert np.array_equal(xg, xb) and np.allclose(xg, b)
    assert rg.iterations == rb.iterations == 1 and rg.converged
