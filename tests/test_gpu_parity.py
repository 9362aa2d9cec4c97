"""GPU parity tests (need a B200): the CUDA path through the public API / C ABI
against (1) the reference's own outputs on the reference's own H-matrices
(tests/golden), (2) the CPU oracle on this repo's H-matrices, and (3) the
bitwise invariants the reference's tests pin.

Tolerances (BASELINE.json north_star):
  matvec, all-FP64 payloads      max|dy| <= 1e-12 max|y|
  matvec, FP32-storage payloads  max|dy| <= 1e-5  max|y|
  BiCG-STAB                      iterations inside the reference's own
      reordering envelope (threads 1..8, golden) widened by max(1, 5%);
      `converged` one of the envelope's outcomes.
"""

import numpy as np
import pytest

from golden_util import FP64_ONLY, SCHEMES, config1_hmatrix, hmatrix_from_fixture, load

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def tol_for(scheme):
    return 1e-12 if scheme in FP64_ONLY else 1e-5


def check_solver(rep, ref):
    env = ref["envelope"]
    slack = max(1, int(0.05 * ref["iterations"]))
    assert min(env["iterations"]) - slack <= rep.iterations <= max(env["iterations"]) + slack, \
        (rep.iterations, env["iterations"])
    assert rep.converged in set(env["converged"]), (rep.converged, env["converged"])
    assert len(rep.residual_history) == rep.iterations + 1


# ---------------------------------------------------------------- reference fixtures

@pytest.fixture(scope="module", params=["ref60", "ref240", "ref240_aca4"])
def fixture_case(request):
    arr, meta = load(request.param)
    return request.param, arr, meta, hmatrix_from_fixture(arr)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_matvec_vs_reference_outputs(hx, fixture_case, scheme):
    _, arr, _, h = fixture_case
    y = hx.matvec(hx.prepare_scheme(h, scheme), arr["x"])
    assert rel(y, arr[f"y/{scheme}"]) <= tol_for(scheme)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_bicgstab_vs_reference_envelope(hx, fixture_case, scheme):
    _, arr, meta, h = fixture_case
    x, rep = hx.bicgstab(hx.prepare_scheme(h, scheme), h, arr["b"],
                         hx.SolverConfig(tol=meta["tol"], max_iter=meta["max_iter"]))
    ref = meta["reports"][scheme]
    check_solver(rep, ref)
    if rep.converged:
        assert rep.true_residual < meta["tol"]
        assert rel(x, arr[f"xsol/{scheme}"]) <= 1e-4


def test_nonfinite_names_reference_block(hx):
    arr, meta = load("ref240")
    h = hmatrix_from_fixture(arr)
    bad = arr["x"].copy()
    bad[0] = np.inf
    with pytest.raises(FloatingPointError) as e:
        hx.matvec(hx.prepare_scheme(h, "m1-double"), bad)
    assert str(e.value) == meta["nonfinite_message"]


# ---------------------------------------------------------------- config 1 (this builder)

@pytest.fixture(scope="module")
def cfg1():
    arr, meta = load("config1")
    mesh, h = config1_hmatrix()
    return arr, meta, mesh, h


@pytest.mark.parametrize("scheme", SCHEMES)
def test_config1_matvec(hx, orc, cfg1, scheme):
    arr, _, _, h = cfg1
    sh = hx.prepare_scheme(h, scheme)
    y = hx.matvec(sh, arr["x"])
    assert rel(y, orc.matvec(sh, arr["x"])) <= tol_for(scheme)
    # against the reference's build (ACA ulp differences; FP32 bound for FP32)
    assert rel(y, arr[f"y/{scheme}"]) <= (1e-10 if scheme in FP64_ONLY else 1e-5)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_config1_bicgstab(hx, cfg1, scheme):
    arr, meta, _, h = cfg1
    x, rep = hx.bicgstab(hx.prepare_scheme(h, scheme), h, arr["b"], hx.SolverConfig(tol=1e-8))
    check_solver(rep, meta["reports"][scheme])
    assert rep.true_residual is not None
    assert abs(hx.true_residual(h, x, arr["b"]) - rep.true_residual) <= 1e-12


def test_config1_bicgstab_vs_oracle(hx, orc, cfg1):
    arr, _, _, h = cfg1
    sh = hx.prepare_scheme(h, "m1-double")
    x, rep = hx.bicgstab(sh, h, arr["b"], hx.SolverConfig(tol=1e-8))
    xo, ro = orc.bicgstab(sh, sh, arr["b"], tol=1e-8)
    assert abs(rep.iterations - ro["iterations"]) <= 2
    assert rep.converged == ro["converged"]
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-6


# ---------------------------------------------------------------- bitwise invariants

@pytest.fixture(scope="module")
def prob240(hx):
    mesh = hx.build_sphere_mesh(hx.axis_centers(3, 3.0), refinement=1)
    h = hx.build_hmatrix(mesh)
    return mesh, h, np.random.default_rng(17).uniform(-1.0, 1.0, mesh.n)


def test_m3_empty_fp32_class_is_bitwise_m2_double(hx, prob240):
    _, h, x = prob240
    assert np.array_equal(hx.matvec(hx.prepare_scheme(h, "m2-double"), x),
                          hx.matvec(hx.prepare_scheme(h, "m3:c=400"), x))


def test_repeat_and_thread_counts_bitwise(hx, prob240):
    _, h, x = prob240
    sh = hx.prepare_scheme(h, "m2-mixed")
    y = hx.matvec(sh, x)
    assert np.array_equal(y, hx.matvec(sh, x))
    for t in (1, 2, 8):
        assert np.array_equal(y, hx.matvec_threaded(sh, x, t))
    assert np.array_equal(y, hx.matvec(sh, hx.SourceVector(x)))


def test_results_are_fresh_arrays(hx, prob240):
    """matvec.py:145-147 returns a new array per call; the pinned result pool
    must never hand a live array's buffer to another result."""
    _, h, x = prob240
    sh = hx.prepare_scheme(h, "m1-double")
    ys = [hx.matvec(sh, x) for _ in range(4)]
    ptrs = {y.ctypes.data for y in ys}
    assert len(ptrs) == 4
    ref = ys[0].copy()
    for y in ys:
        assert y.dtype == np.float64 and y.flags.writeable and y.flags.c_contiguous
        assert np.array_equal(y, ref)
    ys[1][:] = 0.0                        # writing one result leaves the others alone
    assert np.array_equal(ys[2], ref)
    del ys
    for _ in range(8):                    # recycled buffers are fully overwritten
        assert np.array_equal(hx.matvec(sh, x), ref)


def test_single_and_mixed_differ_only_at_fp32_level(hx, prob240):
    _, h, x = prob240
    ys = hx.matvec(hx.prepare_scheme(h, "m1-single"), x)
    ym = hx.matvec(hx.prepare_scheme(h, "m1-mixed"), x)
    d = np.max(np.abs(ys - ym))
    assert 0.0 < d <= 1e-4 * np.max(np.abs(ym))


def _single_block(hx, payload, n, admissible):
    from paper_1911_00093_b200.partition import ClusterNode, ClusterTree
    node = ClusterNode(0, n, np.zeros(3), np.zeros(3))
    tree = ClusterTree(root=node, permutation=np.arange(n), leaf_size=n)
    part = hx.BlockPartition(blocks=[hx.Block(0, n, 0, n, admissible)], n=n, tree=tree)
    return hx.HMatrixF64(partition=part, payloads=[payload])


@pytest.mark.parametrize("scheme", SCHEMES)
def test_identity_block(hx, scheme):
    h = _single_block(hx, hx.DenseBlockF64(np.eye(12)), 12, False)
    x = np.linspace(-3.0, 3.0, 12)
    y = hx.matvec(hx.prepare_scheme(h, scheme), x)
    if scheme.endswith("single"):
        assert np.allclose(y, x, rtol=1e-6, atol=0.0)
    else:
        assert np.array_equal(y, x)


def test_hand_evaluated_lowrank_block(hx):
    h = _single_block(hx, hx.LowRankBlockF64(np.ones((2, 1)), np.ones((1, 2))), 2, True)
    assert np.array_equal(hx.matvec(hx.prepare_scheme(h, "m1-double"), np.array([1.0, 2.0])),
                          [3.0, 3.0])


@pytest.mark.parametrize("scheme", ["m1-double", "m1-mixed", "m2-single", "m3:c=1"])
def test_rank_zero_block_contributes_nothing(hx, scheme):
    from paper_1911_00093_b200.partition import ClusterNode, ClusterTree
    n = 8
    node = ClusterNode(0, n, np.zeros(3), np.zeros(3))
    tree = ClusterTree(root=node, permutation=np.arange(n)[::-1].copy(), leaf_size=4)
    blocks = [hx.Block(0, 4, 0, 4, False), hx.Block(0, 4, 4, 8, True),
              hx.Block(4, 8, 0, 4, True), hx.Block(4, 8, 4, 8, False)]
    part = hx.BlockPartition(blocks=blocks, n=n, tree=tree)
    rng = np.random.default_rng(9)
    pays = [hx.DenseBlockF64(rng.normal(size=(4, 4))),
            hx.LowRankBlockF64(np.zeros((4, 0)), np.zeros((0, 4))),
            hx.LowRankBlockF64(rng.normal(size=(4, 2)), rng.normal(size=(2, 4))),
            hx.DenseBlockF64(rng.normal(size=(4, 4)))]
    h = hx.HMatrixF64(partition=part, payloads=pays)
    from oracle import hmx_oracle as orc
    sh = hx.prepare_scheme(h, scheme)
    x = rng.uniform(-1, 1, n)
    assert rel(hx.matvec(sh, x), orc.matvec(sh, x)) <= tol_for(scheme) * 10


@pytest.mark.parametrize("shape", [(1, 0), (200, 0), (300, 150), (3000, 0)])
def test_unusual_shapes(hx, orc, shape):
    """1x1; tall leaves (> 64 rows: row-chunked segments); a rank-150 block
    (stage-1 rank-row splitting); a 3000-column dense block (> 2048 columns:
    column-chunked stage-2 segments with chunk reduction)."""
    n, r = shape
    rng = np.random.default_rng(n + r)
    if r == 0:
        pay = hx.DenseBlockF64(rng.normal(size=(n, n)) + n * np.eye(n))
    else:
        pay = hx.LowRankBlockF64(rng.normal(size=(n, r)), rng.normal(size=(r, n)))
    h = _single_block(hx, pay, n, r > 0)
    x = rng.uniform(-1, 1, n)
    for scheme in ("m1-double", "m1-single", "m1-mixed", "m2-double", "m2-single", "m2-mixed",
                   "m3:c=1", "m3:c=-1"):
        sh = hx.prepare_scheme(h, scheme)
        assert rel(hx.matvec(sh, x), orc.matvec(sh, x)) <= tol_for(scheme) * 10


# ---------------------------------------------------------------- solver semantics

def test_solver_edge_cases(hx):
    h = _single_block(hx, hx.DenseBlockF64(2.0 * np.eye(10)), 10, False)
    sh = hx.prepare_scheme(h, "m1-double")
    x, rep = hx.bicgstab(sh, h, np.ones(10))
    assert rep.converged and np.allclose(x, 0.5, rtol=1e-14)
    x, rep = hx.bicgstab(sh, h, np.zeros(10))
    assert rep.converged and rep.iterations == 0 and rep.residual_history == [0.0]
    assert rep.true_residual == 0.0 and np.all(x == 0.0)
    hz = _single_block(hx, hx.DenseBlockF64(np.zeros((6, 6))), 6, False)
    _, rep = hx.bicgstab(hx.prepare_scheme(hz, "m1-double"), hz, np.ones(6))
    assert not rep.converged and rep.breakdown is not None and "vanished" in rep.breakdown
    hd = _single_block(hx, hx.DenseBlockF64(np.diag([2.0, 4.0])), 2, False)
    assert hx.true_residual(hd, np.array([1.0, 1.0]), np.array([2.0, 4.0])) == 0.0
    assert hx.true_residual(hd, np.array([1.0, 0.5]), np.array([2.0, 4.0])) == \
        pytest.approx(2.0 / np.sqrt(20.0))


def test_solver_max_iter_report(hx, prob240):
    mesh, h, _ = prob240
    b = hx.right_hand_side(mesh)
    _, rep = hx.bicgstab(hx.prepare_scheme(h, "m1-double"), h, b,
                         hx.SolverConfig(tol=1e-15, max_iter=3))
    assert not rep.converged and rep.iterations == 3
    assert len(rep.residual_history) == 4 and rep.true_residual is None
    assert rep.residual_history[0] == 1.0


# ---------------------------------------------------------------- BASELINE config 2 and 4

@pytest.fixture(scope="module")
def cfg2(hx):
    mesh = hx.jittered_sphere_mesh(5, seed=42)
    h = hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32, eta=2.0)
    return mesh, h, np.random.default_rng(42).uniform(-1.0, 1.0, mesh.n)


@pytest.mark.parametrize("scheme", ["m1-double", "m1-single", "m1-mixed", "m2-mixed", "m3:c=3"])
def test_config2_matvec_vs_oracle(hx, orc, cfg2, scheme):
    _, h, x = cfg2
    sh = hx.prepare_scheme(h, scheme)
    assert rel(hx.matvec(sh, x), orc.matvec(sh, x)) <= tol_for(scheme)


@pytest.fixture(scope="module")
def cfg4(hx):
    mesh = hx.jittered_sphere_mesh(7, seed=42)
    h = hx.build_hmatrix(mesh, aca_tol=1e-5, leaf_size=64, eta=2.0)
    return mesh, h, np.random.default_rng(42).uniform(-1.0, 1.0, mesh.n)


@pytest.mark.parametrize("scheme", ["m1-double", "m2-mixed"])
def test_config4_full_size_vs_oracle(hx, orc, cfg4, scheme):
    """N = 327,680 (the north-star size): the full device product against
    the full CPU oracle product, plus linearity and bitwise repeatability."""
    _, h, x = cfg4
    sh = hx.prepare_scheme(h, scheme)
    y = hx.matvec(sh, x)
    assert rel(y, orc.matvec(sh, x)) <= tol_for(scheme)
    assert np.array_equal(y, hx.matvec(sh, x))
    if scheme == "m1-double":
        w = np.random.default_rng(7).uniform(-1.0, 1.0, x.size)
        lhs = hx.matvec(sh, 2.0 * x - 3.0 * w)
        rhs = 2.0 * y - 3.0 * hx.matvec(sh, w)
        assert rel(lhs, rhs) <= 1e-13


def test_config4_solve_confirms_true_residual(hx, cfg4):
    mesh, h, _ = cfg4
    b = mesh.centroids[:, 2].copy()
    x, rep = hx.bicgstab(hx.prepare_scheme(h, "m1-double"), h, b, hx.SolverConfig(tol=1e-8))
    assert rep.breakdown is None and rep.true_residual is not None
    assert abs(hx.true_residual(h, x, b) - rep.true_residual) <= 1e-12
    assert rep.converged == (rep.true_residual < 1e-8)
    # the stop iteration against the reference algorithm's own envelope
    # (golden, threads 1..8): tests/test_gpu_solver_envelope.py
    import json

    from golden_util import GOLDEN
    from test_gpu_solver_envelope import check
    f = GOLDEN / "solver_envelope_config4.json"
    if f.exists():
        check(rep, list(json.loads(f.read_text())["schemes"]["m1-double"].values()))


def test_cuda_tensor_inputs_are_zero_copy(hx, prob240):
    """torch CUDA tensors go in and come out without host copies;
    the values are the host path's, bitwise."""
    import torch
    _, h, x = prob240
    for scheme in ("m1-double", "m2-mixed"):
        sh = hx.prepare_scheme(h, scheme)
        xt = torch.from_numpy(x).cuda()
        yt = hx.matvec(sh, xt)
        assert yt.is_cuda and yt.dtype == torch.float64 and yt.shape == xt.shape
        assert np.array_equal(yt.cpu().numpy(), hx.matvec(sh, x))
    with pytest.raises(ValueError):
        hx.matvec(sh, torch.zeros(h.n + 1, dtype=torch.float64, device="cuda"))
    bad = torch.from_numpy(x).cuda()
    bad[0] = float("inf")
    with pytest.raises(FloatingPointError, match="block"):
        hx.matvec(hx.prepare_scheme(h, "m1-double"), bad)
