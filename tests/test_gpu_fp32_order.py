"""FP32 accumulation order of the FP32-accumulated items (m1-single, m1-mixed
U slabs, m2-single dense blocks; reference matvec.py:57, :73 -- numpy
`A32 @ x32`, i.e. OpenBLAS SGEMV).

The GPU evaluates every such item in SGEMV's own summation tree (stage 2:
chain_lane / chain_quad in csrc/hmx_kernels.cu, four rows per lane from a
per-lane cp.async FIFO; stage 1 of m1-single: s1_exact_kernel, one row per
thread over the csrc/hmx_internal.cuh chunk_off layout).  Checked here:
  * CPU: the kernel's order, modelled in tools/fp32_accum_emulation.py
    (sgemv_rows: SGEMV's 16/8/4-row kernels and its 2- and 1-row remainder
    kernels), reproduces the reference's products bitwise
    (tests/golden/fp32_order.npz, made by numpy in the build container) for
    every width 1..48 and row counts 8, 40, 30 and 5;
  * GPU: block-diagonal m2-single matrices put one item per row segment, so
    y is exactly the widened FP32 item value: bitwise the model and bitwise
    the reference's own numbers;
  * GPU: the operator error ||y - y64|| of m1-single / m1-mixed / m2-single is
    within 5 % of the reference's ||y_ref - y64|| on the golden fixtures and
    BASELINE configs 1-2 (VERDICT r1 "Next" item 2).
"""

import numpy as np
import pytest

from golden_util import GOLDEN, config1_hmatrix, hmatrix_from_fixture, load

# row counts: 8 and 40 (SGEMV's 8-row kernel), 30 (16 + 8 + 4 + the 2-row
# remainder kernel) and 5 (4-row kernel + the 1-row remainder kernel)
ROWS = (8, 40, 30, 5)


def fixture():
    return dict(np.load(GOLDEN / "fp32_order.npz"))


def test_model_reproduces_reference_products():
    from tools.fp32_accum_emulation import sgemv_rows
    f = fixture()
    for m in ROWS:
        for n in range(1, 49):
            a32 = f[f"a/{m}/{n}"].astype(np.float32)
            x32 = f[f"x/{m}/{n}"].astype(np.float32)
            assert np.array_equal(sgemv_rows(a32, x32), f[f"y/{m}/{n}"]), (m, n)


def test_chunk_layout_is_a_permutation():
    """chunk_off (csrc/hmx_internal.cuh, ported in the emulation tool) places
    every (row, column) of an item exactly once within rp * n elements, and
    4-column chunks of one row are 16-byte aligned vectors."""
    from tools.fp32_accum_emulation import chain_shaped, chunk_off
    for rp in (4, 20, 40, 64):
        for n in range(1, 70):
            offs = sorted(chunk_off(n, rp, r, k) for r in range(rp) for k in range(n))
            assert offs == list(range(rp * n)), (rp, n)
            if not chain_shaped(n):
                for r in range(rp):
                    for c in range(n // 4):
                        o = chunk_off(n, rp, r, 4 * c)
                        assert o % 4 == 0 and [chunk_off(n, rp, r, 4 * c + j) for j in range(4)] == \
                            [o, o + 1, o + 2, o + 3]


def _block_diagonal(hx, m, widths, values):
    """Blocks (rows [k m, (k+1) m), own column range of width n_k): every
    row segment of the plan holds exactly one item."""
    from paper_1911_00093_b200.partition import ClusterNode, ClusterTree
    nrow, ncol = m * len(widths), int(sum(widths))
    n = max(nrow, ncol)
    blocks, pays, c0 = [], [], 0
    for k, (w, a) in enumerate(zip(widths, values)):
        blocks.append(hx.Block(k * m, (k + 1) * m, c0, c0 + w, False))
        pays.append(hx.DenseBlockF64(a))
        c0 += w
    node = ClusterNode(0, n, np.zeros(3), np.zeros(3))
    tree = ClusterTree(root=node, permutation=np.arange(n), leaf_size=n)
    part = hx.BlockPartition(blocks=blocks, n=n, tree=tree)
    return hx.HMatrixF64(partition=part, payloads=pays), n


@pytest.mark.gpu
@pytest.mark.parametrize("m", ROWS)
def test_gpu_items_bitwise_sgemv_order(hx, m):
    from tools.fp32_accum_emulation import sgemv_rows
    f = fixture()
    widths = list(range(1, 49))
    h, n = _block_diagonal(hx, m, widths, [f[f"a/{m}/{w}"] for w in widths])
    x = np.zeros(n)
    c0 = 0
    for w in widths:
        x[c0:c0 + w] = f[f"x/{m}/{w}"]
        c0 += w
    y = hx.matvec(hx.prepare_scheme(h, "m2-single"), x)
    c0 = 0
    for k, w in enumerate(widths):
        got = y[k * m:(k + 1) * m]
        a32 = f[f"a/{m}/{w}"].astype(np.float32)
        x32 = x[c0:c0 + w].astype(np.float32)
        model = sgemv_rows(a32, x32).astype(np.float64)
        assert np.array_equal(got, model), (m, w, got - model)
        assert np.array_equal(got, f[f"y/{m}/{w}"].astype(np.float64)), (m, w)
        c0 += w


def _error_ratio(y, yref, y64):
    return float(np.linalg.norm(y - y64) / np.linalg.norm(yref - y64))


FP32_ACC = ["m1-single", "m1-mixed", "m2-single"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["ref60", "ref240", "ref240_aca4", "config1"])
def test_gpu_fp32_error_vs_reference_fixtures(hx, name):
    arr, _ = load(name)
    h = config1_hmatrix()[1] if name == "config1" else hmatrix_from_fixture(arr)
    y64 = arr["y/m1-double"]
    for s in FP32_ACC:
        y = hx.matvec(hx.prepare_scheme(h, s), arr["x"])
        r = _error_ratio(y, arr[f"y/{s}"], y64)
        assert r <= 1.05, (name, s, r)


@pytest.mark.gpu
def test_gpu_fp32_error_vs_oracle_config2(hx, orc):
    mesh = hx.jittered_sphere_mesh(5, seed=42)
    h = hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32, eta=2.0)
    x = np.random.default_rng(42).uniform(-1.0, 1.0, mesh.n)
    y64 = orc.matvec(hx.prepare_scheme(h, "m1-double"), x)
    for s in FP32_ACC:
        sh = hx.prepare_scheme(h, s)
        r = _error_ratio(hx.matvec(sh, x), orc.matvec(sh, x), y64)
        assert r <= 1.05, (s, r)


@pytest.mark.gpu
def test_gpu_all_lanes_mode(hx, monkeypatch):
    """HMX_ALL_LANES=1 (an experiment kept in the tree):
    the widened items run on the chain lanes too.  The FP32-accumulated item
    values are the same numbers, so only the FP64 order of the row sums moves."""
    arr, _ = load("ref240")
    h = hmatrix_from_fixture(arr)
    y64 = arr["y/m1-double"]
    schemes = ("m1-mixed", "m2-single")
    base = {s: hx.matvec(hx.prepare_scheme(h, s), arr["x"]) for s in schemes}
    monkeypatch.setenv("HMX_ALL_LANES", "1")
    for s in schemes:
        y = hx.matvec(hx.prepare_scheme(h, s), arr["x"])
        assert _error_ratio(y, arr[f"y/{s}"], y64) <= 1.05, s
        assert np.max(np.abs(y - base[s])) <= 1e-13 * np.max(np.abs(base[s])), s


@pytest.mark.gpu
def test_gpu_fp32_chain_order_option(hx, orc, monkeypatch):
    """HMX_FP32_ORDER=chain (HMX_PLAN_FP32_CHAIN): the faster one-chain-per-
    (row, block) order -- within the FP32 tolerance of the reference, bit-
    reproducible, and not the SGEMV order (the default)."""
    arr, _ = load("ref240")
    h = hmatrix_from_fixture(arr)
    x = arr["x"]
    exact = {s: hx.matvec(hx.prepare_scheme(h, s), x) for s in FP32_ACC}
    monkeypatch.setenv("HMX_FP32_ORDER", "chain")
    for s in FP32_ACC:
        sh = hx.prepare_scheme(h, s)          # a fresh object: a fresh plan
        y = hx.matvec(sh, x)
        ref = arr[f"y/{s}"]
        assert np.max(np.abs(y - ref)) <= 1e-5 * np.max(np.abs(ref)), s
        assert np.array_equal(y, hx.matvec(sh, x))
        assert not np.array_equal(y, exact[s]), s
