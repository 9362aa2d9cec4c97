"""GPU H-matrix compression (hmx_master_build: ACA of the admissible blocks
and kernel-entry assembly of the near field on the device, reference
compress.py:79-207, :256-342) against the host builder, which
tests/test_builder_vs_reference.py pins to the reference: the device masters
are bit-identical (kinds, ranks, offsets, every stored value), across mesh
sizes, ACA tolerances (tight ones drive blocks into the host-completed paths:
more than 48 ranks, the rank budget, "ran out of pivot rows" with the
remainder check), max_rank and row-restricted builds."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(h_gpu, h_cpu):
    a, b = h_gpu.packed, h_cpu.packed
    assert np.array_equal(a.kinds, b.kinds)
    assert np.array_equal(a.ranks, b.ranks)
    assert np.array_equal(a.offsets, b.offsets)
    assert a.data.shape == b.data.shape
    assert np.array_equal(a.data.view(np.uint64), b.data.view(np.uint64))
    assert h_gpu.report.to_dict() == h_cpu.report.to_dict()


@pytest.mark.parametrize("level,leaf,tol", [(2, 32, 1e-4), (3, 32, 1e-4), (4, 64, 1e-5),
                                            (3, 32, 1e-10), (4, 32, 1e-13),
                                            (6, 64, 1e-5)])   # 5120 x 5120 blocks: CTA path
def test_device_build_is_bitwise_the_host_build(hx, level, leaf, tol):
    mesh = hx.jittered_sphere_mesh(level, seed=42)
    _same(hx.build_hmatrix(mesh, aca_tol=tol, leaf_size=leaf, device=0),
          hx.build_hmatrix(mesh, aca_tol=tol, leaf_size=leaf))


def test_device_build_three_spheres_max_rank_and_rows(hx):
    mesh = hx.build_sphere_mesh(hx.axis_centers(3, 3.0), refinement=2)
    for kw in ({"aca_tol": 1e-8}, {"aca_tol": 1e-8, "max_rank": 3}, {"aca_tol": 1e-6, "leaf_size": 8}):
        _same(hx.build_hmatrix(mesh, device=0, **kw), hx.build_hmatrix(mesh, **kw))
    h = hx.build_hmatrix(mesh, aca_tol=1e-6)
    n = h.n
    for rows in ((0, n // 3), (n // 3 + 5, n)):
        _same(hx.build_hmatrix(mesh, partition=h.partition, aca_tol=1e-6, rows=rows, device=0),
              hx.build_hmatrix(mesh, partition=h.partition, aca_tol=1e-6, rows=rows))


def test_device_built_masters_serve_device_plans(hx):
    """The masters stay resident: prepare_scheme_device uses them without an
    upload, and the products equal those of the host-built H-matrix."""
    mesh = hx.jittered_sphere_mesh(4, seed=7)
    hg = hx.build_hmatrix(mesh, aca_tol=1e-5, leaf_size=64, device=0)
    hc = hx.build_hmatrix(mesh, aca_tol=1e-5, leaf_size=64)
    assert hx.get_master(hg) is hg._hmx_gpu_master
    x = np.random.default_rng(5).uniform(-1, 1, mesh.n)
    for scheme in ("m1-double", "m2-mixed", "m3:c=2"):
        assert np.array_equal(hx.matvec(hx.prepare_scheme_device(hg, scheme), x),
                              hx.matvec(hx.prepare_scheme(hc, scheme), x))


def test_device_build_matches_dense_assembly(hx):
    """Reference tests/test_compress.py:122-126 on the GPU-compressed matrix:
    relative Frobenius error against the dense kernel matrix <= 1e-6 at ACA
    tolerance 1e-8; payload kinds follow admissibility."""
    mesh = hx.build_sphere_mesh(hx.axis_centers(3, 3.0), refinement=1)
    h = hx.build_hmatrix(mesh, aca_tol=1e-8, device=0)
    a = hx.assemble_dense(mesh)
    assert np.linalg.norm(a - hx.densify(h)) / np.linalg.norm(a) <= 1e-6
    for blk, payload in h.items():
        assert isinstance(payload, hx.LowRankBlockF64) == bool(blk.admissible) or \
            isinstance(payload, hx.DenseBlockF64)
