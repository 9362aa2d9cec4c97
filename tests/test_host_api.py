"""Host-side interface of the drop-in (schemes, scaling, splitting, payload
preparation, containers) against the reference's semantics
(reference pkg/src/hmx/precision.py, compress.py, partition.py, problem.py).
Known answers are the reference's own worked examples."""

import numpy as np
import pytest


def test_scheme_names_roundtrip(hx):
    for name in ["m1-double", "m1-single", "m1-mixed", "m2-double", "m2-single",
                 "m2-mixed", "m3:c=-1", "m3:c=0", "m3:c=7"]:
        assert hx.parse_scheme(name).label == name
    s = hx.parse_scheme(" M2-Mixed ")
    assert (s.method, s.variant, s.c) == (2, "mixed", None)
    s = hx.parse_scheme("m3:c=4")
    assert (s.method, s.variant, s.c) == (3, None, 4)


@pytest.mark.parametrize("bad", ["m4-double", "m1-half", "m3:c=", "m3:c=x", "m3", "", "double"])
def test_scheme_rejects(hx, bad):
    with pytest.raises(ValueError):
        hx.parse_scheme(bad)


def test_scheme_flags(hx):
    assert hx.parse_scheme("m1-single").reads_fp32_source
    assert hx.parse_scheme("m2-single").reads_fp32_source
    assert not hx.parse_scheme("m2-mixed").reads_fp32_source
    assert not hx.parse_scheme("m3:c=2").reads_fp32_source
    assert hx.parse_scheme("m1-mixed").casts_dense_fp32
    assert not hx.parse_scheme("m3:c=2").casts_dense_fp32
    with pytest.raises(ValueError):
        hx.PrecisionScheme(1)
    with pytest.raises(ValueError):
        hx.PrecisionScheme(3, variant="double")


def test_scale_decompose_worked_example(hx):
    s = hx.scale_decompose(np.array([[3.0, 1.0], [-6.0, 2.0]]),
                           np.array([[2.0, 4.0], [-5.0, 10.0]]))
    assert np.array_equal(s.diag, [24.0, 20.0])
    assert np.array_equal(s.u_unit, [[0.5, 0.5], [-1.0, 1.0]])
    assert np.array_equal(s.vt_unit, [[0.5, 1.0], [-0.5, 1.0]])


def test_scale_decompose_zero_column_and_shape(hx):
    s = hx.scale_decompose(np.array([[0.0, 1.0], [0.0, 3.0]]), np.array([[1.0, 2.0], [0.0, 0.0]]))
    assert s.diag[0] == 0.0 and s.diag[1] == 0.0
    assert np.all(np.isfinite(s.u_unit)) and np.all(np.isfinite(s.vt_unit))
    with pytest.raises(ValueError):
        hx.scale_decompose(np.zeros((3, 2)), np.zeros((3, 4)))


def test_split_indices(hx):
    hi, lo = hx.split_indices(np.array([1.0, 1e-3, 1e-9]), c=2)
    assert hi.tolist() == [0] and lo.tolist() == [1, 2]
    hi, lo = hx.split_indices(np.array([1.0, 0.01]), c=2)   # strict '<': boundary stays FP64
    assert hi.tolist() == [0, 1] and lo.tolist() == []
    hi, lo = hx.split_indices(np.array([1.0, 0.5]), c=-1)   # threshold above the max
    assert lo.tolist() == [0, 1]
    hi, lo = hx.split_indices(np.zeros(3), c=1)             # all-zero diag: all FP64
    assert hi.tolist() == [0, 1, 2]
    hi, lo = hx.split_indices(np.array([1.0, 1e-300]), c=400)
    assert lo.tolist() == []
    with pytest.raises(ValueError):
        hx.split_indices(np.array([1.0, -1.0]), c=1)


def _bem(hx, refinement=1, aca_tol=1e-6):
    mesh = hx.build_sphere_mesh(hx.axis_centers(3, 3.0), refinement=refinement)
    return mesh, hx.build_hmatrix(mesh, aca_tol=aca_tol)


def test_payload_dtypes_and_byte_identities(hx):
    _, h = _bem(hx)
    sh = {s: hx.prepare_scheme(h, s) for s in ["m1-double", "m1-single", "m2-double", "m2-mixed", "m3:c=2"]}
    assert sh["m1-single"].payload_bytes * 2 == sh["m1-double"].payload_bytes
    rsum = sum(p.u.shape[1] for p in sh["m1-double"].payloads if hasattr(p, "u"))
    assert sh["m2-double"].payload_bytes - sh["m1-double"].payload_bytes == 8 * rsum
    for p in sh["m1-single"].payloads:
        arrs = [p.values] if hasattr(p, "values") else [p.u, p.vt]
        assert all(a.dtype == np.float32 for a in arrs)
    for p in sh["m2-mixed"].payloads:
        if hasattr(p, "diag"):
            assert p.u.dtype == np.float32 and p.diag.dtype == np.float64
            nz = np.abs(p.u).max(axis=0) > 0
            assert np.all(np.abs(p.u).max(axis=0)[nz] == 1.0)
    for p in sh["m3:c=2"].payloads:
        if hasattr(p, "u_hi"):
            assert p.u_hi.dtype == np.float64 and p.u_lo.dtype == np.float32
            assert p.idx_fp64.size + p.idx_fp32.size == p.diag_hi.size + p.diag_lo.size
        else:
            assert p.values.dtype == np.float64
    # payload_bytes equals the bytes of the arrays a matvec reads
    for s in sh.values():
        total = 0
        for p in s.payloads:
            for f in ("values", "u", "vt", "diag", "u_hi", "vt_hi", "diag_hi", "u_lo", "vt_lo", "diag_lo"):
                if hasattr(p, f):
                    total += getattr(p, f).nbytes
        assert total == hx.payload_bytes(s)


def _single_dense(hx, values):
    from paper_1911_00093_b200.partition import ClusterNode, ClusterTree
    n = values.shape[0]
    node = ClusterNode(0, n, np.zeros(3), np.zeros(3))
    tree = ClusterTree(root=node, permutation=np.arange(n), leaf_size=n)
    part = hx.BlockPartition(blocks=[hx.Block(0, n, 0, n, False)], n=n, tree=tree)
    return hx.HMatrixF64(partition=part, payloads=[hx.DenseBlockF64(values)])


def test_fp32_overflow_names_block_and_underflow_counted(hx):
    with pytest.raises(OverflowError, match="block 0"):
        hx.prepare_scheme(_single_dense(hx, np.full((2, 2), 1e300)), "m1-single")
    sh = hx.prepare_scheme(_single_dense(hx, np.array([[1.0, 1e-50], [0.0, 2.0]])), "m1-mixed")
    assert sh.underflow_count == 1


def test_storage_table(hx):
    t = hx.storage_table("m1-mixed")
    assert t["lowrank"]["intermediate"] == "fp32" and t["lowrank"]["source"] == "fp64"
    assert hx.storage_table("m2-single")["lowrank"]["scale"] == "fp64"
    t3 = hx.storage_table("m3:c=1")
    assert t3["dense"]["matrix"] == "fp64" and t3["lowrank"]["fp32_class"]["right_factor"] == "fp32"


def test_partition_tiles_and_dump(hx, tmp_path):
    mesh, h = _bem(hx, refinement=2)
    assert h.partition.coverage_count() == mesh.n * mesh.n
    path = tmp_path / "p.txt"
    hx.dump_partition(h.partition, path)
    lines = path.read_text().splitlines()
    assert len(lines) == len(h.partition.blocks)
    assert lines[0].split()[:4] == [str(v) for v in h.partition.table[0, :4]]


def test_densify_matches_dense_assembly(hx):
    mesh, h = _bem(hx, refinement=1, aca_tol=1e-10)
    a = hx.assemble_dense(mesh)
    d = hx.densify(h)
    assert np.max(np.abs(a - d)) <= 1e-8 * np.max(np.abs(a))


def test_reference_style_payload_lists_pack(hx, orc):
    """An H-matrix given as per-block payload objects (as the reference builds
    them) packs to the same scheme payloads as the native build."""
    _, h = _bem(hx)
    clone = hx.HMatrixF64(partition=h.partition, payloads=h.payloads)
    for s in ["m1-mixed", "m2-single", "m3:c=1"]:
        a, b = hx.prepare_scheme(h, s), hx.prepare_scheme(clone, s)
        x = np.random.default_rng(3).uniform(-1, 1, h.n)
        assert np.array_equal(orc.matvec(a, x), orc.matvec(b, x))


# names of the reference's public API (pkg/src/hmx/__init__.py:57-72) that are
# deliberately not re-exported: CPU helpers and the dense oracle, out of scope
#
NOT_EXPORTED = {"aca_approximate", "block_mul_dense", "block_mul_lowrank",
                "dense_matvec", "dense_solve", "frobenius_error"}


def test_public_names_match_reference(hx):
    import ast
    from pathlib import Path
    init = Path("/root/reference/pkg/src/hmx/__init__.py")
    if not init.exists():
        pytest.skip("reference not present (GPU box)")
    tree = ast.parse(init.read_text())
    ref_all = next(ast.literal_eval(n.value) for n in tree.body
                   if isinstance(n, ast.Assign) and getattr(n.targets[0], "id", "") == "__all__")
    missing = sorted(set(ref_all) - set(hx.__all__) - NOT_EXPORTED)
    assert missing == []
    for name in set(ref_all) - NOT_EXPORTED:
        assert hasattr(hx, name), name
    import paper_1911_00093_b200.bench as b
    for name in ("BenchConfig", "BenchRecord", "run_matvec_bench", "run_solver_bench",
                 "emit_report", "read_report"):
        assert getattr(b, name) is getattr(hx, name)
