"""Device-side prepare_scheme (hmx_master_create + hmx_plan_create_prepared)
against the host preparation (which itself matches the reference's
precision.py bit for bit, tests/test_host_api.py).

The device plan must be bit-identical to the host-prepared one: the same
matvec bits, payload_bytes, underflow_count and OverflowError text.
"""

import numpy as np
import pytest

from golden_util import config1_hmatrix, hmatrix_from_fixture, load

pytestmark = pytest.mark.gpu

SCHEMES = ["m1-double", "m1-single", "m1-mixed", "m2-double", "m2-single", "m2-mixed",
           "m3:c=-1", "m3:c=0", "m3:c=1", "m3:c=3", "m3:c=5", "m3:c=7", "m3:c=400"]


@pytest.fixture(scope="module")
def cases(hx):
    mesh, h1 = config1_hmatrix()
    arr, _ = load("ref240_aca4")
    h2 = hmatrix_from_fixture(arr)                       # the reference's own H-matrix
    mesh3 = hx.jittered_sphere_mesh(4, seed=7)
    h3 = hx.build_hmatrix(mesh3, aca_tol=1e-5, leaf_size=64, eta=2.0)
    return [h1, h2, h3]


@pytest.mark.parametrize("scheme", SCHEMES)
def test_device_prepared_plan_is_bitwise_host_plan(hx, cases, scheme):
    from paper_1911_00093_b200 import _gpu
    from paper_1911_00093_b200.device_prepare import get_master, prepare_scheme_device
    from paper_1911_00093_b200.precision import _split_factor
    for h in cases:
        x = np.random.default_rng(5).uniform(-1.0, 1.0, h.n)
        sh = hx.prepare_scheme(h, scheme)
        sd = prepare_scheme_device(h, scheme)
        assert sd.payload_bytes == sh.payload_bytes
        assert sd.underflow_count == sh.underflow_count
        assert np.array_equal(hx.matvec(sd, x), hx.matvec(sh, x))
        # fresh plans on both paths (m1-double plans are otherwise shared)
        factor = _split_factor(sh.scheme.c) if sh.scheme.method == 3 else 0.0
        pd, info = _gpu.Plan.prepared(get_master(h), sh.scheme.label, factor)
        ph = _gpu.Plan(sh.packed, h.partition.table, np.asarray(h.permutation), sh.scheme.label, h.n)
        assert pd.info() == ph.info()
        yd, _ = pd.matvec(x)
        yh, _ = ph.matvec(x)
        assert np.array_equal(yd, yh)
        pd.close()
        ph.close()


def test_device_prepared_solve_is_bitwise(hx, cases):
    from paper_1911_00093_b200.device_prepare import prepare_scheme_device
    h = cases[0]
    b = np.random.default_rng(3).uniform(-1.0, 1.0, h.n)
    for scheme in ("m2-mixed", "m3:c=3"):
        xs, rs = hx.bicgstab(hx.prepare_scheme(h, scheme), h, b, hx.SolverConfig(tol=1e-8))
        xd, rd = hx.bicgstab(prepare_scheme_device(h, scheme), h, b, hx.SolverConfig(tol=1e-8))
        assert rd.iterations == rs.iterations and rd.converged == rs.converged
        assert np.array_equal(xd, xs)
        assert rd.residual_history == rs.residual_history


def _scaled_copy(hx, h, factor):
    from paper_1911_00093_b200.compress import HMatrixF64, PackedMaster
    pm = h.packed
    return HMatrixF64(h.partition, packed=PackedMaster(pm.data * factor, pm.kinds, pm.ranks,
                                                       pm.offsets))


def test_overflow_error_matches_host(hx, cases):
    from paper_1911_00093_b200.device_prepare import prepare_scheme_device
    big = _scaled_copy(hx, cases[0], 1e40)
    for scheme in ("m1-single", "m1-mixed"):
        with pytest.raises(OverflowError) as eh:
            hx.prepare_scheme(big, scheme)
        with pytest.raises(OverflowError) as ed:
            prepare_scheme_device(big, scheme)
        assert str(ed.value) == str(eh.value)
        assert "block" in str(ed.value)
    # scaled factors have max-abs 1: no overflow for Method 2/3
    prepare_scheme_device(big, "m2-single")


def test_underflow_count_matches_host(hx, cases):
    from paper_1911_00093_b200.device_prepare import prepare_scheme_device
    tiny = _scaled_copy(hx, cases[2], 1e-36)
    for scheme in ("m1-single", "m1-mixed", "m2-single", "m3:c=1"):
        sh = hx.prepare_scheme(tiny, scheme)
        sd = prepare_scheme_device(tiny, scheme)
        assert sd.underflow_count == sh.underflow_count
        if scheme.startswith("m1"):
            assert sd.underflow_count > 0
        x = np.random.default_rng(1).uniform(-1.0, 1.0, tiny.n)
        assert np.array_equal(hx.matvec(sd, x), hx.matvec(sh, x))


def test_host_payloads_on_demand(hx, cases):
    from paper_1911_00093_b200.device_prepare import prepare_scheme_device
    h = cases[0]
    sd = prepare_scheme_device(h, "m3:c=3")
    sh = hx.prepare_scheme(h, "m3:c=3")
    for a, b in zip(sd.payloads[:50], sh.payloads[:50]):
        for f in ("values", "u_hi", "vt_hi", "u_lo", "vt_lo", "diag_hi", "diag_lo"):
            if hasattr(b, f):
                assert np.array_equal(getattr(a, f), getattr(b, f))
