"""The drop-in with the REFERENCE's own payload objects.

tests/refshape.py rebuilds, from arrays the reference produced
(tests/golden/make_refpayloads.py), reference-shaped SchemeHMatrix /
DensePayload / FactorPayload / ScaledPayload / SplitLowRank objects of the
ref240_aca4 fixture.  CPU: this repo's prepare_scheme reproduces every
reference payload array bitwise.  GPU: installed into a package with the
reference's module layout, `hmx.matvec`, `hmx.bicgstab` and
`hmx.true_residual` run those objects on the device and reproduce the
reference's outputs (golden)."""
import numpy as np
import pytest

import refshape as R
from golden_util import FP64_ONLY, SCHEMES


def test_prepare_scheme_reproduces_reference_payloads_bitwise(hx):
    h, arr, _ = R.hmatrix()
    from golden_util import hmatrix_from_fixture
    ours = hmatrix_from_fixture(arr)
    for s in SCHEMES:
        ref = R.scheme_hmatrix(h, s)
        sh = hx.prepare_scheme(ours, s)
        assert sh.payload_bytes == ref.payload_bytes and sh.underflow_count == ref.underflow_count, s
        for k, (p, q) in enumerate(zip(sh.payloads, ref.payloads)):
            assert type(p).__name__ == type(q).__name__, (s, k)
            for f in type(q).__dataclass_fields__:
                a, b = np.asarray(getattr(p, f)), np.asarray(getattr(q, f))
                assert a.dtype == b.dtype and a.shape == b.shape and np.array_equal(a, b), (s, k, f)


@pytest.mark.gpu
def test_reference_objects_through_drop_in_on_the_gpu(hx):
    from paper_1911_00093_b200 import drop_in

    import sys
    h, arr, meta = R.hmatrix()
    pkg = R.fake_reference_package()
    mv, sv = sys.modules[pkg.__name__ + ".matvec"], sys.modules[pkg.__name__ + ".solver"]
    saved = drop_in.install(pkg)
    try:
        for s in SCHEMES:
            sh = R.scheme_hmatrix(h, s)
            y = mv.matvec(sh, arr["x"])
            tol = 1e-12 if s in FP64_ONLY else 1e-5
            ref = arr[f"y/{s}"]
            assert np.max(np.abs(y - ref)) <= tol * np.max(np.abs(ref)), s
            assert np.array_equal(mv.matvec_threaded(sh, arr["x"], 4), y)
            x, rep = sv.bicgstab(sh, h, arr["b"], hx.SolverConfig(tol=meta["tol"],
                                                                         max_iter=meta["max_iter"]))
            env = meta["reports"][s]["envelope"]
            slack = max(1, int(0.05 * meta["reports"][s]["iterations"]))
            assert min(env["iterations"]) - slack <= rep.iterations <= max(env["iterations"]) + slack, s
            assert rep.converged in set(env["converged"]), s
            tr = pkg.true_residual(h, x, arr["b"])
            if rep.true_residual is not None:
                assert tr == pytest.approx(rep.true_residual, rel=1e-10, abs=1e-14)
            assert rep.scheme == s
    finally:
        drop_in.uninstall(saved)
