"""Pin the CPU oracle (oracle/hmx_oracle.py) to the reference: on the
reference's own H-matrices (tests/golden), the oracle's matvec and BiCG-STAB
must reproduce the reference's outputs bit for bit, and this repo's
prepare_scheme must reproduce the reference's payload bytes/underflow counts."""

import numpy as np
import pytest

from golden_util import SCHEMES, hmatrix_from_fixture, load

CASES = ["ref60", "ref240", "ref240_aca4"]


@pytest.fixture(scope="module", params=CASES)
def case(request):
    arr, meta = load(request.param)
    return request.param, arr, meta, hmatrix_from_fixture(arr)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_oracle_matvec_bitwise(hx, orc, case, scheme):
    _, arr, _, h = case
    sh = hx.prepare_scheme(h, scheme)
    assert sh.payload_bytes == int(arr[f"bytes/{scheme}"])
    assert sh.underflow_count == int(arr[f"underflow/{scheme}"])
    y = orc.matvec(sh, arr["x"])
    assert np.array_equal(y, arr[f"y/{scheme}"])


@pytest.mark.parametrize("scheme", ["m1-double", "m1-single", "m2-mixed", "m3:c=-1", "m3:c=3"])
def test_oracle_bicgstab_matches_reference(hx, orc, case, scheme):
    name, arr, meta, h = case
    sh = hx.prepare_scheme(h, scheme)
    sh64 = hx.prepare_scheme(h, "m1-double")
    x, rep = orc.bicgstab(sh, sh64, arr["b"], tol=meta["tol"], max_iter=meta["max_iter"])
    ref = meta["reports"][scheme]
    assert rep["iterations"] == ref["iterations"]
    assert rep["converged"] == ref["converged"]
    assert rep["breakdown"] == ref["breakdown"]
    assert rep["residual_history"] == ref["residual_history"]
    assert np.array_equal(x, arr[f"xsol/{scheme}"])


def test_oracle_nonfinite_message(hx, orc):
    arr, meta = load("ref240")
    h = hmatrix_from_fixture(arr)
    bad = arr["x"].copy()
    bad[0] = np.inf
    with pytest.raises(FloatingPointError) as e:
        orc.matvec(hx.prepare_scheme(h, "m1-double"), bad)
    assert str(e.value) == meta["nonfinite_message"]


def test_oracle_threaded_matches_sequential(hx, orc):
    arr, _ = load("ref240")
    h = hmatrix_from_fixture(arr)
    sh = hx.prepare_scheme(h, "m2-mixed")
    y1 = orc.matvec(sh, arr["x"])
    for t in (2, 3, 8):
        yt = orc.matvec_threaded(sh, arr["x"], t)
        assert np.max(np.abs(yt - y1)) <= 1e-12 * np.max(np.abs(y1))
    assert np.array_equal(orc.matvec_threaded(sh, arr["x"], 1), y1)
