"""BiCG-STAB parity at BASELINE configs 2-4 against the REFERENCE ALGORITHM's
own reordering envelope.

tests/golden/solver_envelope_config<k>.json holds, for the headline schemes,
the oracle BiCG-STAB (pinned bit-for-bit to reference solver.py:68-168) run
with matvec_threaded(threads = 1..8) -- the summation reorderings the
reference itself accepts (matvec.py:161-197) -- on THIS repo's H-matrix of
the config (made by tests/golden/make_solver_envelope.py in the build
container; the matrix fingerprint is checked here).  North-star criterion:
the GPU's stop iteration lies in [min - max(1, 5 %), max + max(1, 5 %)] of
that envelope, and its `converged` flag is one the envelope produced (for a
scheme that never converges, whose stop is noise-driven: 10 %, and the true
residual floor within 10 % of the reference's).
"""
import json

import numpy as np
import pytest

from golden_util import GOLDEN, fingerprint

pytestmark = pytest.mark.gpu


def envelope(cfg):
    f = GOLDEN / f"solver_envelope_config{cfg}.json"
    if not f.exists():
        pytest.skip(f"{f.name} not generated")
    return json.loads(f.read_text())


def check(rep, runs):
    its = [r["iterations"] for r in runs]
    # A scheme whose FP32 floor lies above tol never converges: the recurrence
    # residual wanders around tol and the stop is the first time it dips
    # below -- a noise-driven event (config 4 m1-mixed: 89-99 over the
    # reference's own 16 reorderings).  There the band is 10 % and the true
    # residual (the floor) must match the reference's to 10 %.
    stagnant = not any(r["converged"] for r in runs)
    frac = 0.10 if stagnant else 0.05
    lo = min(its) - max(1.0, frac * min(its))
    hi = max(its) + max(1.0, frac * max(its))
    assert lo <= rep.iterations <= hi, (rep.iterations, sorted(its))
    assert rep.converged in {r["converged"] for r in runs}, (rep.converged, [r["converged"] for r in runs])
    assert rep.breakdown is None and rep.true_residual is not None
    assert rep.converged == (rep.true_residual < 1e-8)
    if stagnant:
        trs = [r["true_residual"] for r in runs]
        assert 0.9 * min(trs) <= rep.true_residual <= 1.1 * max(trs), (rep.true_residual, min(trs), max(trs))


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_bicgstab_inside_reference_envelope(hx, cfg):
    import bench
    env = envelope(cfg)
    _, h, _, b, _ = bench.build_workload(cfg)
    assert fingerprint(h) == env["fingerprint"], "not the H-matrix the envelope was made on"
    out = {}
    for s, runs in env["schemes"].items():
        sh = hx.prepare_scheme(h, s)
        _, rep = hx.bicgstab(sh, h, b, hx.SolverConfig(tol=env["tol"], max_iter=env["max_iter"]))
        out[s] = (rep.iterations, rep.converged, rep.true_residual)
        check(rep, list(runs.values()))
        # the first iteration follows the reference algorithm's residual
        # history; later entries are chaotic (the reference's own reorderings
        # spread them by 1e-7 at iteration 2 and 1 % at iteration 4 at config
        # 4), so only the stop point above is compared
        ref = np.asarray(runs["1"]["residual_history"][:2])
        assert np.allclose(np.asarray(rep.residual_history[:2]), ref, rtol=1e-8), s
        del sh
    print(out)
