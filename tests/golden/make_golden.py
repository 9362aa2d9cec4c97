"""Generate the golden fixtures of tests/golden/ from the REFERENCE package.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every number stored here is produced by the reference's own code
(hmx.build_hmatrix, hmx.prepare_scheme, hmx.matvec, hmx.bicgstab); only the
jittered config-1 mesh vertices come from this repo's recipe
(paper_1911_00093_b200.problem.jittered_sphere_mesh), fed to the
reference's PanelMesh.  The fixtures pin oracle/hmx_oracle.py (bit-for-bit)
and this repo's host builder (block table, ranks, payload bytes) to the
reference, and give the GPU tests reference outputs to compare against.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, str(ROOT))

import hmx  # noqa: E402  (the reference)

import paper_1911_00093_b200 as ours  # noqa: E402  (mesh recipe only)

SCHEMES = ["m1-double", "m1-single", "m1-mixed", "m2-double", "m2-single", "m2-mixed",
           "m3:c=-1", "m3:c=1", "m3:c=3", "m3:c=5", "m3:c=7"]


def pack_hmatrix(h):
    """Reference HMatrixF64 -> flat arrays (block table, kinds, ranks, data)."""
    blocks = h.partition.blocks
    table = np.array([[b.row_start, b.row_end, b.col_start, b.col_end, int(b.admissible)]
                      for b in blocks], dtype=np.int64)
    kinds, ranks, parts = [], [], []
    for p in h.payloads:
        if isinstance(p, hmx.DenseBlockF64):
            kinds.append(0)
            ranks.append(0)
            parts.append(p.values.ravel())
        else:
            kinds.append(1)
            ranks.append(p.rank)
            parts += [p.u.ravel(), p.vt.ravel()]
    return dict(table=table, kinds=np.array(kinds, np.int32), ranks=np.array(ranks, np.int64),
                data=np.concatenate(parts), perm=np.asarray(h.permutation, np.int64))


def report_dict(rep):
    return {"scheme": rep.scheme, "converged": bool(rep.converged),
            "iterations": int(rep.iterations),
            "residual_history": [float(v) for v in rep.residual_history],
            "true_residual": None if rep.true_residual is None else float(rep.true_residual),
            "breakdown": rep.breakdown}


def envelope(sh, h, b, tol, max_iter):
    """The reference's own spread under admissible summation reorderings:
    bicgstab with matvec_threaded(threads = 1..8), whose results may differ
    from the sequential matvec by 1e-12 (reference tests/test_matvec.py:158-166)."""
    its, conv = [], []
    for t in range(1, 9):
        _, rep = hmx.bicgstab(sh, h, b, hmx.SolverConfig(tol=tol, max_iter=max_iter, threads=t))
        its.append(int(rep.iterations))
        conv.append(bool(rep.converged))
    return {"iterations": its, "converged": conv}


def full_case(name, mesh, aca_tol, x, b, tol, max_iter, leaf_size=32):
    """Stores the reference H-matrix itself plus outputs of every scheme."""
    h = hmx.build_hmatrix(mesh, aca_tol=aca_tol, leaf_size=leaf_size)
    arrays = pack_hmatrix(h)
    arrays["x"] = x
    arrays["b"] = b
    reports = {}
    for s in SCHEMES:
        sh = hmx.prepare_scheme(h, s)
        arrays[f"y/{s}"] = hmx.matvec(sh, x)
        arrays[f"bytes/{s}"] = np.array(sh.payload_bytes, np.int64)
        arrays[f"underflow/{s}"] = np.array(sh.underflow_count, np.int64)
        xs, rep = hmx.bicgstab(sh, h, b, hmx.SolverConfig(tol=tol, max_iter=max_iter))
        arrays[f"xsol/{s}"] = xs
        reports[s] = report_dict(rep)
        reports[s]["envelope"] = envelope(sh, h, b, tol, max_iter)
    # non-finite input: the reference names the first offending block
    bad = x.copy()
    bad[0] = np.inf
    try:
        hmx.matvec(hmx.prepare_scheme(h, "m1-double"), bad)
        msg = None
    except FloatingPointError as e:
        msg = str(e)
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    meta = {"n": int(mesh.n), "aca_tol": aca_tol, "leaf_size": leaf_size, "tol": tol,
            "max_iter": max_iter, "reports": reports, "nonfinite_message": msg}
    (HERE / f"{name}.json").write_text(json.dumps(meta, indent=1))
    print(name, mesh.n, "blocks", arrays["table"].shape[0], "payload", arrays["data"].nbytes)


def config1_case():
    """BASELINE config 1: outputs only (the H-matrix is rebuilt by the tests
    with this repo's builder and compared through them)."""
    m = ours.jittered_sphere_mesh(3, seed=42)
    mesh = hmx.PanelMesh(np.array(m.vertices), np.array(m.triangles), np.array(m.sphere_ids),
                         np.array(m.voltages))
    h = hmx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32, eta=2.0)
    arrays = pack_hmatrix(h)
    x = np.random.default_rng(42).uniform(-1.0, 1.0, mesh.n)
    b = np.array(mesh.centroids[:, 2])
    out = {"table": arrays["table"], "ranks": arrays["ranks"], "kinds": arrays["kinds"],
           "perm": arrays["perm"], "x": x, "b": b,
           "centroids": np.array(mesh.centroids), "areas": np.array(mesh.areas)}
    reports = {}
    for s in SCHEMES:
        sh = hmx.prepare_scheme(h, s)
        out[f"y/{s}"] = hmx.matvec(sh, x)
        out[f"bytes/{s}"] = np.array(sh.payload_bytes, np.int64)
        _, rep = hmx.bicgstab(sh, h, b, hmx.SolverConfig(tol=1e-8, max_iter=1000))
        reports[s] = report_dict(rep)
        reports[s]["envelope"] = envelope(sh, h, b, 1e-8, 1000)
    np.savez_compressed(HERE / "config1.npz", **out)
    meta = {"n": int(mesh.n), "aca_tol": 1e-4, "leaf_size": 32, "eta": 2.0, "tol": 1e-8,
            "recipe": "jittered_sphere_mesh(3, seed=42); x = default_rng(42).uniform(-1,1,N); "
                      "b = centroid z", "reports": reports}
    (HERE / "config1.json").write_text(json.dumps(meta, indent=1))
    print("config1", mesh.n, "blocks", out["table"].shape[0])


def main():
    m60 = hmx.build_sphere_mesh(hmx.axis_centers(3, 3.0), refinement=0)
    full_case("ref60", m60, 1e-8, np.random.default_rng(41).uniform(-1.0, 1.0, m60.n),
              hmx.right_hand_side(m60), 1e-6, 200)
    m240 = hmx.build_sphere_mesh(hmx.axis_centers(3, 3.0), refinement=1)
    full_case("ref240", m240, 1e-8, np.random.default_rng(17).uniform(-1.0, 1.0, m240.n),
              hmx.right_hand_side(m240), 1e-8, 200)
    full_case("ref240_aca4", m240, 1e-4, np.random.default_rng(43).uniform(-1.0, 1.0, m240.n),
              np.array(m240.centroids[:, 2]), 1e-8, 200)
    config1_case()


if __name__ == "__main__":
    main()
