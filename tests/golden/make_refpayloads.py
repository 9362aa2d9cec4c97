"""Dump the REFERENCE's own prepared payloads (hmx.prepare_scheme ->
SchemeHMatrix.payloads, reference precision.py:169-234, :256-329) of the
ref240_aca4 fixture for every scheme, so the GPU drop-in test can rebuild
reference-shaped objects (DensePayload / FactorPayload / ScaledPayload /
SplitLowRank) on a box where the reference is absent:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_refpayloads.py

Writes tests/golden/ref240_aca4_payloads.npz: per scheme and block k the
payload's arrays under "<scheme>/<k>/<field>", plus "<scheme>/kind"
(0 dense, 1 factor, 2 scaled, 3 split), payload_bytes and underflow_count.
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
import hmx  # noqa: E402  (the reference)
from hmx import precision as P  # noqa: E402

SCHEMES = ["m1-double", "m1-single", "m1-mixed", "m2-double", "m2-single", "m2-mixed",
           "m3:c=-1", "m3:c=1", "m3:c=3", "m3:c=5", "m3:c=7"]
FIELDS = {P.DensePayload: (0, ("values",)), P.FactorPayload: (1, ("u", "vt")),
          P.ScaledPayload: (2, ("u", "vt", "diag")),
          P.SplitLowRank: (3, ("idx_fp64", "idx_fp32", "u_hi", "vt_hi", "diag_hi", "u_lo", "vt_lo",
                               "diag_lo"))}


def main():
    m240 = hmx.build_sphere_mesh(hmx.axis_centers(3, 3.0), refinement=1)
    h = hmx.build_hmatrix(m240, aca_tol=1e-4, leaf_size=32)
    fx = np.load(HERE / "ref240_aca4.npz")
    table = np.array([[b.row_start, b.row_end, b.col_start, b.col_end, int(b.admissible)]
                      for b in h.partition.blocks], dtype=np.int64)
    assert np.array_equal(table, fx["table"]), "reference build differs from the ref240_aca4 fixture"
    out = {}
    for s in SCHEMES:
        sh = hmx.prepare_scheme(h, s)
        kinds = []
        for k, p in enumerate(sh.payloads):
            kind, fields = FIELDS[type(p)]
            kinds.append(kind)
            for f in fields:
                out[f"{s}/{k}/{f}"] = np.asarray(getattr(p, f))
        out[f"{s}/kind"] = np.array(kinds, np.int8)
        out[f"{s}/payload_bytes"] = np.array(sh.payload_bytes, np.int64)
        out[f"{s}/underflow_count"] = np.array(sh.underflow_count, np.int64)
    np.savez_compressed(HERE / "ref240_aca4_payloads.npz", **out)
    print("wrote", HERE / "ref240_aca4_payloads.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
