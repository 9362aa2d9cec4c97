"""Golden hashes of the reference's interchange formats for config 1:
`hmx.dump_partition` (partition.py:172-177) and `hmx.export_mesh`
(problem.py:260-267), written by the REFERENCE's own functions on its own
config-1 build.  Run in the build container:

    python tests/golden/make_interchange.py
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, str(ROOT))

import hmx  # noqa: E402  (the reference)

import paper_1911_00093_b200 as ours  # noqa: E402  (mesh recipe only)


def main():
    m = ours.jittered_sphere_mesh(3, seed=42)
    mesh = hmx.PanelMesh(np.array(m.vertices), np.array(m.triangles), np.array(m.sphere_ids),
                         np.array(m.voltages))
    h = hmx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32, eta=2.0)
    out = {}
    with tempfile.TemporaryDirectory() as d:
        hmx.dump_partition(h.partition, Path(d) / "p.txt")
        hmx.export_mesh(mesh, Path(d) / "m.txt")
        for key, name in (("dump_partition", "p.txt"), ("export_mesh", "m.txt")):
            data = (Path(d) / name).read_bytes()
            out[key] = {"sha256": hashlib.sha256(data).hexdigest(), "bytes": len(data),
                        "lines": data.count(b"\n")}
    out["recipe"] = "config 1: jittered_sphere_mesh(3, seed=42), build_hmatrix(aca_tol=1e-4, leaf_size=32, eta=2.0)"
    (HERE / "interchange.json").write_text(json.dumps(out, indent=1))
    print(out)


if __name__ == "__main__":
    main()
