"""Small end-to-end workload touching every device path: every scheme's
matvec and solve, device preparation (checked bitwise against host
preparation), GPU compression (checked bitwise against the host build) and
the world-1 multi-GPU solver, at N = 1,280.  (Meant for compute-sanitizer,
which the GPU pool of round 1 does not allow.)

  python tools/small_workload.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1911_00093_b200 as hx  # noqa: E402

SCHEMES = ["m1-double", "m1-single", "m1-mixed", "m2-double", "m2-single", "m2-mixed",
           "m3:c=-1", "m3:c=1", "m3:c=3"]


def main():
    mesh = hx.jittered_sphere_mesh(3, seed=42)
    h = hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32)
    x = np.random.default_rng(1).uniform(-1, 1, mesh.n)
    b = mesh.centroids[:, 2].copy()
    for s in SCHEMES:
        sh = hx.prepare_scheme(h, s)
        y = hx.matvec(sh, x)
        _, rep = hx.bicgstab(sh, h, b, hx.SolverConfig(tol=1e-8))
        shd = hx.prepare_scheme_device(h, s)
        yd = hx.matvec(shd, x)
        assert np.array_equal(y, yd), s
        print(s, rep.iterations, rep.converged, flush=True)
    hg = hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32, device=0)
    assert np.array_equal(hg.packed.data, h.packed.data)
    import torch
    from paper_1911_00093_b200 import _gpu
    from paper_1911_00093_b200 import distributed as D
    perm = np.asarray(h.permutation)
    comm = D.make_comm(D.RowSlices([0, h.n]), 0, torch.device("cuda", 0))
    sh = hx.prepare_scheme(h, "m2-mixed")
    plan = _gpu.Plan(sh.packed, h.partition.table, perm, "m2-mixed", h.n, row_range=(0, h.n),
                     local_first=True)
    D.bicgstab_gpu(comm, plan, None, b[perm], tol=1e-8)
    plan.close()
    comm.close()
    print("small workload done")


if __name__ == "__main__":
    main()
