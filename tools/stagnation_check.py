"""Is BiCG-STAB's stagnation near 6e-6 at the level-8 jittered meshes a
property of the PROBLEM (the reference algorithm does the same) or of the
GPU path?  (VERDICT r1 item 10.)

Runs, on one H-matrix, the GPU solve and the CPU oracle solve (the
reference algorithm, oracle/hmx_oracle.py, bit-pinned to solver.py) for the
first K iterations each, and writes both residual histories side by side.

  python tools/stagnation_check.py [--level 8] [--spheres 1|2] [--iters 30] [--out f.json]

Diagnostic tool (imports the oracle as the checker).  At level 8 one oracle
matvec costs several seconds, so K = 30 takes minutes of host time.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1911_00093_b200 as hx  # noqa: E402
from oracle import hmx_oracle as orc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=8)
    ap.add_argument("--spheres", type=int, default=1, choices=(1, 2))
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--full-gpu", type=int, default=300, help="max_iter of the extra full GPU solve")
    ap.add_argument("--scheme", default="m1-double")
    ap.add_argument("--out", default=None)
    ap.add_argument("--part", choices=("both", "oracle", "gpu"), default="both",
                    help="run only one side (the oracle on a CPU host, the GPU solve on the box) and "
                         "merge the two JSON files with --merge")
    ap.add_argument("--merge", nargs=2, default=None, metavar=("GPU_JSON", "ORACLE_JSON"))
    a = ap.parse_args()
    if a.merge:
        g, o = (json.loads(Path(f).read_text()) for f in a.merge)
        gh, oh = np.asarray(g["gpu_history"]), np.asarray(o["oracle_history"])
        k = min(gh.size, oh.size)
        res = {**o, **g, "oracle_history": oh.tolist(), "oracle_s": o.get("oracle_s"),
               "max_rel_diff_first_k": float(np.max(np.abs(gh[:k] - oh[:k]) / oh[:k]))}
        Path(a.out).write_text(json.dumps(res, indent=1))
        for i in range(k):
            print(f"{i:3d}  gpu {gh[i]:.6e}  oracle {oh[i]:.6e}")
        return
    centers = ((0.0, 0.0, 0.0),) if a.spheres == 1 else ((0.0, 0.0, 0.0), (3.0, 0.0, 0.0))
    volts = None if a.spheres == 1 else (1.0, -1.0)
    t0 = time.perf_counter()
    mesh = hx.jittered_sphere_mesh(a.level, seed=42, centers=centers, voltages=volts)
    h = hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=64, eta=2.0)
    b = mesh.centroids[:, 2].copy() if a.spheres == 1 else hx.right_hand_side(mesh)
    sh = hx.prepare_scheme(h, a.scheme)
    t_build = time.perf_counter() - t0
    res = {"mesh": f"{a.spheres} jittered sphere(s), level {a.level}, N={mesh.n}, leaf 64, ACA 1e-4",
           "scheme": a.scheme, "iters": a.iters, "build_s": t_build}
    if a.part in ("both", "gpu"):
        cfg = hx.SolverConfig(tol=1e-8, max_iter=a.iters)
        _, g = hx.bicgstab(sh, h, b, cfg)
        _, gfull = hx.bicgstab(sh, h, b, hx.SolverConfig(tol=1e-8, max_iter=a.full_gpu))
        res["gpu_history"] = list(g.residual_history)
        res["gpu_full"] = {"max_iter": a.full_gpu, "iterations": gfull.iterations,
                           "converged": gfull.converged, "true_residual": gfull.true_residual,
                           "min_residual": float(np.min(gfull.residual_history)),
                           "history_every_10": gfull.residual_history[::10]}
    if a.part in ("both", "oracle"):
        t1 = time.perf_counter()
        sh64 = sh if a.scheme == "m1-double" else hx.prepare_scheme(h, "m1-double")
        _, o = orc.bicgstab(sh, sh64, b, tol=1e-8, max_iter=a.iters)
        res["oracle_s"] = time.perf_counter() - t1
        res["oracle_history"] = list(o["residual_history"])
    if a.part != "both":
        Path(a.out).write_text(json.dumps(res, indent=1))
        print(json.dumps({k_: v for k_, v in res.items() if "history" not in k_}), flush=True)
        return
    gh, oh = np.asarray(res["gpu_history"]), np.asarray(res["oracle_history"])
    k = min(gh.size, oh.size)
    res["max_rel_diff_first_k"] = float(np.max(np.abs(gh[:k] - oh[:k]) / oh[:k]))
    print(json.dumps({k_: v for k_, v in res.items() if "history" not in k_}), flush=True)
    for i in range(k):
        print(f"{i:3d}  gpu {gh[i]:.6e}  oracle {oh[i]:.6e}")
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
