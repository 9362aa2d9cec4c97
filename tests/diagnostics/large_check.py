"""Parity and solver diagnostics at a large BASELINE config (default 5).

  python tests/diagnostics/large_check.py [--config 5] [--schemes m1-double ...] [--max-iter 300]

GPU matvec of each scheme against the oracle's full matvec (numpy, one pass),
then a BiCG-STAB solve whose residual history is printed every 10 iterations.
Test/diagnostic tool: it imports the oracle as the checker.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402
from oracle import hmx_oracle as orc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--schemes", nargs="*", default=["m1-double"])
    ap.add_argument("--max-iter", type=int, default=300)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--level", type=int, default=None, help="override the config's refinement level")
    ap.add_argument("--sigma", type=float, default=None, help="override the vertex jitter")
    a = ap.parse_args()
    if a.level is not None:
        bench.CONFIGS[a.config] = dict(bench.CONFIGS[a.config], level=a.level)
    if a.sigma is not None:
        orig = hx.jittered_sphere_mesh
        hx.jittered_sphere_mesh = lambda *args, **kw: orig(*args, **dict(kw, sigma=a.sigma))
    mesh, h, x, b, tb = bench.build_workload(a.config)
    print(f"config {a.config}: n={mesh.n} blocks={h.partition.table.shape[0]} build {tb:.1f} s", flush=True)
    for name in a.schemes:
        sh = hx.prepare_scheme(h, name)
        y = hx.matvec(sh, x)
        if not a.no_oracle:
            t0 = time.perf_counter()
            yo = orc.matvec(sh, x)
            err = np.linalg.norm(y - yo) / np.linalg.norm(yo)
            print(f"{name}: matvec rel err vs oracle {err:.3e} (oracle {time.perf_counter() - t0:.1f} s)",
                  flush=True)
        xs, rep = hx.bicgstab(sh, h, b, hx.SolverConfig(tol=1e-8, max_iter=a.max_iter))
        hist = rep.residual_history
        print(f"{name}: iterations {rep.iterations} converged {rep.converged} true {rep.true_residual} "
              f"breakdown {rep.breakdown} wall {rep.wall_time_s:.2f} s", flush=True)
        print("  history:", " ".join(f"{i}:{hist[i]:.2e}" for i in range(0, len(hist), 10)), flush=True)
        print(f"  min residual {min(hist):.3e} at {int(np.argmin(hist))}", flush=True)
        if name != "m1-double":
            get = getattr(sh, "_hmx_gpu_plan", None)
            if get is not None:
                get.close()


if __name__ == "__main__":
    main()
