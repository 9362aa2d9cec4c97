"""Median device time of repeated BiCG-STAB solves (A/B of solver builds:
HMX_GPU_LIB selects the library).

  python tools/solve_ab.py --config 2 --schemes m1-double m2-mixed --reps 7
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--schemes", nargs="*", default=["m1-double", "m2-mixed"])
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    mesh, h, x, b, _ = bench.build_workload(a.config)
    cfg = hx.SolverConfig(tol=1e-8)
    for s in a.schemes:
        sh = hx.prepare_scheme(h, s)
        hx.bicgstab(sh, h, b, cfg)
        ts, its = [], set()
        for _ in range(a.reps):
            _, rep = hx.bicgstab(sh, h, b, cfg)
            ts.append(rep.device_time_s)
            its.add((rep.iterations, rep.matvecs, rep.converged, rep.true_residual))
        print(f"config{a.config} {s:10s} device {1e3 * np.median(ts):8.3f} ms  {sorted(its)}")


if __name__ == "__main__":
    main()
