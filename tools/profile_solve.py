"""One BiCG-STAB solve of one scheme at one BASELINE config (for an ncu
launch list of the solver's kernels).

  python tools/profile_solve.py --config 4 --scheme m1-double
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--scheme", default="m1-double")
    a = ap.parse_args()
    mesh, h, x, b, _ = bench.build_workload(a.config)
    sh = hx.prepare_scheme(h, a.scheme)
    cfg = hx.SolverConfig(tol=1e-8)
    hx.bicgstab(sh, h, b, cfg)
    _, rep = hx.bicgstab(sh, h, b, cfg)
    print(f"{a.scheme} config{a.config}: {rep.iterations} it, {rep.matvecs} matvecs, "
          f"device {rep.device_time_s * 1e3:.2f} ms")


if __name__ == "__main__":
    main()
