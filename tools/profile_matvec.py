"""Run a few device matvecs of one scheme at one BASELINE config (for ncu).

  python tools/profile_matvec.py --config 4 --scheme m1-mixed --iters 3
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402
from paper_1911_00093_b200.matvec import get_plan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--scheme", default="m1-double")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    mesh, h, x, b, _ = bench.build_workload(a.config)
    sh = hx.prepare_scheme(h, a.scheme)
    plan = get_plan(sh)
    y = hx.matvec(sh, x)
    r = plan.bench(1, a.iters)
    info = plan.info()
    print(f"{a.scheme} config{a.config}: {r} stage1_bytes={info['stage1_bytes']} "
          f"stage2_bytes={info['stage2_bytes']} s1_ctas={info['s1_grid']} s2_ctas={info['s2_grid']} "
          f"checksum={float(np.sum(y)):.17g}")


if __name__ == "__main__":
    main()
