"""Save the products of a few schemes at one BASELINE config (A/B of two builds
of libhmx_gpu.so through HMX_GPU_LIB: the saved arrays must be bitwise equal
when a change claims to keep the arithmetic).

  python tools/ab_bitwise.py --config 2 --out gpurun_out/y_a.npz
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
    ap.add_argument("--schemes", nargs="+", default=["m1-single", "m1-mixed", "m2-single"])
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    mesh, h, x, b, _ = bench.build_workload(a.config)
    out = {}
    for s in a.schemes:
        out[s] = hx.matvec(hx.prepare_scheme(h, s), x)
    np.savez(a.out, **out)


if __name__ == "__main__":
    main()
