"""Golden FP32 block products of the reference's arithmetic (numpy `A32 @ x32`,
reference matvec.py:57 / :73, OpenBLAS SGEMV) for block widths 1..48 and
row counts 8, 40, 30 and 5 (30 and 5: OpenBLAS's two- and one-row remainder
kernels for rows 28-29 and 4), computed in the build container:

    python tests/golden/make_fp32_order.py

tests/test_gpu_fp32_order.py runs the same blocks through the GPU's
FP32-accumulated item path (m2-single dense items) and checks them bitwise
against these products and against the CPU model of the kernel's order
(tools/fp32_accum_emulation.py sgemv_tree).  The probe that recovered the
order is tools/sgemv_order_probe.py; its output for this container is
profiles/round2_sgemv_order_container.json.
"""
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def blocks():
    rng = np.random.default_rng(2024)
    for m in (8, 40, 30, 5):
        for n in range(1, 49):
            a = rng.standard_normal((m, n))          # FP64 masters
            x = rng.uniform(-1.0, 1.0, n)
            yield m, n, a, x


def main():
    out = {}
    for m, n, a, x in blocks():
        a32, x32 = a.astype(np.float32), x.astype(np.float32)
        out[f"a/{m}/{n}"] = a
        out[f"x/{m}/{n}"] = x
        out[f"y/{m}/{n}"] = a32 @ x32                # the reference's FP32 GEMV
    np.savez_compressed(HERE / "fp32_order.npz", **out)
    print("wrote", HERE / "fp32_order.npz", len(out) // 3, "blocks")


if __name__ == "__main__":
    main()
