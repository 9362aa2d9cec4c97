"""CPU emulation of FP32 accumulation orders for the FP32-accumulated items of
m1-single, m1-mixed and m2-single (reference matvec.py:57, :68-74: numpy
`A32 @ x32` / `U32 @ z32`, i.e. an OpenBLAS SGEMV).

For each scheme it evaluates the matvec with the FP32-accumulated products
computed in a chosen summation order -- everything else exactly as the
reference (numpy) -- and reports ||y - y64|| / ||y_ref - y64||, y64 being the
FP64 (m1-double) product and y_ref the reference's own FP32 result.  Orders:

  numpy   the reference itself (ratio 1 by definition)
  chain   one sequential FP32 FMA chain per (row, block) -- the round-1 GPU kernel
  lanesK  K interleaved FP32 lane chains (column j -> lane j mod K), combined
          by a pairwise tree over the lanes in the order the GPU kernel uses
          (K = 8: ((l0+l4)+(l1+l5))+((l2+l6)+(l3+l7)), what OpenBLAS's SGEMV
          does on this container for widths that are multiples of 8 --
          probed with tools/sgemv_order_probe.py)
  sgemv   the GPU kernel's order since round 2 (obl_col + lane tree of
          csrc/hmx_internal.cuh): OpenBLAS SGEMV-T's own tree

FMA is emulated as round32(round64(a*b) + c) with the product exact in FP64;
the double rounding differs from a true fused FMA in rare ties only, which is
immaterial for these norms.  Test/diagnostic tool: imports the oracle.

  python tools/fp32_accum_emulation.py [golden|config1|config2 ...]
  python tools/fp32_accum_emulation.py bitwise   # sgemv order vs numpy, per width
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import hmx_oracle as orc  # noqa: E402

F32, F64 = np.float32, np.float64


def lane_order(k: int) -> list[int]:
    """Leaf order of the lane tree: pairwise over this order."""
    if k == 8:
        return [0, 4, 1, 5, 2, 6, 3, 7]
    return list(range(k))


def pairwise(parts):
    """Balanced pairwise FP32 sum in the given leaf order (binary counter)."""
    while len(parts) > 1:
        nxt = [(parts[i].astype(F64) + parts[i + 1].astype(F64)).astype(F32)
               for i in range(0, len(parts) - 1, 2)]
        if len(parts) % 2:
            nxt.append(parts[-1])
        parts = nxt
    return parts[0]


def fma_chain(a, g, acc=None):
    """Sequential FP32 FMA over the columns of a (m x n, f32) times g (n, f32)."""
    m = a.shape[0]
    acc = np.zeros(m, F32) if acc is None else acc
    for j in range(a.shape[1]):
        acc = (acc.astype(F64) + a[:, j].astype(F64) * F64(g[j])).astype(F32)
    return acc


OB_NONE, OB_ITEM_CHAIN, OB_ITEM_MAIN, OB_B, OB_A1, OB_TAIL1, OB_TAIL = 0, 1, 2, 3, 4, 7, 8


def obl_col(n: int, k: int):
    """Port of csrc/hmx_internal.cuh obl_col: (original column, OB_* code) of
    stored position k of an n-wide FP32-accumulated item."""
    if n <= 3 or 5 <= n <= 7:
        return k, (OB_ITEM_CHAIN if k == 0 else OB_NONE)
    mainw = n & ~3
    nch = mainw >> 2
    if k < mainw:
        j, r = divmod(k, nch)
        na = (nch + 1) >> 1
        code = OB_NONE
        if r == 0:
            code = OB_ITEM_MAIN if j == 0 else OB_A1 + (j - 1)
        elif r == na:
            code = OB_B
        if n == 8:
            return k, code
        if r < na:
            chunk = (0 if r == 0 else 2 * r - 1) if nch & 1 else 2 * r
        else:
            chunk = 2 * (r - na) + 2 if nch & 1 else 2 * (r - na) + 1
        return 4 * chunk + j, code
    t, tt = k - mainw, n - mainw
    code = (OB_TAIL1 if tt == 1 else OB_TAIL) if t == 0 else OB_NONE
    if tt == 1:
        return mainw, code
    return (mainw + 1 if t == 0 else mainw if t == 1 else mainw + 2), code


def _fma(a, b, c):
    """FP32 fused multiply-add, exact product and one rounding (x87 extended
    sum: a 48-bit product plus a 24-bit addend is exact there unless their
    exponents are > 40 apart)."""
    ld = np.longdouble
    return (a.astype(ld) * b.astype(ld) + c.astype(ld)).astype(F32)


def sgemv_tree(a, g):
    """The GPU kernel's FP32 product of one item (consume32 in
    csrc/hmx_kernels.cu): columns in obl_col storage order, one FMA chain per
    sub-chain, the lane tree folded at every sub-chain start."""
    m, n = a.shape
    z = np.zeros(m, F32)
    cur, tp, s01, s2, mode = z, z, z, z, 0
    for k in range(n):
        c, code = obl_col(n, k)
        if code in (OB_ITEM_CHAIN, OB_ITEM_MAIN):
            mode = 1 if code == OB_ITEM_MAIN else 0
        elif code == OB_B:
            tp, cur, mode = cur, z, 1
        elif OB_A1 <= code < OB_TAIL1:
            lv = tp + cur
            if code == OB_A1:
                s01 = lv
            elif code == OB_A1 + 1:
                s01 = s01 + lv
            else:
                s2 = lv
            tp, cur, mode = z, z, 1
        elif code in (OB_TAIL1, OB_TAIL):
            mv = s01 + (s2 + (tp + cur))
            tp, s2 = z, z
            if code == OB_TAIL1:
                cur, s01, mode = mv, z, 0
            else:
                s01, cur, mode = mv, z, 2
        cur = _fma(a[:, c], np.full(m, g[c], F32), cur)
    if mode == 1:
        return s01 + (s2 + (tp + cur))
    if mode == 2:
        return s01 + cur
    return cur


def prod32(a, g, order: str):
    a = np.asarray(a, F32)
    g = np.asarray(g, F32)
    if order == "numpy":
        return a @ g
    n = a.shape[1]
    if n == 0:
        return np.zeros(a.shape[0], F32)
    if order == "chain":
        return fma_chain(a, g)
    if order == "sgemv":
        return sgemv_tree(a, g)
    if order.startswith("lanes"):
        k = int(order[5:])
        lanes = [fma_chain(a[:, j::k], g[j::k]) for j in range(min(k, n))]
        lanes += [np.zeros(a.shape[0], F32)] * (k - len(lanes))
        return pairwise([lanes[j] for j in lane_order(k)])
    raise ValueError(order)


def matvec_model(sh, x, order: str, stage1_order: str | None = None):
    """orc.matvec with the FP32-accumulated products in `order`."""
    xp, xp32 = orc.gather(sh, x)
    yp = np.zeros(sh.n)
    s1 = stage1_order or order
    for blk, pay in sh.items():
        r0, r1, c0, c1 = blk.row_start, blk.row_end, blk.col_start, blk.col_end
        xs = xp[c0:c1]
        xs32 = xp32[c0:c1] if xp32 is not None else None
        if hasattr(pay, "values"):
            if pay.values.dtype == F32 and xs32 is not None:
                yp[r0:r1] += prod32(pay.values, xs32, order)
            else:
                yp[r0:r1] += orc.dense_partial(pay.values, xs, xs32)
        elif not hasattr(pay, "diag") and not hasattr(pay, "u_hi") and pay.u.dtype == F32:
            if xs32 is not None:   # m1-single: z = Vt32 x32 in FP32 too
                z = prod32(pay.vt.T.T, xs32, s1) if s1 != "numpy" else pay.vt @ xs32
            else:                  # m1-mixed: FP64 sum, rounded once
                z = (pay.vt @ xs).astype(F32)
            yp[r0:r1] += prod32(pay.u, z, order)
        else:
            yp[r0:r1] += orc.lowrank_partial(pay, xs, xs32)
    y = np.empty(sh.n)
    y[sh.base.permutation] = yp
    return y


def cases(names):
    import golden_util as gu
    import paper_1911_00093_b200 as hx
    for name in names:
        if name == "golden":
            for fx in ("ref60", "ref240", "ref240_aca4"):
                arr, _ = gu.load(fx)
                yield fx, gu.hmatrix_from_fixture(arr), arr["x"]
        elif name.startswith("config"):
            import bench
            _, h, x, _, _ = bench.build_workload(int(name[6:]))
            yield name, h, x


def bitwise_check():
    """sgemv_tree vs numpy's own `A32 @ g32` on random data: prints the
    widths where they differ (per row count)."""
    rng = np.random.default_rng(7)
    for m in (4, 8, 20, 40, 64, 3, 7):
        bad = []
        for n in range(1, 70):
            for _ in range(6):
                a = rng.standard_normal((m, n)).astype(F32)
                g = rng.standard_normal(n).astype(F32)
                if not np.array_equal(sgemv_tree(a, g), a @ g):
                    bad.append(n)
                    break
        print(f"rows {m:3d}: widths 1..69 differing from numpy: {bad if bad else 'none'}")


def main():
    import paper_1911_00093_b200 as hx
    names = sys.argv[1:] or ["golden", "config1", "config2"]
    if names == ["bitwise"]:
        return bitwise_check()
    orders = ["chain", "lanes4", "lanes8", "sgemv"]
    print(f"{'case':12s} {'scheme':10s} " + " ".join(f"{o:>8s}" for o in orders)
          + "   (||y - y64|| / ||y_ref - y64||)")
    for name, h, x in cases(names):
        y64 = orc.matvec(hx.prepare_scheme(h, "m1-double"), x)
        for s in ("m1-single", "m1-mixed", "m2-single"):
            sh = hx.prepare_scheme(h, s)
            ref = np.linalg.norm(orc.matvec(sh, x) - y64)
            row = [np.linalg.norm(matvec_model(sh, x, o, "numpy") - y64) / ref for o in orders]
            print(f"{name:12s} {s:10s} " + " ".join(f"{v:8.4f}" for v in row), flush=True)


if __name__ == "__main__":
    main()
