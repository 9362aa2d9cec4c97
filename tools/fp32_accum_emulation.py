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
  sgemv   OpenBLAS SGEMV-T's tree as its four-row kernel computes it, for
          every row (sgemv_tree)
  sgemv-rows  the GPU kernel's order since round 2 (chain_item /
          s1_exact_kernel in csrc/hmx_kernels.cu): each row in the order of
          the SGEMV row kernel that computes it (16/8/4-row kernels, 2- and
          1-row remainder kernels; sgemv_rows) -- numpy's own products bitwise

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


def chain_shaped(n: int) -> bool:
    return n <= 3 or 5 <= n <= 7


def chunk_off(n: int, rp: int, row: int, k: int) -> int:
    """Port of csrc/hmx_internal.cuh chunk_off: element offset of (row, column
    k) inside an n-wide FP32-accumulated item stored in SGEMV chunk layout."""
    nch = 0 if chain_shaped(n) else n >> 2
    if k < 4 * nch:
        return ((k >> 2) * rp + row) * 4 + (k & 3)
    return 4 * nch * rp + (k - 4 * nch) * rp + row


def _fma(a, b, c):
    """FP32 fused multiply-add, exact product and one rounding (x87 extended
    sum: a 48-bit product plus a 24-bit addend is exact there unless their
    exponents are > 40 apart)."""
    ld = np.longdouble
    return (np.asarray(a, F32).astype(ld) * np.asarray(b, F32).astype(ld) + np.asarray(c, F32).astype(ld)).astype(F32)


def _mul(a, b):
    return (np.asarray(a, F32).astype(F64) * np.asarray(b, F32).astype(F64)).astype(F32)


def sgemv_tree(a, g):
    """The GPU kernel's FP32 product of one item, per row (chain_items in
    csrc/hmx_kernels.cu): OpenBLAS SGEMV-T's tree -- A/B 4-wide FMA
    accumulators over 4-column chunks, (l0 + l1) + (l2 + l3), then the tail
    rule; n = 8 pairs adjacent columns; n <= 3 and 5..7 one FMA chain."""
    a = np.asarray(a, F32)
    g = np.asarray(g, F32)
    m, n = a.shape
    z = np.zeros(m, F32)
    if chain_shaped(n):
        v = z
        for k in range(n):
            v = _fma(a[:, k], g[k], v)
        return v
    nch, tt = n >> 2, n & 3
    if n == 8:
        lanes = [_mul(a[:, 2 * j], g[2 * j]) + _mul(a[:, 2 * j + 1], g[2 * j + 1]) for j in range(4)]
    else:
        if nch % 2:
            ca, cb = [0] + list(range(1, nch, 2)), list(range(2, nch, 2))
        else:
            ca, cb = list(range(0, nch, 2)), list(range(1, nch, 2))
        lanes = []
        for j in range(4):
            va, vb = z, z
            for c in ca:
                va = _fma(a[:, 4 * c + j], g[4 * c + j], va)
            for c in cb:
                vb = _fma(a[:, 4 * c + j], g[4 * c + j], vb)
            lanes.append(va + vb)
    v = (lanes[0] + lanes[1]) + (lanes[2] + lanes[3])
    mm = 4 * nch
    if tt == 1:
        v = _fma(a[:, mm], g[mm], v)
    elif tt >= 2:
        t = _fma(a[:, mm], g[mm], _mul(a[:, mm + 1], g[mm + 1]))
        if tt == 3:
            t = _fma(a[:, mm + 2], g[mm + 2], t)
        v = v + t
    return v


def row_kind(i: int, m: int) -> int:
    """OpenBLAS SGEMV-T computes the rows (outputs) of an m-row block in blocks
    of 16, then 8, then 4 rows, then a two-row and a one-row remainder kernel;
    their summation orders differ (the 16-, 8- and 4-row kernels only for
    rows shorter than 8).  Kind 16, 8, 4, 2 or 1 for row i."""
    a16 = m & ~15
    if i < a16:
        return 16
    b8 = a16 + (m & 8)
    if i < b8:
        return 8
    c4 = b8 + (m & 4)
    if i < c4:
        return 4
    if (m & 3) >= 2 and i < c4 + 2:
        return 2
    return 1


def sgemv_kind(a, g, kind: int):
    """One row class of SGEMV-T (probed with tools/sgemv_order_probe.py and
    the brute-force family search described in DESIGN.md):
      kinds 16, 8, 4: A/B accumulators, FMA chains (sgemv_tree); rows
        shorter than 8 differ: 8: n = 2 is a plain sum; 4: n = 2, 3, 6, 7 use
        the trees below;
      kind 2: ONE 4-lane accumulator over all chunks, multiply-then-add;
      kind 1: A/B accumulators, multiply-then-add;
    then (l0 + l1) + (l2 + l3) and the tail rule of sgemv_tree.  Short rows:
    kind 4 as sgemv_tree; kinds 2/1: n = 2..7 a sequential multiply-add chain
    (kind 1, n = 3: the tail rule), n = 4
    pairwise (kind 1: sequential), n = 8 (kind 1): A/B with a sequential
    horizontal sum; kind 2, n = 8: ((p0 + p1) + (p4 + p5)) + ((p2 + p3) + (p6 + p7))."""
    a = np.asarray(a, F32)
    g = np.asarray(g, F32)
    m, n = a.shape
    z = np.zeros(m, F32)
    G = lambda k: np.full(m, g[k], F32)
    P = lambda k: _mul(a[:, k], G(k))
    F = lambda k, acc: _fma(a[:, k], G(k), acc)
    if kind in (16, 8, 4):
        if kind == 8 and n == 2:
            return P(0) + P(1)
        if kind == 4 and n in (2, 3, 6, 7):  # the four-row kernel's short-row trees
            if n == 2:
                return P(0) + P(1)
            if n == 3:
                return F(2, F(0, P(1)))
            if n == 6:
                return (P(0) + F(1, P(2))) + (P(3) + F(4, P(5)))
            return (F(0, P(1)) + F(4, P(5))) + (F(2, P(3)) + P(6))
        return sgemv_tree(a, g)
    if n == 1:
        return P(0)
    if kind == 1 and n == 3:
        return _fma(a[:, 2], G(2), _fma(a[:, 0], G(0), P(1)))
    if kind == 2 and n == 8:
        return ((P(0) + P(1)) + (P(4) + P(5))) + ((P(2) + P(3)) + (P(6) + P(7)))
    if n <= 7 and n != 4:
        v = P(0)
        for k in range(1, n):
            v = v + P(k)
        return v
    nch, tt = n >> 2, n & 3
    if kind == 2:
        ca, cb = list(range(nch)), []
    elif nch % 2:
        ca, cb = [0] + list(range(1, nch, 2)), list(range(2, nch, 2))
    else:
        ca, cb = list(range(0, nch, 2)), list(range(1, nch, 2))
    lanes = []
    for j in range(4):
        va, vb = z, z
        for c in ca:
            va = va + P(4 * c + j)
        for c in cb:
            vb = vb + P(4 * c + j)
        lanes.append(va + vb)
    seq = kind == 1 and n <= 8
    v = ((lanes[0] + lanes[1]) + lanes[2]) + lanes[3] if seq else (lanes[0] + lanes[1]) + (lanes[2] + lanes[3])
    mm = 4 * nch
    if tt == 1:
        v = _fma(a[:, mm], G(mm), v)
    elif tt >= 2:
        t = _fma(a[:, mm], G(mm), P(mm + 1))
        if tt == 3:
            t = _fma(a[:, mm + 2], G(mm + 2), t)
        v = v + t
    return v


def sgemv_rows(a, g):
    """SGEMV-T of an m-row block, every row in its kernel's order (row_kind)."""
    m = a.shape[0]
    out = np.empty(m, F32)
    kinds = np.array([row_kind(i, m) for i in range(m)])
    for k in (16, 8, 4, 2, 1):
        sel = kinds == k
        if sel.any():
            out[sel] = sgemv_kind(a[sel], g, k)
    return out


def sgemv_blocked(a, g, block: int = 4096, rows: bool = False):
    """OpenBLAS SGEMV-T over long rows: 4096-column blocks, each reduced by
    sgemv_tree (the tail in the last block), added in order -- the order of
    the GPU's m1-single stage 1 (s1_exact_kernel)."""
    n = a.shape[1]
    y = None
    for s0 in range(0, n, block):
        v = (sgemv_rows if rows else sgemv_tree)(a[:, s0:s0 + block], g[s0:s0 + block])
        y = v if y is None else (y + v).astype(F32)
    return y


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
    if order == "sgemv-rows":
        return sgemv_rows(a, g)
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
                if s1 in ("sgemv", "sgemv-rows"):
                    z = sgemv_blocked(pay.vt, xs32, rows=s1 == "sgemv-rows")
                else:
                    z = prod32(pay.vt, xs32, s1) if s1 != "numpy" else pay.vt @ xs32
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
    """The GPU's order (sgemv_rows / sgemv_blocked) against numpy's own
    `A32 @ g32` on random data, for row counts 2..64 and widths 1..48, then
    long rows: prints the (rows, widths) that differ."""
    rng = np.random.default_rng(7)
    for m in list(range(2, 25)) + [30, 40, 48, 64]:
        bad = []
        for n in range(1, 49):
            for _ in range(6):
                a = rng.standard_normal((m, n)).astype(F32)
                g = rng.standard_normal(n).astype(F32)
                if not np.array_equal(sgemv_rows(a, g), a @ g):
                    bad.append(n)
                    break
        print(f"rows {m:3d}: widths 1..48 differing from numpy: {bad if bad else 'none'}")
    for n in (100, 1280, 4096, 4100, 5120, 10240, 20480):
        a = rng.standard_normal((13, n)).astype(F32)
        g = rng.standard_normal(n).astype(F32)
        print(f"long row n={n}, 13 rows: blocked model == numpy: "
              f"{np.array_equal(sgemv_blocked(a, g, rows=True), a @ g)}")


def main():
    import paper_1911_00093_b200 as hx
    names = sys.argv[1:] or ["golden", "config1", "config2"]
    if names == ["bitwise"]:
        return bitwise_check()
    orders = ["chain", "lanes4", "lanes8", "sgemv", "sgemv-rows"]
    print(f"{'case':12s} {'scheme':10s} " + " ".join(f"{o:>8s}" for o in orders)
          + "   (||y - y64|| / ||y_ref - y64||)")
    for name, h, x in cases(names):
        y64 = orc.matvec(hx.prepare_scheme(h, "m1-double"), x)
        for s in ("m1-single", "m1-mixed", "m2-single"):
            sh = hx.prepare_scheme(h, s)
            ref = np.linalg.norm(orc.matvec(sh, x) - y64)
            row = [np.linalg.norm(matvec_model(sh, x, o, o if o.startswith("sgemv") else "numpy") - y64) / ref
                   for o in orders]
            print(f"{name:12s} {s:10s} " + " ".join(f"{v:8.4f}" for v in row), flush=True)


if __name__ == "__main__":
    main()
