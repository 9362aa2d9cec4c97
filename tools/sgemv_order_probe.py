"""Reveal the FP32 summation tree numpy/OpenBLAS uses for `A32 @ x32` (C-order
A, the reference's FP32-accumulated block products, matvec.py:57 and :73).

For every pair of columns (p, q) the row is set to ones except A[p] = 2^30,
A[q] = -2^30 and x = ones: the result counts the ones that were added after
p and q cancelled, so n - result is the number of leaves under the lowest
common ancestor of p and q in the summation tree ("FPRev"-style probing).  The
tree is rebuilt from those counts and printed / saved as nested lists.

  python tools/sgemv_order_probe.py [max_n] [--json out.json]

Diagnostic tool; the output documents the order the GPU's FP32 lane tree
mirrors ("FP32 accumulation order").
"""
from __future__ import annotations

import json
import sys

import numpy as np

BIG = np.float32(2.0 ** 30)


def lca_sizes(n: int, m: int = 8, row: int = 0) -> np.ndarray:
    lsz = np.zeros((n, n), int)
    z = np.ones(n, np.float32)
    for p in range(n):
        for q in range(p + 1, n):
            a = np.ones((m, n), np.float32)
            a[:, p] = BIG
            a[:, q] = -BIG
            lsz[p, q] = lsz[q, p] = n - int((a @ z)[row])
    return lsz


def tree(ids, lsz):
    if len(ids) == 1:
        return ids[0]
    n = len(ids)
    groups: list[list[int]] = []
    for i in ids:
        for g in groups:
            if lsz[i, g[0]] < n:
                g.append(i)
                break
        else:
            groups.append([i])
    if len(groups) == 1:
        raise RuntimeError(f"cannot split {ids}")
    sub = [tree(g, lsz) for g in groups]
    out = sub[0]
    for s in sub[1:]:
        out = [out, s]
    return out


def show(t) -> str:
    return str(t) if isinstance(t, int) else f"({show(t[0])} + {show(t[1])})"


def main():
    args = sys.argv[1:]
    out = None
    if "--json" in args:
        i = args.index("--json")
        out = args[i + 1]
        del args[i:i + 2]
    nmax = int(args[0]) if args else 24
    res = {}
    for n in range(1, nmax + 1):
        t = tree(list(range(n)), lca_sizes(n))
        res[n] = t
        print(n, show(t), flush=True)
    if out:
        import platform
        info = {"numpy": np.__version__, "machine": platform.machine(), "processor": platform.processor()}
        try:
            cfg = np.show_config(mode="dicts")
            info["blas"] = cfg.get("Build Dependencies", {}).get("blas", {})
        except Exception:
            pass
        try:
            with open("/proc/cpuinfo") as f:
                info["cpu"] = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
        except OSError:
            pass
        json.dump({"info": info, "trees": res}, open(out, "w"))


if __name__ == "__main__":
    main()
