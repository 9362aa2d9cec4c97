"""Golden BiCG-STAB envelopes of the REFERENCE ALGORITHM at BASELINE configs 2-4.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_solver_envelope.py <config> <scheme> [...]

For each scheme this runs the oracle's BiCG-STAB (oracle/hmx_oracle.py, pinned
bit for bit to the reference's solver.py:68-168 by tests/test_oracle_golden.py)
with `matvec_threaded(threads = 1..8)` -- the reference's own admissible
summation reorderings (matvec.py:161-197; its tests accept them at 1e-12,
tests/test_matvec.py:158-166) -- on THIS repo's H-matrix of the config
(bench.build_workload: the same host build the GPU tests use).  It writes
tests/golden/solver_envelope_config<k>.json: per scheme and thread count the
stop iteration, converged flag, true residual, breakdown and the full
residual history, plus a fingerprint of the H-matrix so a test can assert
that it is solving the same matrix.

At config 4 one solve costs ~5 min of one core; run one process per scheme.
The file is merged under a lock-free read-modify-write per scheme, so run the
processes on different schemes of one config one after the other, or give
each its own --out and merge with --merge.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_util import fingerprint  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("schemes", nargs="*")
    ap.add_argument("--threads", default="1,2,3,4,5,6,7,8",
                    help="reorderings matvec_threaded(threads=k) to run (config 4 m1-mixed: 1..16)")
    ap.add_argument("--out", default=None)
    ap.add_argument("--merge", nargs="*", default=None, help="merge these partial files into --out")
    a = ap.parse_args()
    out = Path(a.out) if a.out else HERE / f"solver_envelope_config{a.config}.json"
    if a.merge is not None:
        res = json.loads(out.read_text()) if out.exists() else {}
        for p in a.merge:
            part = json.loads(Path(p).read_text())
            for k, v in part.items():
                if k == "schemes":  # per scheme, the thread counts of both files
                    for sname, runs in v.items():
                        res.setdefault("schemes", {}).setdefault(sname, {}).update(runs)
                else:
                    res[k] = v
        out.write_text(json.dumps(res, indent=1))
        return

    import bench
    import paper_1911_00093_b200 as hx
    from oracle import hmx_oracle as orc

    mesh, h, x, b, build_s = bench.build_workload(a.config)
    fp = fingerprint(h)
    sh64 = hx.prepare_scheme(h, "m1-double")
    res = json.loads(out.read_text()) if out.exists() else {}
    if res.get("fingerprint") not in (None, fp):
        raise SystemExit(f"{out} was made on a different H-matrix: {res['fingerprint']} vs {fp}")
    res.update({"config": a.config, "n": int(h.n), "workload": bench.workload_name(a.config),
                "fingerprint": fp, "tol": 1e-8, "max_iter": 1000,
                "openblas_num_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
                "numpy": np.__version__,
                "made_by": "tests/golden/make_solver_envelope.py (oracle bicgstab, "
                           "matvec_threaded threads=k; reference solver.py:68-168, matvec.py:161-197)"})
    res.setdefault("schemes", {})
    for s in a.schemes:
        sh = sh64 if s == "m1-double" else hx.prepare_scheme(h, s)
        runs = res["schemes"].get(s, {})
        for t in [int(v) for v in a.threads.split(",")]:
            if str(t) in runs:
                continue
            t0 = time.perf_counter()
            _, rep = orc.bicgstab(sh, sh64, b, tol=1e-8, max_iter=1000, threads=t)
            runs[str(t)] = {"iterations": rep["iterations"], "converged": bool(rep["converged"]),
                            "true_residual": rep["true_residual"], "breakdown": rep["breakdown"],
                            "residual_history": [float(v) for v in rep["residual_history"]],
                            "cpu_s": round(time.perf_counter() - t0, 2)}
            res["schemes"][s] = runs
            # re-read before writing so concurrent processes on other schemes are kept
            cur = json.loads(out.read_text()) if out.exists() else {}
            cur.update({k: v for k, v in res.items() if k != "schemes"})
            cur.setdefault("schemes", {})[s] = runs
            out.write_text(json.dumps(cur, indent=1))
            print(f"config {a.config} {s} threads={t}: {rep['iterations']} it, "
                  f"converged={rep['converged']}, true {rep['true_residual']}, "
                  f"{time.perf_counter() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
