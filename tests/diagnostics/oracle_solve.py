"""Reference-algorithm BiCG-STAB (the oracle port of solver.py, numpy, CPU)
on this repo's config-4 H-matrix, for comparison with the GPU solves.

  python tests/diagnostics/oracle_solve.py <out.json> <scheme> [<scheme> ...]
  (HMX_CONFIG=<n> selects another BASELINE config; default 4)

Test/diagnostic tool (imports the oracle as the checker); ~5-10 min per
scheme at config 4.
"""
import json
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
    out, schemes = sys.argv[1], sys.argv[2:]
    import os
    mesh, h, x, b, _ = bench.build_workload(int(os.environ.get("HMX_CONFIG", "4")))
    sh64 = hx.prepare_scheme(h, "m1-double")
    res = json.loads(Path(out).read_text()) if Path(out).exists() else {}
    for s in schemes:
        sh = hx.prepare_scheme(h, s)
        t0 = time.perf_counter()
        _, rep = orc.bicgstab(sh, sh64, b, tol=1e-8, max_iter=1000)
        res[s] = {"iterations": rep["iterations"], "converged": rep["converged"],
                  "true_residual": rep["true_residual"], "breakdown": rep["breakdown"],
                  "history_tail": rep["residual_history"][-4:], "cpu_s": time.perf_counter() - t0}
        Path(out).write_text(json.dumps(res, indent=1))
        print(s, res[s], flush=True)


if __name__ == "__main__":
    main()
