"""GPU BiCG-STAB at one config under summation-order perturbations: the
stage-1 chunk size changes how each z entry's FP64 sum is split, an
ulp-level reordering like the reference's own `threads` option.  Prints the
spread of stop iterations / converged flags / true residuals per scheme."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402
from paper_1911_00093_b200 import _gpu  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    out = sys.argv[2] if len(sys.argv) > 2 else None
    schemes = ["m1-double", "m1-mixed", "m2-mixed", "m3:c=3"]
    chunks = [96 << 10, 160 << 10, 256 << 10, 384 << 10, 640 << 10]
    mesh, h, x, b, _ = bench.build_workload(cfg)
    perm = np.asarray(h.permutation)
    res = {}
    for s in schemes:
        rows = []
        for cb in chunks:
            sh = hx.prepare_scheme(h, s)
            plan = _gpu.Plan(sh.packed, h.partition.table, perm, sh.scheme.label, h.n, s1_chunk_bytes=cb)
            if s == "m1-double":
                object.__setattr__(h, "_hmx_gpu_plan64", plan)
            else:
                sh._hmx_gpu_plan = plan
            _, rep = hx.bicgstab(sh, h, b, hx.SolverConfig(tol=1e-8, max_iter=1000))
            rows.append({"s1_chunk_kb": cb >> 10, "iterations": rep.iterations, "converged": rep.converged,
                         "true_residual": rep.true_residual})
            if s != "m1-double":
                plan.close()
        res[s] = rows
        its = [r["iterations"] for r in rows]
        print(f"{s:9s} iterations {min(its)}-{max(its)} {its} converged {sorted({r['converged'] for r in rows})} "
              f"true residual {min(r['true_residual'] for r in rows):.3g}-{max(r['true_residual'] for r in rows):.3g}",
              flush=True)
    if out:
        Path(out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
