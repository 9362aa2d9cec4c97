"""Method-3 cut-off sweep (the paper's accuracy / speed trade-off): for each
c, the scheme prepared on the device from resident masters, its matvec time
and bandwidth, the FP32 share of the ranks, and a BiCG-STAB solve to 1e-8.

  python tools/c_sweep.py 4 out.json
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402
from paper_1911_00093_b200.matvec import get_plan  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    out = sys.argv[2] if len(sys.argv) > 2 else None
    mesh, h, x, b, _ = bench.build_workload(cfg)
    total_rank = int(h.packed.ranks[h.packed.kinds == 1].sum())
    rows = []
    for name in ["m2-double"] + [f"m3:c={c}" for c in (7, 5, 4, 3, 2, 1, 0, -1)] + ["m2-mixed"]:
        sh = hx.prepare_scheme_device(h, name)
        plan = get_plan(sh)
        r = plan.bench(5, 100)
        algo = sh.payload_bytes + 16 * h.n
        _, rep = hx.bicgstab(sh, h, b, hx.SolverConfig(tol=1e-8))
        row = {"scheme": name, "matvec_ms": r["ms"], "GBps": algo / r["ms"] / 1e6,
               "payload_bytes": sh.payload_bytes,
               "fp32_rank_share": getattr(sh, "fp32_ranks", 0) / total_rank if name.startswith("m3") else None,
               "iterations": rep.iterations, "converged": rep.converged,
               "true_residual": rep.true_residual, "solve_device_s": rep.device_time_s}
        rows.append(row)
        print(f"{name:10s} {r['ms']*1e3:8.1f} us {row['GBps']:7.0f} GB/s  payload {sh.payload_bytes/1e9:6.3f} GB  "
              f"fp32 ranks {row['fp32_rank_share'] if row['fp32_rank_share'] is not None else '-'}  "
              f"solve {rep.iterations} it {rep.converged} {rep.true_residual:.2e} "
              f"{rep.device_time_s*1e3:.1f} ms", flush=True)
        plan.close()
    if out:
        Path(out).write_text(json.dumps({"config": cfg, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
