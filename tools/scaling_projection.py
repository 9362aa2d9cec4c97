"""Projected strong scaling of the multi-GPU mode from one GPU.

For world = 1, 2, 4, 8 the rows are cut exactly as `bench.py --gpus N`
does (distributed.partition_rows on estimated ranks), every rank's
row-restricted H-matrix and device plan (HMX_PLAN_LOCAL_FIRST) are built in
turn on this one GPU, and each rank's local two-stage product is timed with
CUDA events (plan.bench): the per-rank compute and its balance are
MEASURED.  Only the exchange is modelled: one allgather per matvec, each
rank receiving (N - N/world) x 8 bytes at an assumed 600 GB/s effective
NVLink-5 rate plus 15 us of NCCL latency, with no credit for the overlap
with the local-first stage-1 work.

  python tools/scaling_projection.py --config 4 --schemes m1-double m2-mixed
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402
from paper_1911_00093_b200 import _gpu  # noqa: E402
from paper_1911_00093_b200 import distributed as D  # noqa: E402

LINK_GBPS, LATENCY_US = 600.0, 15.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--schemes", nargs="*", default=["m1-double", "m2-mixed"])
    ap.add_argument("--worlds", nargs="*", type=int, default=[1, 2, 4, 8])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    c = bench.CONFIGS[a.config]
    mesh = hx.jittered_sphere_mesh(c["level"], seed=42, centers=c.get("centers", ((0.0, 0.0, 0.0),)),
                                   voltages=c.get("voltages"))
    part = hx.build_block_partition(hx.build_cluster_tree(mesh, c["leaf"]), 2.0)
    n, table = part.n, part.table
    perm = np.asarray(part.tree.permutation)
    kinds = table[:, 4].astype(np.int32)
    est = np.where(kinds == 1, 11, 0)
    out = {"config": a.config, "n": int(n), "model": {"allgather_GBps": LINK_GBPS,
                                                      "latency_us": LATENCY_US}, "schemes": {}}
    for scheme in a.schemes:
        rows = []
        t1 = None
        for world in a.worlds:
            cuts = D.partition_rows(table, kinds, est, n, world)
            ms, nbytes = [], []
            for r in range(world):
                span = (cuts[r], cuts[r + 1])
                hk = hx.build_hmatrix(mesh, partition=part, aca_tol=c["aca"], rows=span)
                sh = hx.prepare_scheme(hk, scheme)
                plan = _gpu.Plan(sh.packed, table, perm, sh.scheme.label, n, row_range=span,
                                 local_first=world > 1)
                ms.append(plan.bench(5, 50)["ms"])
                nbytes.append(plan.info()["payload_bytes"])
                plan.close()
            comm_ms = 0.0 if world == 1 else (LATENCY_US * 1e-3 +
                                              (n - n / world) * 8 / (LINK_GBPS * 1e9) * 1e3)
            step = max(ms) + comm_ms
            t1 = step if world == 1 else t1
            row = {"world": world, "cuts": [int(v) for v in cuts],
                   "local_ms": ms, "local_max_ms": max(ms), "balance_max_over_mean": max(ms) / np.mean(ms),
                   "payload_bytes": nbytes, "allgather_model_ms": comm_ms,
                   "projected_ms_per_matvec": step, "projected_matvec_per_s": 1e3 / step,
                   "projected_efficiency": t1 / (world * step) if t1 else None}
            rows.append(row)
            print(f"{scheme} world {world}: local max {max(ms):.4f} ms (balance {row['balance_max_over_mean']:.3f}), "
                  f"allgather model {comm_ms:.4f} ms -> {1e3 / step:.0f} matvec/s, "
                  f"efficiency {row['projected_efficiency']:.2f}", flush=True)
        out["schemes"][scheme] = rows
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
