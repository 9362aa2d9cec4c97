"""One rank of the multi-process test of libhmx_gpu's multi-GPU mode on one
GPU (tests/test_gpu_dist_shim.py; NCCL replaced by tests/shim via
HMX_NCCL_LIB, the unique id broadcast over a gloo group).

    python tests/dist_shim_worker.py <rank> <world> <port> <out.json> <cuts|auto>

Runs the PRODUCT path: row-restricted plans (build_hmatrix(rows=...)), the
library's communicator (hmx_comm_create), hmx_dist_matvec and
hmx_bicgstab_dist.  Writes this rank's slices and reports to out.json.<rank>.
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

SCHEMES = ["m1-double", "m1-mixed", "m2-mixed", "m3:c=1"]


def main():
    import faulthandler
    import os
    # a stuck rank dumps its Python stack (and exits) instead of hanging the test
    faulthandler.dump_traceback_later(float(os.environ.get("HMX_SHIM_WORKER_TIMEOUT", "240")), exit=True)
    rank, world, port, out, cuts_arg = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
    import torch
    import torch.distributed as dist

    import paper_1911_00093_b200 as hx
    from paper_1911_00093_b200 import distributed as D

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    mesh = hx.jittered_sphere_mesh(4, seed=42)
    part = hx.build_block_partition(hx.build_cluster_tree(mesh, 32), 2.0)
    n = mesh.n
    if cuts_arg == "auto":
        # measured-bytes cut: build on the estimate, exchange real ranks, re-cut
        cuts = D.measured_cuts(mesh, part, aca_tol=1e-4, world=world, rank=rank)
    else:
        cuts = [int(v) for v in cuts_arg.split(",")]
    slices = D.RowSlices(cuts)
    a, b = slices.span(rank)
    h = hx.build_hmatrix(mesh, partition=part, aca_tol=1e-4, rows=(a, b))
    perm = np.asarray(h.permutation)
    x = np.random.default_rng(3).uniform(-1.0, 1.0, n)
    rhs = mesh.centroids[:, 2].copy()
    res = {"rank": rank, "cuts": cuts, "schemes": {}}
    comm = D.make_comm(slices, rank, dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    op64, _ = D.make_gpu_operator(h, "m1-double", slices, rank, dev)
    for s in SCHEMES:
        op = op64 if s == "m1-double" else D.make_gpu_operator(h, s, slices, rank, dev)[0]
        xl = torch.from_numpy(np.ascontiguousarray(x[perm[a:b]])).to(dev)
        y = torch.empty(b - a, dtype=torch.float64, device=dev)
        comm.matvec(op.plan, xl.data_ptr(), y.data_ptr(), stream=stream)
        torch.cuda.synchronize()
        y_dist = y.cpu().numpy().copy()
        # the same row-restricted plan on the full permuted x, no exchange
        xp = torch.from_numpy(np.ascontiguousarray(x[perm])).to(dev)
        op.plan.apply_local(xp.data_ptr(), y.data_ptr(), stream=stream)
        torch.cuda.synchronize()
        y_local = y.cpu().numpy().copy()
        xs, rep = D.bicgstab_gpu(comm, op.plan, op64.plan, rhs[perm[a:b]], tol=1e-8, max_iter=1000,
                                 scheme_label=s)
        print(f"rank {rank} {s}: {rep.iterations} it, converged {rep.converged}, true {rep.true_residual}, "
              f"breakdown {rep.breakdown}, matvecs {rep.matvecs}", flush=True)
        res["schemes"][s] = {
            "y_dist": y_dist.tolist(), "y_local": y_local.tolist(), "x_solve": np.asarray(xs).tolist(),
            "iterations": rep.iterations, "converged": rep.converged, "true_residual": rep.true_residual,
            "residual_history": rep.residual_history, "matvecs": rep.matvecs, "breakdown": rep.breakdown}
        if op is not op64:
            op.plan.close()
    op64.plan.close()
    comm.close()
    Path(f"{out}.{rank}").write_text(json.dumps(res))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
