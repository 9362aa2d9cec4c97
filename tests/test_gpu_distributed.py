"""Multi-GPU machinery on one B200: row-restricted device plans
(hmx_apply_local) for a byte-balanced row split reproduce the full product,
including cuts that straddle blocks; the distributed BiCG-STAB runs over a
real NCCL process group (world 1) with the GPU local product."""

import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def cfg(hx):
    mesh = hx.jittered_sphere_mesh(4, seed=42)
    h = hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32)
    return mesh, h, np.random.default_rng(3).uniform(-1, 1, mesh.n)


@pytest.mark.parametrize("scheme", ["m1-double", "m1-mixed", "m2-single", "m3:c=1"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_slices_reproduce_full_product(hx, cfg, scheme, world):
    import torch

    from paper_1911_00093_b200 import _gpu
    from paper_1911_00093_b200 import distributed as D

    mesh, h, x = cfg
    perm = np.asarray(h.permutation)
    table = h.partition.table
    cuts = D.partition_rows(table, h.packed.kinds, h.packed.ranks, h.n, world)
    if world == 3:  # force a cut through the middle of a leaf (straddles blocks)
        cuts[1] += 7
    y_full = hx.matvec(hx.prepare_scheme(h, scheme), x)[perm]
    dev = torch.device("cuda", 0)
    xp = torch.from_numpy(np.ascontiguousarray(x[perm])).to(dev)
    pieces = []
    for k in range(world):
        a, b = cuts[k], cuts[k + 1]
        hk = hx.build_hmatrix(mesh, partition=h.partition, aca_tol=1e-4, rows=(a, b))
        sh = hx.prepare_scheme(hk, scheme)
        plan = _gpu.Plan(sh.packed, table, perm, sh.scheme.label, h.n, row_range=(a, b))
        y = torch.empty(b - a, dtype=torch.float64, device=dev)
        plan.apply_local(xp.data_ptr(), y.data_ptr(),
                         stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        pieces.append(y.cpu().numpy())
        plan.close()
    y = np.concatenate(pieces)
    tol = 1e-13 if scheme == "m1-double" else 1e-6
    assert np.max(np.abs(y - y_full)) <= tol * np.max(np.abs(y_full))


def test_distributed_solver_nccl_world1(hx, cfg):
    """The distributed solver (torch vector arithmetic, NCCL collectives)
    against the device solver on the same operator.  Their vector arithmetic
    differs at the ulp level, so near tol the stop iteration may move: m1-double
    is compared tightly, m2-mixed (which stalls at ~1e-8, where even the
    reference's own reorderings move the stop and the converged flag) loosely."""
    import os

    import torch
    import torch.distributed as dist

    from paper_1911_00093_b200 import distributed as D

    mesh, h, _ = cfg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        slices = D.RowSlices([0, h.n])
        op64, _ = D.make_gpu_operator(h, "m1-double", slices, 0, dev)
        perm = np.asarray(h.permutation)
        b = mesh.centroids[:, 2].copy()
        bl = torch.from_numpy(np.ascontiguousarray(b[perm])).to(dev)
        for scheme in ("m1-double", "m2-mixed"):
            op = op64 if scheme == "m1-double" else D.make_gpu_operator(h, scheme, slices, 0, dev)[0]
            xs, rep = D.bicgstab_distributed(op, op64, bl, tol=1e-8, scheme_label=scheme)
            x_ref, ref = hx.bicgstab(hx.prepare_scheme(h, scheme), h, b, hx.SolverConfig(tol=1e-8))
            x = np.empty(h.n)
            x[perm] = xs.cpu().numpy()
            assert rep.true_residual is not None and ref.true_residual is not None
            assert rep.converged == (rep.true_residual < 1e-8)
            if scheme == "m1-double":
                assert abs(rep.iterations - ref.iterations) <= 2
                assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-6
            else:
                assert abs(rep.iterations - ref.iterations) <= max(3, ref.iterations // 5)
                assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-5
                assert abs(rep.true_residual - ref.true_residual) <= 0.5 * max(rep.true_residual,
                                                                             ref.true_residual)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("local_first", [False, True, "split"])
@pytest.mark.parametrize("scheme", ["m1-double", "m1-mixed", "m2-mixed", "m3:c=1"])
def test_cxx_dist_path_world1_is_the_single_gpu_path(hx, cfg, scheme, local_first, monkeypatch):
    """hmx_dist_matvec and hmx_bicgstab_dist (libhmx_gpu's own NCCL
    communicator, device-side decisions, batched iterations) at world 1 run
    the single-GPU kernels in the same order: bitwise the single-GPU matvec
    and graph-resident solver (solution, history, report).  local_first:
    the plans order stage 1 local-slice first and the stage-1 work on the
    local slice runs on a side stream during the allgather ("split": half of
    stage 1 on each stream, the test hook that exercises both launches)."""
    import torch

    if local_first == "split":
        monkeypatch.setenv("HMX_TEST_SPLIT_STAGE1", "1")

    from paper_1911_00093_b200 import _gpu
    from paper_1911_00093_b200 import distributed as D

    mesh, h, x = cfg
    n = h.n
    perm = np.asarray(h.permutation)
    slices = D.RowSlices([0, n])
    dev = torch.device("cuda", 0)
    comm = D.make_comm(slices, 0, dev)
    sh = hx.prepare_scheme(h, scheme)
    sh64 = hx.prepare_scheme(h, "m1-double")
    lf = bool(local_first)
    plan = _gpu.Plan(sh.packed, h.partition.table, perm, sh.scheme.label, n, row_range=(0, n),
                     local_first=lf)
    plan64 = _gpu.Plan(sh64.packed, h.partition.table, perm, "m1-double", n, row_range=(0, n),
                       local_first=lf)
    try:
        xp = torch.from_numpy(np.ascontiguousarray(x[perm])).to(dev)
        y = torch.empty(n, dtype=torch.float64, device=dev)
        comm.matvec(plan, xp.data_ptr(), y.data_ptr(),
                    stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), hx.matvec(sh, x)[perm])

        b = mesh.centroids[:, 2].copy()
        xl, rep = D.bicgstab_gpu(comm, plan, plan64, b[perm], tol=1e-8, max_iter=1000,
                                 scheme_label=scheme)
        x_ref, ref = hx.bicgstab(sh, h, b, hx.SolverConfig(tol=1e-8))
        assert (rep.iterations, rep.converged, rep.matvecs, rep.breakdown) == \
            (ref.iterations, ref.converged, ref.matvecs, ref.breakdown)
        assert rep.residual_history == ref.residual_history
        assert rep.true_residual == ref.true_residual
        xs = np.empty(n)
        xs[perm] = xl
        assert np.array_equal(xs, x_ref)
    finally:
        plan.close()
        plan64.close()
        comm.close()


def test_cxx_dist_solver_edge_cases_world1(hx, cfg):
    """Zero right-hand side and max_iter exhaustion through hmx_bicgstab_dist
    report like the single-GPU solver (solver.py:92-97, :160-168)."""
    import torch

    from paper_1911_00093_b200 import _gpu
    from paper_1911_00093_b200 import distributed as D

    mesh, h, _ = cfg
    n = h.n
    perm = np.asarray(h.permutation)
    comm = D.make_comm(D.RowSlices([0, n]), 0, torch.device("cuda", 0))
    sh = hx.prepare_scheme(h, "m2-mixed")
    plan = _gpu.Plan(sh.packed, h.partition.table, perm, sh.scheme.label, n, row_range=(0, n))
    try:
        x0, r0 = D.bicgstab_gpu(comm, plan, None, np.zeros(n), tol=1e-8)
        assert r0.converged and r0.iterations == 0 and r0.true_residual == 0.0
        assert np.array_equal(x0, np.zeros(n))
        b = mesh.centroids[:, 2].copy()
        _, rk = D.bicgstab_gpu(comm, plan, None, b[perm], tol=1e-14, max_iter=3)
        _, ref = hx.bicgstab(sh, h, b, hx.SolverConfig(tol=1e-14, max_iter=3))
        assert rk.iterations == ref.iterations == 3 and not rk.converged
        assert rk.residual_history == ref.residual_history
    finally:
        plan.close()
        comm.close()
