"""The multi-GPU mode's host logic on CPU with gloo, world_size 2 and 3: byte-
balanced row partition, padded allgather of the iterate (the one collective
per matvec), allreduced dots, and the distributed BiCG-STAB control flow.
The local product is a CPU stand-in (the oracle restricted to the rank's
rows) injected by the test; on GPUs it is the row-restricted CUDA plan."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, shift=0):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch
    import torch.distributed as dist

    import paper_1911_00093_b200 as hx
    from golden_util import hmatrix_from_fixture, load
    from oracle import hmx_oracle as orc
    from paper_1911_00093_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    arr, meta = load("ref240_aca4")
    h = hmatrix_from_fixture(arr)
    perm = np.asarray(h.permutation)
    table = h.partition.table
    cuts = D.partition_rows(table, h.packed.kinds, h.packed.ranks, h.n, world)
    cuts[1] += shift   # uneven slices whose cut straddles blocks
    slices = D.RowSlices(cuts)
    a, b = slices.span(rank)

    def stand_in(sh):
        def apply(x_full, w1, yy):
            xo = np.empty(h.n)
            xo[perm] = x_full.numpy()
            y = torch.from_numpy(orc.matvec(sh, xo)[perm][a:b].copy())
            d0 = float(torch.dot(y, w1)) if w1 is not None else 0.0
            d1 = float(torch.dot(y, y)) if yy else 0.0
            return y, torch.tensor([d0, d1], dtype=torch.float64)
        return apply

    sh = hx.prepare_scheme(h, "m2-mixed")
    sh64 = hx.prepare_scheme(h, "m1-double")
    op = D.DistributedOperator(slices, rank, local_apply=stand_in(sh))
    op64 = D.DistributedOperator(slices, rank, local_apply=stand_in(sh64))
    # one matvec: gathered local slices reproduce the full product
    x = arr["x"]
    y_local, _ = op.apply(torch.from_numpy(x[perm][a:b].copy()))
    b_local = torch.from_numpy(arr["b"][perm][a:b].copy())
    xs, rep = D.bicgstab_distributed(op, op64, b_local, tol=1e-8, max_iter=200,
                                     scheme_label="m2-mixed")
    np.savez(Path(out_dir) / f"r{rank}.npz", y=y_local.numpy(), x=xs.numpy(), cuts=slices.cuts,
             it=rep.iterations, conv=rep.converged, tres=rep.true_residual,
             hist=np.array(rep.residual_history))
    dist.destroy_process_group()


def test_partition_balances_bytes(hx):
    mesh = hx.jittered_sphere_mesh(4, seed=1)
    h = hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32)
    from paper_1911_00093_b200 import distributed as D
    for world in (2, 4, 8):
        cuts = D.partition_rows(h.partition.table, h.packed.kinds, h.packed.ranks, h.n, world)
        assert cuts[0] == 0 and cuts[-1] == h.n and all(np.diff(cuts) > 0)
        bounds, cum = D.row_costs(h.partition.table, h.packed.kinds, h.packed.ranks, h.n)
        share = np.interp(cuts, bounds, cum)
        parts = np.diff(share)
        assert parts.max() / parts.mean() < 1.10


def test_row_restricted_build_matches_full(hx, orc):
    mesh = hx.jittered_sphere_mesh(3, seed=42)
    full = hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32)
    lo, hi = 320, 960
    part = hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32, rows=(lo, hi))
    t = full.partition.table
    meet = (t[:, 1] > lo) & (t[:, 0] < hi)
    assert np.all(part.packed.kinds[~meet] == 2)
    assert np.array_equal(part.packed.kinds[meet], full.packed.kinds[meet])
    for k in np.flatnonzero(meet)[:50]:
        a, b = full.payloads[k], part.payloads[k]
        if hasattr(a, "values"):
            assert np.array_equal(a.values, b.values)
        else:
            assert np.array_equal(a.u, b.u) and np.array_equal(a.vt, b.vt)
    sh = hx.prepare_scheme(part, "m2-mixed")   # preparation skips unbuilt blocks
    assert sh.packed.kind.tolist().count(2) == int((~meet).sum())


@pytest.mark.parametrize("world,shift", [(2, 0), (3, 7)])
def test_gloo_world2_matvec_and_bicgstab(tmp_path, hx, orc, world, shift):
    """world 2 with the byte-balanced cuts; world 3 with a cut moved 7 rows
    into a leaf (uneven, padded slices; blocks straddling the cut)."""
    import torch.multiprocessing as mp

    from golden_util import hmatrix_from_fixture, load
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path), shift), nprocs=world, join=True,
                       start_method="spawn")
    rs = [np.load(tmp_path / f"r{k}.npz") for k in range(world)]
    arr, _ = load("ref240_aca4")
    h = hmatrix_from_fixture(arr)
    perm = np.asarray(h.permutation)
    sh = hx.prepare_scheme(h, "m2-mixed")
    y_full = np.concatenate([r["y"] for r in rs])
    assert np.array_equal(y_full, orc.matvec(sh, arr["x"])[perm])
    # every rank took the same decisions
    for r in rs[1:]:
        assert int(r["it"]) == int(rs[0]["it"]) and bool(r["conv"]) == bool(rs[0]["conv"])
        assert np.array_equal(r["hist"], rs[0]["hist"])
    # and they match the single-process solve up to the dots' summation order
    xo, ref = orc.bicgstab(sh, hx.prepare_scheme(h, "m1-double"), arr["b"], tol=1e-8)
    assert abs(int(rs[0]["it"]) - ref["iterations"]) <= 1
    assert bool(rs[0]["conv"]) == ref["converged"]
    x = np.empty(h.n)
    x[perm] = np.concatenate([r["x"] for r in rs])
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-6


def _cuts_worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    import json

    import torch.distributed as dist

    import paper_1911_00093_b200 as hx
    from paper_1911_00093_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mesh = hx.jittered_sphere_mesh(4, seed=42)
    part = hx.build_block_partition(hx.build_cluster_tree(mesh, 32), 2.0)
    cuts = D.measured_cuts(mesh, part, aca_tol=1e-4, world=world, rank=rank)
    Path(out_dir, f"cuts{rank}.json").write_text(json.dumps(cuts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_measured_cuts_match_the_full_build(tmp_path, world):
    """distributed.measured_cuts (estimate cut, row-restricted builds, real
    ranks exchanged, re-cut) gives every rank the cuts partition_rows makes
    from the FULL build's stored bytes (balanced by stored bytes)."""
    import json

    import torch.multiprocessing as mp

    import paper_1911_00093_b200 as hx
    from paper_1911_00093_b200 import distributed as D

    mp.spawn(_cuts_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = [json.loads((tmp_path / f"cuts{r}.json").read_text()) for r in range(world)]
    mesh = hx.jittered_sphere_mesh(4, seed=42)
    h = hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32)
    want = D.partition_rows(h.partition.table, h.packed.kinds, h.packed.ranks, h.n, world)
    assert all(g == want for g in got), (got, want)
