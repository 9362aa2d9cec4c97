"""Multi-GPU H-matvec and BiCG-STAB (BASELINE.json north_star item 4).

One process per GPU.  The permuted row space is cut at leaf boundaries into
contiguous slices balanced by the payload bytes each slice reads (dense rows,
U rows, and the Vt rows of every low-rank block the slice touches).  Each rank
builds only the blocks meeting its rows (compress.build_hmatrix(rows=...)),
and holds a row-restricted device plan (hmx_plan_options / hmx_apply_local).

Per matvec there is exactly one collective: an allgather of the iterate's
slices into the full permuted vector every rank's stage 1 reads.  BiCG-STAB
dot products are local partial sums (fused into the stage-2 epilogue on the
GPU) finished by one small allreduce per reduction point.  Control flow
mirrors reference pkg/src/hmx/solver.py:68-168 on every rank (identical
scalars after the allreduces), so all ranks take the same decisions.

Two implementations of that protocol:

* the GPU product path (`make_comm`, `bicgstab_gpu`, `bench_main`):
  libhmx_gpu.so's own NCCL communicator (hmx_comm_create), the allgather as
  grouped NCCL send/recv straight into the full vector (uneven slices, no
  padding or copies; hmx_dist_matvec), and the whole BiCG-STAB iteration in
  C++/CUDA (hmx_bicgstab_dist): the single-GPU fused vector kernels on local
  rows, scalars and every decision on the device, iterations enqueued in
  guarded batches -- no host synchronisation per matvec;
* `DistributedOperator` / `bicgstab_distributed`: the same protocol written
  with torch.distributed collectives and torch vector arithmetic, whose
  local product is injectable.  It runs the multi-process tests on CPU
  (gloo, world 2, tests/test_distributed_gloo.py) with a CPU stand-in for
  the local product.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .solver import SolverReport, _breakdown_message

_EPS = 1e-300  # reference solver.py:27


# ---------------------------------------------------------------------------
# row partition

def leaf_boundaries(table: np.ndarray, n: int) -> np.ndarray:
    """Sorted unique row boundaries of all blocks (the leaf row clusters)."""
    return np.unique(np.concatenate([[0, n], table[:, 0], table[:, 1]]))


def row_costs(table: np.ndarray, kinds: np.ndarray, ranks: np.ndarray, n: int,
              bytes_per_elem: float = 8.0):
    """Bytes a rank reads per leaf interval if it owns that interval: dense and
    U rows, plus the Vt of each low-rank block spread over its rows (a block
    cut between ranks has its Vt read by both; the cut search avoids that)."""
    bounds = leaf_boundaries(table, n)
    m = table[:, 1] - table[:, 0]
    w = table[:, 3] - table[:, 2]
    per_row = np.zeros(n + 1)
    dense = kinds == 0
    low = kinds == 1
    rate = np.where(dense, w, 0.0) + np.where(low, ranks * (1.0 + w / np.maximum(m, 1)), 0.0)
    np.add.at(per_row, table[:, 0], rate)
    np.add.at(per_row, table[:, 1], -rate)
    dens = np.cumsum(per_row)[:n]
    pref = np.concatenate([[0.0], np.cumsum(dens)]) * bytes_per_elem
    return bounds, pref[bounds]


def partition_rows(table: np.ndarray, kinds: np.ndarray, ranks: np.ndarray, n: int,
                   world: int) -> list[int]:
    """Cut points r_0 = 0 < r_1 < ... < r_world = n at leaf boundaries with
    balanced bytes; prefers cuts that no block straddles (tree-aligned).
    O(blocks + n): straddled boundaries come from a difference array."""
    if world == 1:
        return [0, n]
    if world > n:
        raise ValueError(f"cannot cut {n} rows into {world} non-empty slices")
    bounds, cum = row_costs(table, kinds, ranks, n)
    total = cum[-1]
    # boundary b is straddled when some block has rs < b < re: count the
    # blocks covering each row index in (rs, re) with a difference array
    cover = np.zeros(n + 2, dtype=np.int64)
    np.add.at(cover, table[:, 0] + 1, 1)
    np.add.at(cover, table[:, 1], -1)
    clean = np.cumsum(cover)[bounds] == 0
    cand = np.flatnonzero(clean)
    cuts = [0]
    for k in range(1, world):
        target = total * k / world
        j = cand[np.argmin(np.abs(cum[cand] - target))] if cand.size else 0
        # accept a straddled boundary if a clean one is more than 5% off
        if not cand.size or abs(cum[j] - target) > 0.05 * total / world:
            j = int(np.argmin(np.abs(cum - target)))
        # strictly increasing, and room left for the remaining ranks
        cuts.append(int(min(max(bounds[j], cuts[-1] + 1), n - (world - k))))
    cuts.append(n)
    return cuts


def measured_cuts(mesh, partition, aca_tol: float, world: int, rank: int, group=None,
                  device=None) -> list[int]:
    """Row cuts balanced on the MEASURED stored bytes: cut on an
    estimate (rank 11 per admissible block), build this rank's rows, take the
    real ranks of every block from the rank(s) that built it (an allreduce
    max over the group: a block meeting several slices has the same rank on
    each), and cut again on them.  Collective over `group`."""
    import torch
    import torch.distributed as dist

    from .compress import build_hmatrix

    table = partition.table
    kinds = table[:, 4].astype(np.int32)
    n = int(mesh.n)
    if world == 1:
        return [0, n]
    est = np.where(kinds == 1, 11, 0)
    cuts0 = partition_rows(table, kinds, est, n, world)
    h0 = build_hmatrix(mesh, partition=partition, aca_tol=aca_tol, rows=(cuts0[rank], cuts0[rank + 1]))
    built = np.asarray(h0.packed.kinds) != 2
    r = np.where(built, np.asarray(h0.packed.ranks), 0).astype(np.int64)
    t = torch.from_numpy(r)
    if device is not None and dist.get_backend(group) == "nccl":
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    ranks = t.cpu().numpy()
    return partition_rows(table, kinds, ranks, n, world)


@dataclass
class RowSlices:
    """Row cuts of the permuted index space, one contiguous slice per rank (`cuts[r]:cuts[r+1]`)."""
    cuts: list

    @property
    def world(self):
        return len(self.cuts) - 1

    def span(self, rank):
        return self.cuts[rank], self.cuts[rank + 1]

    @property
    def padded(self):
        return max(self.cuts[k + 1] - self.cuts[k] for k in range(self.world))


# ---------------------------------------------------------------------------
# distributed operator

class DistributedOperator:
    """Rows [r0, r1) of one scheme's operator on this rank.

    `local_apply(x_full, w1, yy) -> (y_local, (y.w1, y.y))` computes the local
    rows; by default the row-restricted GPU plan (hmx_apply_local), with the
    dots fused into the stage-2 epilogue.
    """

    def __init__(self, slices: RowSlices, rank: int, group=None, device=None,
                 local_apply=None, plan=None):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.dist = dist
        self.slices = slices
        self.rank = rank
        self.group = group
        self.r0, self.r1 = slices.span(rank)
        self.n = slices.cuts[-1]
        self.device = device if device is not None else torch.device("cpu")
        self.plan = plan
        self.local_apply = local_apply or self._gpu_apply
        L = slices.padded
        self._pad_in = torch.zeros(L, dtype=torch.float64, device=self.device)
        self._gathered = torch.zeros(L * slices.world, dtype=torch.float64, device=self.device)
        self._full = torch.zeros(self.n, dtype=torch.float64, device=self.device)
        # position of every permuted index in the padded allgather buffer
        # (one index_select un-pads it)
        self._unpad = torch.cat([torch.arange(k * L, k * L + (b - a), dtype=torch.int64)
                                 for k, (a, b) in enumerate(slices.span(q) for q in range(slices.world))]
                                ).to(self.device)
        if plan is not None:
            self._dots = torch.zeros(2, dtype=torch.float64, device=self.device)
            self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)

    def gather(self, x_local):
        """The ONE collective per matvec: allgather of the iterate's slices."""
        m = self.r1 - self.r0
        self._pad_in[:m].copy_(x_local)
        self.dist.all_gather_into_tensor(self._gathered, self._pad_in, group=self.group)
        self.torch.index_select(self._gathered, 0, self._unpad, out=self._full)
        return self._full

    def _gpu_apply(self, x_full, w1, yy):
        torch = self.torch
        y = torch.empty(self.r1 - self.r0, dtype=torch.float64, device=self.device)
        self._flag.zero_()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.plan.apply_local(x_full.data_ptr(), y.data_ptr(),
                              w1.data_ptr() if w1 is not None else 0, yy,
                              self._dots.data_ptr(), self._flag.data_ptr(), stream)
        return y, self._dots, self._flag

    def apply(self, x_local, w1=None, yy=False):
        """y_local = (A x)[r0:r1] and global dots [y.w1, y.y] (allreduced)."""
        torch = self.torch
        x_full = self.gather(x_local)
        out = self.local_apply(x_full, w1, yy)
        y, dots = out[0], out[1]
        flag = out[2] if len(out) > 2 else None
        red = torch.zeros(3, dtype=torch.float64, device=self.device)
        red[:2] = dots
        if flag is not None:
            red[2] = flag.to(torch.float64)[0]
        else:
            red[2] = float(not bool(torch.isfinite(y).all()))
        self.dist.all_reduce(red, group=self.group)
        if red[2].item() != 0.0:
            raise FloatingPointError("non-finite matvec result")
        return y, red[:2]


def _allsum(op, *vals):
    torch = op.torch
    t = torch.stack([v if torch.is_tensor(v) else torch.tensor(v, dtype=torch.float64,
                                                                device=op.device) for v in vals])
    op.dist.all_reduce(t, group=op.group)
    return [float(v) for v in t.tolist()]


def bicgstab_distributed(op: DistributedOperator, op64: DistributedOperator, b_local, tol=1e-6,
                         max_iter=1000, scheme_label=""):
    """BiCG-STAB with the reference's control flow (solver.py:68-168) on row
    slices.  Returns (x_local, SolverReport) identical on every rank."""
    torch = op.torch
    t0 = time.perf_counter()
    b = b_local
    nb = float(np.sqrt(_allsum(op, torch.dot(b, b))[0]))
    if nb == 0.0:
        return torch.zeros_like(b), SolverReport(scheme_label, True, 0, [0.0], 0.0,
                                                 time.perf_counter() - t0)
    x = torch.zeros_like(b)
    ax, _ = op.apply(x)
    r = b - ax
    r_hat = r.clone()
    rr = _allsum(op, torch.dot(r, r))[0]
    hist = [float(np.sqrt(rr)) / nb]
    converged, breakdown, tres, its = False, None, None, 0
    rho_prev = alpha = omega = 1.0
    p = v = None
    rho = _allsum(op, torch.dot(r_hat, r))[0]

    def true_res(xv):
        y, _ = op64.apply(xv)
        e = b - y
        ne, nb2 = _allsum(op64, torch.dot(e, e), torch.dot(b, b))
        nr, nbb = float(np.sqrt(ne)), float(np.sqrt(nb2))
        return 0.0 if nbb == 0.0 and nr == 0.0 else (float("inf") if nbb == 0.0 else nr / nbb)

    for i in range(1, max_iter + 1):
        if abs(rho) < _EPS:
            breakdown = _breakdown_message(1, rho, i)
            break
        if i == 1:
            p = r.clone()
        else:
            beta = (rho / rho_prev) * (alpha / omega)
            p = r + beta * (p - omega * v)
        v, d = op.apply(p, w1=r_hat)
        denom = float(d[0])
        if abs(denom) < _EPS:
            breakdown = _breakdown_message(2, denom, i)
            break
        alpha = rho / denom
        s = r - alpha * v
        s_rel = float(np.sqrt(_allsum(op, torch.dot(s, s))[0])) / nb
        if s_rel < tol:
            x = x + alpha * p
            hist.append(s_rel)
            its = i
            tres = true_res(x)
            converged = tres < tol
            break
        t, d = op.apply(s, w1=s, yy=True)
        ts, tt = float(d[0]), float(d[1])
        if tt == 0.0:
            breakdown = _breakdown_message(3, 0.0, i)
            break
        omega = ts / tt
        x = x + alpha * p + omega * s
        r = s - omega * t
        rr, rho_next = _allsum(op, torch.dot(r, r), torch.dot(r_hat, r))
        rel = float(np.sqrt(rr)) / nb
        hist.append(rel)
        its = i
        if rel < tol:
            tres = true_res(x)
            converged = tres < tol
            break
        if abs(omega) < _EPS:
            breakdown = _breakdown_message(4, omega, i)
            break
        rho_prev, rho = rho, rho_next
    return x, SolverReport(scheme=scheme_label, converged=converged, iterations=its,
                           residual_history=hist, true_residual=tres,
                           wall_time_s=time.perf_counter() - t0, breakdown=breakdown)


# ---------------------------------------------------------------------------
# GPU setup and benchmark (torchrun, one rank per GPU)

def make_comm(slices: RowSlices, rank: int, device, group=None):
    """This rank's libhmx_gpu NCCL communicator over the row slices.  The
    NCCL unique id is made on rank 0 and broadcast through the
    torch.distributed group (any backend) when world > 1."""
    from . import _gpu

    uid = _gpu.Comm.unique_id() if rank == 0 else None
    if slices.world > 1:
        import torch.distributed as dist
        box = [uid]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = box[0]
    index = device.index if hasattr(device, "index") else int(device)
    return _gpu.Comm(uid, slices.world, rank, index or 0, slices.cuts)


def bicgstab_gpu(comm, plan, plan64, b_local, tol=1e-6, max_iter=1000, scheme_label=""):
    """BiCG-STAB on this rank's rows through hmx_bicgstab_dist.  b_local is
    this rank's slice of b in permuted order (host array); returns
    (x_local, SolverReport), the report identical on every rank."""
    from . import _gpu

    t0 = time.perf_counter()
    x, rep, hist, rc = comm.bicgstab(plan, plan64, b_local, tol, max_iter)
    wall = time.perf_counter() - t0
    if rc == _gpu.HMX_ERR_NONFINITE:
        raise FloatingPointError("non-finite matvec result")
    return x, SolverReport(
        scheme=scheme_label, converged=bool(rep.converged), iterations=int(rep.iterations),
        residual_history=[float(v) for v in hist[:rep.history_len]],
        true_residual=float(rep.true_residual) if rep.has_true_residual else None,
        wall_time_s=wall,
        breakdown=_breakdown_message(rep.breakdown, rep.breakdown_value, rep.breakdown_iteration),
        device_time_s=rep.device_ms / 1e3, matvecs=int(rep.matvecs))


def make_gpu_operator(h, scheme: str, slices: RowSlices, rank: int, device, group=None):
    """Row-restricted device plan of `scheme` for this rank."""
    from . import _gpu
    from .precision import prepare_scheme

    sh = prepare_scheme(h, scheme)
    plan = _gpu.Plan(sh.packed, h.partition.table, np.asarray(h.permutation), sh.scheme.label,
                     h.n, device=device.index or 0, row_range=slices.span(rank), local_first=True)
    return DistributedOperator(slices, rank, group=group, device=device, plan=plan), sh


def bench_main(args, build_workload, workload_name, metric):
    """bench.py --gpus N under torchrun: the whole-job matvec rate of the
    row-partitioned operator (one allgather per matvec), max over ranks.
    Same JSON contract as the single-GPU line (roofline of rank 0's stage-2
    kernel, end-to-end rate with host slices, clocks of rank 0's GPU)."""
    import json
    import os

    import torch
    import torch.distributed as dist

    import bench as bench_mod
    from .compress import build_hmatrix
    from .partition import build_block_partition, build_cluster_tree
    from .problem import jittered_sphere_mesh, right_hand_side

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", device_id=device, rank=rank, world_size=world)
    c = bench_mod.CONFIGS[args.config]
    t0 = time.perf_counter()
    mesh = jittered_sphere_mesh(c["level"], seed=42, centers=c.get("centers", ((0.0, 0.0, 0.0),)),
                                voltages=c.get("voltages"))
    part = build_block_partition(build_cluster_tree(mesh, c["leaf"]), 2.0)
    # cut on the measured stored bytes (an estimate cut, a build, the real
    # ranks exchanged, a re-cut)
    slices = RowSlices(measured_cuts(mesh, part, c["aca"], world, rank, device=device))
    h = build_hmatrix(mesh, partition=part, aca_tol=c["aca"], rows=slices.span(rank))
    t_build = time.perf_counter() - t0
    peak, peak_src = bench_mod.measured_peak()
    a, b_ = slices.span(rank)
    x_np = np.random.default_rng(42).uniform(-1.0, 1.0, mesh.n)
    perm = np.asarray(h.permutation)
    x_host = torch.from_numpy(np.ascontiguousarray(x_np[perm[a:b_]])).pin_memory()
    y_host = torch.empty(b_ - a, dtype=torch.float64).pin_memory()
    b_full = right_hand_side(mesh) if c.get("voltages") else mesh.centroids[:, 2].copy()
    b_local = np.ascontiguousarray(b_full[perm[a:b_]])
    comm = make_comm(slices, rank, device)
    y_dev = torch.empty(b_ - a, dtype=torch.float64, device=device)
    results, clocks, headline = {}, None, None
    op64 = None

    def step(op, x_local):
        # the one allgather (NCCL send/recv into the full vector) + local product
        comm.matvec(op.plan, x_local.data_ptr(), y_dev.data_ptr(),
                    stream=torch.cuda.current_stream(device).cuda_stream)
        return y_dev

    def timed(fn, k):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / k], device=device)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms)

    names = [bench_mod.HEADLINE] + [s for s in args.variants if s != bench_mod.HEADLINE][:1]
    for name in names:
        op, sh = make_gpu_operator(h, name, slices, rank, device)
        x_local = x_host.to(device)
        for _ in range(args.warmup):
            step(op, x_local)
        if name == bench_mod.HEADLINE and rank == 0:
            with bench_mod.ClockSampler(local) as clk:
                ms = timed(lambda: step(op, x_local), args.steps)
            clocks = clk.summary()
        else:
            ms = timed(lambda: step(op, x_local), args.steps)
        local_bytes = torch.tensor([float(op.plan.info()["payload_bytes"])], device=device)
        dist.all_reduce(local_bytes)
        r = op.plan.bench(3, max(10, args.steps // 2))  # local two-stage product alone
        info = op.plan.info()
        entry = {"ms": ms, "matvec_per_s": 1e3 / ms, "payload_bytes_all_ranks": float(local_bytes),
                 "local_ms_rank0": r["ms"], "stage1_ms_rank0": r["stage1_ms"],
                 "stage2_ms_rank0": r["stage2_ms"], "rows_rank0": b_ - a}
        if not args.no_solve:
            if op64 is None:
                op64 = op if name == bench_mod.HEADLINE else make_gpu_operator(
                    h, bench_mod.HEADLINE, slices, rank, device)[0]
            dist.barrier()
            _, srep = bicgstab_gpu(comm, op.plan, op64.plan, b_local, tol=1e-8, max_iter=1000,
                                   scheme_label=name)
            t_solve = torch.tensor([srep.device_time_s], device=device)
            dist.all_reduce(t_solve, op=dist.ReduceOp.MAX)
            entry["solve"] = {"iterations": srep.iterations, "converged": srep.converged,
                              "true_residual": srep.true_residual,
                              "device_s_max_over_ranks": float(t_solve),
                              "matvecs": srep.matvecs, "breakdown": srep.breakdown}
        if name == bench_mod.HEADLINE:
            # end to end: this rank's x slice from pinned host memory, the
            # allgather, the local product, its y slice back to the host
            def e2e_step():
                x_local.copy_(x_host, non_blocking=True)
                y = step(op, x_local)
                y_host.copy_(y, non_blocking=True)
            e2e_ms = timed(e2e_step, max(5, min(args.steps, 50)))
            entry["e2e_ms"] = e2e_ms
            s2_bytes = info["stage2_bytes"] + 8 * (b_ - a)
            headline = (entry, s2_bytes, r, info)
        results[name] = entry
        if op is not op64:
            op.plan.close()
    if op64 is not None:
        op64.plan.close()
    comm.close()
    dist.barrier()
    if rank == 0:
        entry, s2_bytes, r, info = headline
        ms = entry["ms"]
        dom = s2_bytes / (r["stage2_ms"] * 1e6)
        print(json.dumps({
            "metric": metric, "value": 1e3 / ms, "unit": "matvec/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded jittered icosphere, BASELINE.json recipe)",
            "config": {"workload": workload_name(args.config), "scheme": bench_mod.HEADLINE,
                       "n": int(mesh.n), "parallelism": f"row partition x{world}",
                       "cuts": slices.cuts, "build_s": t_build,
                       "l2": "per-rank payload >> 126 MB L2 at configs 4-5 (no flush)"},
            "roofline": {"bound": "hbm", "achieved": dom, "peak": peak, "unit": "GB/s",
                         "frac": dom / peak, "traffic": None, "peak_source": peak_src,
                         "kernel": "rank 0 stage-2 seg_kernel (local rows)",
                         "algorithmic_bytes_per_launch": s2_bytes},
            "cpu_baseline": None,
            "e2e": {"value": 1e3 / entry["e2e_ms"], "unit": "matvec/s",
                    "h2d_bytes_per_step": 8 * int(mesh.n), "d2h_bytes_per_step": 8 * int(mesh.n)},
            # our kernels per step: stage 1 (at world > 1 two launches: the
            # local-first segments on the side stream, the rest after the
            # allgather) and stage 2; NCCL's own kernels not counted
            "gpu_launches": (3 if world > 1 else 2) * args.steps, "clocks": clocks,
            "variants": results,
            "note": "each step = one NCCL allgather of the iterate (grouped send/recv into the "
                    "full vector) + the local two-stage product; solves: hmx_bicgstab_dist; "
                    "cpu_baseline is reported by the N=1 run",
        }), flush=True)
    dist.destroy_process_group()
