"""`python -m paper_1911_00093_b200 info|solve|bench ...` -- the reference
CLI's subcommands (reference cli.py:58-226: same geometry / build / sweep
flags, same exit codes) on the GPU path:

* `info`   builds the H-matrix (`--gpu-build`: compressed on the device) and
           prints its report; `--dump-partition` / `--export-mesh` write the
           reference's interchange formats;
* `solve`  one BiCG-STAB solve on the device (exit 0 converged, 3 not);
* `bench`  matvec or solve sweeps emitting the reference's BenchRecord
           CSV/JSON schema plus the GPU columns; `--cpu-report PATH` merges
           a report of the reference's own CLI (speedups against CPU
           m1-double).

`--device k` picks the CUDA device.
"""

from __future__ import annotations

import argparse
import json
import sys


def _list(conv):
    return lambda text: tuple(conv(t.strip()) for t in text.split(",") if t.strip())


def _geometry_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(add_help=False)
    g = p.add_argument_group("geometry")
    g.add_argument("--spheres", type=int, default=3)
    g.add_argument("--refine", type=int, default=2)
    g.add_argument("--spacing", type=float, default=3.0)
    g.add_argument("--radius", type=float, default=1.0)
    g.add_argument("--voltages", type=_list(float), default=None)
    m = p.add_argument_group("matrix build")
    m.add_argument("--aca-tol", type=float, default=1e-8)
    m.add_argument("--leaf", type=int, default=32)
    m.add_argument("--eta", type=float, default=2.0)
    m.add_argument("--max-rank", type=int, default=None)
    m.add_argument("--device", type=int, default=0, help="CUDA device")
    m.add_argument("--gpu-build", action="store_true", help="compress the H-matrix on the GPU")
    return p


def build_parser() -> argparse.ArgumentParser:
    """Argument parser of the `info` / `solve` / `bench` subcommands (reference cli.py:160-210)."""
    geo = _geometry_parser()
    ap = argparse.ArgumentParser(prog="python -m paper_1911_00093_b200",
                                 description="B200 H-matrix matvec / BiCG-STAB (the reference "
                                             "hmx CLI on the GPU path).")
    sub = ap.add_subparsers(dest="command", required=True)
    i = sub.add_parser("info", parents=[geo], help="build the H-matrix and print its report")
    i.add_argument("--json", action="store_true")
    i.add_argument("--dump-partition", metavar="PATH", default=None)
    i.add_argument("--export-mesh", metavar="PATH", default=None)
    s = sub.add_parser("solve", parents=[geo], help="run one BiCG-STAB solve on the GPU")
    s.add_argument("--scheme", default="m1-double")
    s.add_argument("--tol", type=float, default=1e-6)
    s.add_argument("--max-iter", type=int, default=1000)
    s.add_argument("--json", action="store_true")
    b = sub.add_parser("bench", parents=[geo], help="run a benchmark sweep on the GPU")
    b.add_argument("mode", choices=("matvec", "solve"))
    b.add_argument("--schemes", type=_list(str), default=("all",))
    b.add_argument("--c-list", type=_list(int), default=())
    b.add_argument("--reps", type=int, default=1000)
    b.add_argument("--sets", type=int, default=10)
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--tol", type=float, default=1e-6)
    b.add_argument("--max-iter", type=int, default=1000)
    b.add_argument("--format", choices=("csv", "json"), default="csv")
    b.add_argument("--out", default=None, help="output file (default: stdout)")
    b.add_argument("--cpu-report", default=None,
                   help="a report of the reference's CLI to merge (speedups against CPU m1-double)")
    return ap


def _problem(args):
    from . import build_hmatrix, build_sphere_mesh
    from .problem import axis_centers
    mesh = build_sphere_mesh(axis_centers(args.spheres, args.spacing), radius=args.radius,
                             refinement=args.refine, voltages=args.voltages)
    h = build_hmatrix(mesh, aca_tol=args.aca_tol, max_rank=args.max_rank, leaf_size=args.leaf,
                      eta=args.eta, device=args.device if args.gpu_build else None)
    return mesh, h


def _cmd_info(args) -> int:
    from . import dump_partition, export_mesh
    mesh, h = _problem(args)
    if args.dump_partition:
        dump_partition(h.partition, args.dump_partition)
    if args.export_mesh:
        export_mesh(mesh, args.export_mesh)
    rep = h.report
    if args.json:
        print(json.dumps(rep.to_dict(), indent=2))
        return 0
    print(f"panels: {rep.n}")
    print(f"blocks: {rep.dense_blocks + rep.lowrank_blocks} ({rep.dense_blocks} dense, "
          f"{rep.lowrank_blocks} low-rank, {rep.fallback_blocks} fallbacks)")
    hist = " ".join(f"{r}:{c}" for r, c in sorted(rep.rank_histogram.items()))
    print(f"rank histogram: {hist or '(none)'}")
    print(f"stored scalars: {rep.stored_scalars} (compression ratio {rep.compression_ratio:.4f})")
    print(f"aca tol: {rep.aca_tol:g}")
    return 0


def _cmd_solve(args) -> int:
    import dataclasses
    import os

    import numpy as np

    from . import SolverConfig, bicgstab, prepare_scheme, right_hand_side
    os.environ["HMX_DEVICE"] = str(args.device)
    mesh, h = _problem(args)
    x, rep = bicgstab(prepare_scheme(h, args.scheme), h, right_hand_side(mesh),
                      SolverConfig(tol=args.tol, max_iter=args.max_iter))
    if args.json:
        out = dataclasses.asdict(rep)
        out["solution_norm"] = float(np.linalg.norm(x))
        print(json.dumps(out, indent=2))
    else:
        print(f"scheme: {rep.scheme}")
        print(f"converged: {rep.converged}")
        print(f"iterations: {rep.iterations}")
        res = rep.true_residual
        print(f"true residual: {res if res is not None else 'not evaluated'}")
        print(f"wall time: {rep.wall_time_s:.3f} s (device {rep.device_time_s:.4f} s)")
        if rep.breakdown:
            print(f"breakdown: {rep.breakdown}")
    return 0 if rep.converged else 3


def _cmd_bench(args) -> int:
    from . import benchrec as br
    cfg = br.BenchConfig(spheres=args.spheres, refinement=args.refine, spacing=args.spacing,
                         radius=args.radius, voltages=args.voltages, aca_tol=args.aca_tol,
                         leaf_size=args.leaf, eta=args.eta, max_rank=args.max_rank,
                         schemes=args.schemes, c_list=args.c_list, reps=args.reps, sets=args.sets,
                         seed=args.seed, tol=args.tol, max_iter=args.max_iter, device=args.device)
    run = br.run_matvec_bench if args.mode == "matvec" else br.run_solver_bench
    records = run(cfg)
    if args.cpu_report:
        records = br.merge_speedups(br.read_report(args.cpu_report), records)
    text = br.emit_report(records, format=args.format, path=args.out)
    if args.out is None:
        sys.stdout.write(text)
    else:
        print(f"wrote {len(records)} records to {args.out}")
    return 0


def main(argv=None) -> int:
    """CLI entry point; returns the process exit code (reference cli.py:212-226: 1 on a reported error)."""
    import numpy as np

    args = build_parser().parse_args(argv)
    run = {"info": _cmd_info, "solve": _cmd_solve, "bench": _cmd_bench}[args.command]
    try:
        return run(args)
    except (ValueError, OverflowError, FloatingPointError, OSError, RuntimeError,
            np.linalg.LinAlgError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
