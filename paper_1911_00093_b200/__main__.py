"""`python -m paper_1911_00093_b200 bench matvec|solve ...` -- the reference
CLI's `bench` subcommand (reference cli.py:160-209: same geometry / build /
sweep flags) run on the GPU, emitting the reference's BenchRecord CSV/JSON
schema plus the GPU columns.  `--device k` picks the
CUDA device; `--cpu-report PATH` merges a report written by the reference's
own CLI so both sit in one table with speedups against CPU m1-double.
"""

from __future__ import annotations

import argparse
import sys


def _list(conv):
    return lambda text: tuple(conv(t.strip()) for t in text.split(",") if t.strip())


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_1911_00093_b200",
                                 description="B200 H-matrix benchmark sweeps (the reference's "
                                             "bench subcommand on the GPU).")
    sub = ap.add_subparsers(dest="command", required=True)
    b = sub.add_parser("bench", help="run a benchmark sweep on the GPU")
    b.add_argument("mode", choices=("matvec", "solve"))
    g = b.add_argument_group("geometry")
    g.add_argument("--spheres", type=int, default=3)
    g.add_argument("--refine", type=int, default=2)
    g.add_argument("--spacing", type=float, default=3.0)
    g.add_argument("--radius", type=float, default=1.0)
    g.add_argument("--voltages", type=_list(float), default=None)
    m = b.add_argument_group("matrix build")
    m.add_argument("--aca-tol", type=float, default=1e-8)
    m.add_argument("--leaf", type=int, default=32)
    m.add_argument("--eta", type=float, default=2.0)
    m.add_argument("--max-rank", type=int, default=None)
    b.add_argument("--schemes", type=_list(str), default=("all",))
    b.add_argument("--c-list", type=_list(int), default=())
    b.add_argument("--reps", type=int, default=1000)
    b.add_argument("--sets", type=int, default=10)
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--tol", type=float, default=1e-6)
    b.add_argument("--max-iter", type=int, default=1000)
    b.add_argument("--device", type=int, default=0, help="CUDA device")
    b.add_argument("--format", choices=("csv", "json"), default="csv")
    b.add_argument("--out", default=None, help="output file (default: stdout)")
    b.add_argument("--cpu-report", default=None,
                   help="a report of the reference's CLI to merge (speedups against CPU m1-double)")
    return ap


def main(argv=None) -> int:
    import numpy as np

    from . import benchrec as br

    args = build_parser().parse_args(argv)
    try:
        cfg = br.BenchConfig(spheres=args.spheres, refinement=args.refine, spacing=args.spacing,
                             radius=args.radius, voltages=args.voltages, aca_tol=args.aca_tol,
                             leaf_size=args.leaf, eta=args.eta, max_rank=args.max_rank,
                             schemes=args.schemes, c_list=args.c_list, reps=args.reps,
                             sets=args.sets, seed=args.seed, tol=args.tol, max_iter=args.max_iter,
                             device=args.device)
        run = br.run_matvec_bench if args.mode == "matvec" else br.run_solver_bench
        records = run(cfg)
        if args.cpu_report:
            records = br.merge_speedups(br.read_report(args.cpu_report), records)
        text = br.emit_report(records, format=args.format, path=args.out)
        if args.out is None:
            sys.stdout.write(text)
        return 0
    except (ValueError, OverflowError, FloatingPointError, OSError, RuntimeError,
            np.linalg.LinAlgError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
