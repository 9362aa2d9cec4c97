"""Report schema of the GPU bench drivers (reference bench.py record format)
and the on-disk H-matrix cache."""

import numpy as np
import pytest

from paper_1911_00093_b200 import benchrec as B


def _rec(scheme, t, device="", **kw):
    return B.BenchRecord(scheme=scheme, threads=1, mean_time_s=t, stddev_s=t / 10,
                         payload_bytes=1000, iterations=None, true_residual=None,
                         speedup=1.0, device=device, **kw)


def test_report_roundtrip_csv_json(tmp_path):
    recs = [_rec("m1-double", 1.23456789012e-3, "cuda:0", matvecs_per_s=810.0,
                 achieved_GBps=6000.5, roofline_frac=0.91, algorithmic_bytes=123),
            _rec("m2-mixed", 6.7e-4, "cuda:0", matvecs_per_s=1500.0)]
    for fmt, name in (("csv", "r.csv"), ("json", "r.json")):
        B.emit_report(recs, fmt, tmp_path / name)
        back = B.read_report(tmp_path / name)
        assert back == recs
    # records round to nine significant digits on construction
    assert recs[0].mean_time_s == float("1.23456789e-3")


def test_reference_style_report_is_readable(tmp_path):
    text = ("scheme,threads,mean_time_s,stddev_s,payload_bytes,iterations,true_residual,speedup\n"
            "m1-double,1,0.25,0.01,238608640,,,1\n")
    p = tmp_path / "cpu.csv"
    p.write_text(text)
    cpu = B.read_report(p)
    assert cpu[0].scheme == "m1-double" and cpu[0].device == ""
    merged = B.merge_speedups(cpu, [_rec("m1-double", 0.0005, "cuda:0")])
    assert merged[1].speedup == pytest.approx(500.0)
    assert B.emit_report(cpu).splitlines()[0] == ",".join(B.CSV_COLUMNS)
    with pytest.raises(ValueError):
        B.emit_report([])


def test_scheme_labels_baseline_first():
    cfg = B.BenchConfig(schemes=("m2-mixed",), c_list=(3, -1))
    assert B.scheme_labels(cfg) == ["m1-double", "m2-mixed", "m3:c=3", "m3:c=-1"]


def test_hmatrix_cache_roundtrip(tmp_path, hx, orc):
    mesh = hx.jittered_sphere_mesh(2, seed=5)
    h = hx.build_hmatrix(mesh, aca_tol=1e-5)
    B.save_hmatrix(h, tmp_path / "h.npz")
    g = B.load_hmatrix(tmp_path / "h.npz")
    assert np.array_equal(g.permutation, h.permutation)
    assert np.array_equal(g.partition.table, h.partition.table)
    x = np.random.default_rng(1).uniform(-1, 1, h.n)
    for s in ("m1-double", "m3:c=1"):
        assert np.array_equal(orc.matvec(hx.prepare_scheme(g, s), x),
                              orc.matvec(hx.prepare_scheme(h, s), x))


@pytest.mark.gpu
def test_gpu_bench_drivers(hx):
    cfg = B.BenchConfig(refinement=1, aca_tol=1e-6, schemes=("m2-mixed",), reps=20, sets=3,
                        tol=1e-8, max_iter=200)
    recs = B.run_matvec_bench(cfg)
    assert [r.scheme for r in recs] == ["m1-double", "m2-mixed"]
    assert all(r.mean_time_s > 0 and r.device == "cuda:0" and r.matvecs_per_s > 0 for r in recs)
    assert recs[0].speedup == 1.0
    srec = B.run_solver_bench(cfg)
    assert all(r.iterations and r.true_residual is not None for r in srec)
    assert "achieved_GBps" in B.emit_report(recs)


def test_cli_parser_and_no_gpu_error(capsys):
    """`python -m paper_1911_00093_b200 bench ...` (the reference CLI's bench
    subcommand on the GPU): flags parse like the reference's; without a GPU
    it reports the error and exits 1 instead of computing on the CPU."""
    from paper_1911_00093_b200 import _gpu
    from paper_1911_00093_b200.__main__ import build_parser, main
    args = build_parser().parse_args(["bench", "matvec", "--schemes", "m1-double,m2-mixed",
                                      "--c-list", "1,3", "--refine", "1", "--device", "0"])
    assert args.schemes == ("m1-double", "m2-mixed") and args.c_list == (1, 3)
    try:
        has_gpu = _gpu.device_count() > 0
    except Exception:
        has_gpu = False
    if not has_gpu:
        rc = main(["bench", "matvec", "--spheres", "1", "--refine", "0", "--reps", "2", "--sets", "2"])
        assert rc == 1 and "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_bench_writes_reference_schema(tmp_path, hx):
    from paper_1911_00093_b200.__main__ import main
    out = tmp_path / "r.json"
    assert main(["bench", "matvec", "--spheres", "2", "--refine", "1", "--reps", "5", "--sets", "2",
                 "--schemes", "m1-double,m2-mixed", "--c-list", "3", "--format", "json",
                 "--out", str(out)]) == 0
    recs = hx.read_report(out)
    assert [r.scheme for r in recs] == ["m1-double", "m2-mixed", "m3:c=3"]
    assert all(r.device == "cuda:0" and r.matvecs_per_s > 0 for r in recs)
    assert main(["bench", "solve", "--spheres", "2", "--refine", "1", "--sets", "1",
                 "--schemes", "m1-double", "--out", str(tmp_path / "s.csv")]) == 0
    assert hx.read_report(tmp_path / "s.csv")[0].iterations > 0


def test_cli_info_on_host(tmp_path, capsys):
    """`info` builds on the host and writes the reference's interchange files."""
    from paper_1911_00093_b200.__main__ import main
    part, mesh = tmp_path / "p.txt", tmp_path / "m.txt"
    assert main(["info", "--spheres", "1", "--refine", "1", "--json",
                 "--dump-partition", str(part), "--export-mesh", str(mesh)]) == 0
    out = capsys.readouterr().out
    assert '"n": 80' in out and part.exists() and mesh.exists()


@pytest.mark.gpu
def test_cli_solve_and_gpu_build(capsys):
    from paper_1911_00093_b200.__main__ import main
    assert main(["solve", "--spheres", "2", "--refine", "1", "--scheme", "m2-mixed", "--json",
                 "--gpu-build"]) == 0
    assert '"converged": true' in capsys.readouterr().out
    assert main(["info", "--spheres", "2", "--refine", "1", "--gpu-build"]) == 0
