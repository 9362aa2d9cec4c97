"""The C ABI (include/hmx_gpu.h): libhmx_gpu.so loads and exports every
declared entry point, the ctypes structures match the C layout, and without
a GPU the product path fails loudly instead of falling back to the CPU."""

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "hmx_gpu.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(hmx_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1911_00093_b200 import _gpu
    lib = _gpu.load_library()
    names = declared_functions()
    assert len(names) >= 9
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_gpu.SIGNATURES)


def test_ctypes_layouts_match_header(tmp_path):
    from paper_1911_00093_b200 import _gpu
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "hmx_gpu.h"\n'
                   "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\","
                   "sizeof(hmx_matrix_desc), offsetof(hmx_matrix_desc, buf32),"
                   "sizeof(hmx_plan_options), sizeof(hmx_plan_info),"
                   "sizeof(hmx_solve_report), offsetof(hmx_solve_report, device_ms),"
                   "sizeof(hmx_master_desc), offsetof(hmx_master_desc, n_data),"
                   "sizeof(hmx_prepare_info));return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [ctypes.sizeof(_gpu.MatrixDesc), _gpu.MatrixDesc.buf32.offset,
            ctypes.sizeof(_gpu.PlanOptions), ctypes.sizeof(_gpu.PlanInfo),
            ctypes.sizeof(_gpu.SolveReport), _gpu.SolveReport.device_ms.offset,
            ctypes.sizeof(_gpu.MasterDesc), _gpu.MasterDesc.n_data.offset,
            ctypes.sizeof(_gpu.PrepareInfo)]
    assert got == want


def _cuda_available():
    from paper_1911_00093_b200 import _gpu
    try:
        return _gpu.device_count() > 0
    except Exception:
        return False


@pytest.mark.skipif(_cuda_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu(hx):
    mesh = hx.build_sphere_mesh(hx.axis_centers(1, 3.0), refinement=0)
    h = hx.build_hmatrix(mesh)
    sh = hx.prepare_scheme(h, "m1-double")
    with pytest.raises(RuntimeError, match="CUDA"):
        hx.matvec(sh, np.ones(mesh.n))
    with pytest.raises(RuntimeError, match="CUDA"):
        hx.bicgstab(sh, h, np.ones(mesh.n))


def test_shape_errors_before_device(hx):
    mesh = hx.build_sphere_mesh(hx.axis_centers(1, 3.0), refinement=0)
    h = hx.build_hmatrix(mesh)
    sh = hx.prepare_scheme(h, "m1-double")
    with pytest.raises(ValueError):
        hx.matvec(sh, np.ones(mesh.n + 1))
    with pytest.raises(ValueError):
        hx.bicgstab(sh, h, np.ones(mesh.n + 1))
    with pytest.raises(ValueError):
        hx.matvec_threaded(sh, np.ones(mesh.n), threads=0)
    with pytest.raises(ValueError):
        hx.SourceVector(np.zeros((2, 2)))
    with pytest.raises(ValueError):
        hx.SolverConfig(tol=0.0)
    # true_residual checks both operands before any device work
    with pytest.raises(ValueError, match="does not match"):
        hx.true_residual(h, np.ones(mesh.n - 1), np.ones(mesh.n))
    with pytest.raises(ValueError, match="broadcast"):
        hx.true_residual(h, np.ones(mesh.n), np.ones(mesh.n + 3))


def test_nccl_shim_builds_and_exports_the_resolved_symbols():
    """tests/shim (the multi-process GPU test's NCCL stand-in) compiles and
    exports the nine functions hmx_solver.cu's nccl_api() resolves."""
    import ctypes

    from test_gpu_dist_shim import build_shim
    lib = ctypes.CDLL(str(build_shim()))
    for name in ("ncclGetUniqueId", "ncclCommInitRank", "ncclCommDestroy", "ncclGetErrorString",
                 "ncclGroupStart", "ncclGroupEnd", "ncclSend", "ncclRecv", "ncclAllReduce"):
        assert hasattr(lib, name), name
    src = (Path(__file__).resolve().parent.parent / "paper_1911_00093_b200" / "csrc" / "hmx_solver.cu").read_text()
    for name in ("ncclGetUniqueId", "ncclCommInitRank", "ncclGroupEnd", "ncclAllReduce"):
        assert f'"{name}"' in src
