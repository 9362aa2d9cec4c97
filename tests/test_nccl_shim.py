"""CPU test of the NCCL stand-in used by tests/test_gpu_dist_shim.py: built
host-only (-DHMX_SHIM_HOST_ONLY: cudaMemcpy = memcpy), three processes run
50 rounds of the allgather (grouped send/recv, uneven slices) and grouped
allreduce sequence libhmx_gpu's multi-GPU mode issues; every rank must see
every slice and the reduced values, with no deadlock."""
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent


def test_shim_protocol_three_processes(tmp_path):
    so = tmp_path / "libshim_host.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-DHMX_SHIM_HOST_ONLY",
                    str(HERE / "shim" / "hmx_nccl_shim.cpp"), "-o", str(so)], check=True)
    uid = tmp_path / "uid.bin"
    procs = [subprocess.Popen([sys.executable, str(HERE / "shim" / "shim_protocol_worker.py"), str(so),
                               str(r), "3", str(uid)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                              text=True) for r in range(3)]
    outs = [p.communicate(timeout=120)[0] for p in procs]
    for r, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0 and f"rank {r} ok" in out, out
