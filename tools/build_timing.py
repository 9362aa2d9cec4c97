"""Host vs device H-matrix compression time at one BASELINE config, and a
bitwise comparison of the two masters.

  python tools/build_timing.py 4
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    c = bench.CONFIGS[cfg]
    mesh = hx.jittered_sphere_mesh(c["level"], seed=42, centers=c.get("centers", ((0.0, 0.0, 0.0),)),
                                   voltages=c.get("voltages"))
    t0 = time.perf_counter()
    part = hx.build_block_partition(hx.build_cluster_tree(mesh, c["leaf"]), 2.0)
    t_part = time.perf_counter() - t0
    import torch
    torch.cuda.init()
    hx.build_hmatrix(hx.jittered_sphere_mesh(2, seed=1), device=0)  # context + module load
    t0 = time.perf_counter()
    hg = hx.build_hmatrix(mesh, partition=part, aca_tol=c["aca"], device=0)
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    _ = hg.packed.data
    t_dl = time.perf_counter() - t0
    t0 = time.perf_counter()
    hc = hx.build_hmatrix(mesh, partition=part, aca_tol=c["aca"])
    t_host = time.perf_counter() - t0
    same = (np.array_equal(hg.packed.ranks, hc.packed.ranks)
            and np.array_equal(hg.packed.data.view(np.uint64), hc.packed.data.view(np.uint64)))
    print(f"config {cfg}: N={mesh.n} blocks={part.table.shape[0]} partition {t_part:.2f} s | "
          f"device build {t_dev:.2f} s (+ {t_dl:.2f} s to copy the {hg.packed.data.nbytes/1e9:.2f} GB "
          f"masters to the host on demand) | "
          f"host build ({hx._native.host_threads()} threads) {t_host:.2f} s | bitwise equal: {same}")


if __name__ == "__main__":
    main()
