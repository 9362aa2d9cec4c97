"""Stage-1 chunk-size sweep (hmx_plan_options.s1_chunk_bytes) at one config."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import numpy as np  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402
from paper_1911_00093_b200 import _gpu  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    sizes = [int(s) for s in sys.argv[2:]] or [128 << 10, 256 << 10, 512 << 10, 1 << 20]
    mesh, h, x, b, _ = bench.build_workload(cfg)
    for name in ["m1-double", "m2-mixed"]:
        sh = hx.prepare_scheme(h, name)
        for cb in sizes:
            p = _gpu.Plan(sh.packed, h.partition.table, np.asarray(h.permutation), sh.scheme.label,
                          h.n, s1_chunk_bytes=cb)
            p.matvec(x)
            r = p.bench(5, 100)
            print(f"{name} chunk {cb >> 10} KB: {r['ms']:.4f} ms  s1 {r['stage1_ms']:.4f}  s2 {r['stage2_ms']:.4f}  "
                  f"s1 CTAs {p.info()['s1_grid']}", flush=True)
            p.close()


if __name__ == "__main__":
    main()
