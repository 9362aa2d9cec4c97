"""Scheme / c-sweep preparation cost: host prepare_scheme + plan upload vs
prepare_scheme_device from resident masters (config 4 by default)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402
from paper_1911_00093_b200 import _gpu  # noqa: E402
from paper_1911_00093_b200.device_prepare import get_master  # noqa: E402
from paper_1911_00093_b200.precision import _split_factor, parse_scheme  # noqa: E402

import numpy as np  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    mesh, h, x, b, _ = bench.build_workload(cfg)
    perm = np.asarray(h.permutation)
    t0 = time.perf_counter()
    master = get_master(h)
    print(f"config {cfg}: masters uploaded once in {time.perf_counter() - t0:.3f} s "
          f"({h.packed.data.nbytes / 1e9:.2f} GB)", flush=True)
    schemes = ["m1-double", "m1-mixed", "m2-mixed", "m2-single"] + [f"m3:c={c}" for c in (-1, 0, 1, 3, 5, 7)]
    for name in schemes:
        s = parse_scheme(name)
        t0 = time.perf_counter()
        sh = hx.prepare_scheme(h, name)
        t1 = time.perf_counter()
        ph = _gpu.Plan(sh.packed, h.partition.table, perm, s.label, h.n)
        t2 = time.perf_counter()
        yh, _ = ph.matvec(x)
        ph.close()
        del sh
        t3 = time.perf_counter()
        pd, info = _gpu.Plan.prepared(master, s.label, _split_factor(s.c) if s.method == 3 else 0.0)
        t4 = time.perf_counter()
        yd, _ = pd.matvec(x)
        pd.close()
        print(f"{name:9s} host: prepare {t1 - t0:.3f} s + plan {t2 - t1:.3f} s = {t2 - t0:.3f} s | "
              f"device: {t4 - t3:.3f} s | payload {info['payload_bytes'] / 1e9:.2f} GB, "
              f"FP32 ranks {info['fp32_ranks']} | bitwise equal {bool(np.array_equal(yd, yh))}",
              flush=True)


if __name__ == "__main__":
    main()
