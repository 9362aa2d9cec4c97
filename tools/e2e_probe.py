"""Break down the host-pointer matvec (public API) wall time at one config."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402
from paper_1911_00093_b200.matvec import get_plan  # noqa: E402


def wall(fn, reps=30):
    for _ in range(3):
        fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(t)), 1e3 * float(np.min(t))


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    import torch
    mesh, h, x, b, _ = bench.build_workload(cfg)
    sh = hx.prepare_scheme(h, "m1-double")
    plan = get_plan(sh)
    n = mesh.n
    print("device bench ms", plan.bench(3, 50)["ms"])
    print("hx.matvec           median/min ms %.3f %.3f" % wall(lambda: hx.matvec(sh, x)))
    import torch as _t
    xpin = _t.from_numpy(x).pin_memory().numpy()
    print("hx.matvec pinned x  median/min ms %.3f %.3f" % wall(lambda: hx.matvec(sh, xpin)))
    print("plan.matvec         median/min ms %.3f %.3f" % wall(lambda: plan.matvec(x)))
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    print("device-ptr matvec   median/min ms %.3f %.3f" % wall(
        lambda: plan.matvec_device(xd.data_ptr(), yd.data_ptr(), permuted=False)))
    print("np.empty(n)         median/min ms %.3f %.3f" % wall(lambda: np.empty(n)))
    y = np.empty(n)
    print("np.copyto fresh     median/min ms %.3f %.3f" % wall(lambda: np.copyto(np.empty(n), x)))
    print("np.copyto warm      median/min ms %.3f %.3f" % wall(lambda: np.copyto(y, x)))


if __name__ == "__main__" and len(sys.argv) <= 2:
    main()


def transfers(n=327680):
    import torch
    x = np.random.default_rng(0).uniform(-1, 1, n)
    xt = torch.from_numpy(x)
    xp = torch.empty(n, dtype=torch.float64).pin_memory()
    xd = torch.empty(n, dtype=torch.float64, device="cuda")

    def pageable_h2d():
        xd.copy_(xt)
        torch.cuda.synchronize()

    def pinned_h2d():
        xd.copy_(xp, non_blocking=True)
        torch.cuda.synchronize()

    def pinned_d2h():
        xp.copy_(xd, non_blocking=True)
        torch.cuda.synchronize()

    def pageable_d2h():
        xt.copy_(xd)
    print("pageable H2D  %.3f %.3f" % wall(pageable_h2d))
    print("pinned H2D    %.3f %.3f" % wall(pinned_h2d))
    print("pinned D2H    %.3f %.3f" % wall(pinned_d2h))
    print("pageable D2H  %.3f %.3f" % wall(pageable_d2h))


if __name__ == "__main__" and len(sys.argv) > 2:
    transfers()
