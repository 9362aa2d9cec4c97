"""Print the device plan layout (segments, grids, stage bytes) and stage
timings of every variant at one BASELINE config.

  python tools/plan_info.py --config 2
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
import paper_1911_00093_b200 as hx  # noqa: E402
from paper_1911_00093_b200.matvec import get_plan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--variants", nargs="*", default=["m1-double", "m1-mixed", "m2-mixed", "m3:c=3",
                                                       "m3:c=-1", "m1-single", "m2-single"])
    a = ap.parse_args()
    mesh, h, x, b, _ = bench.build_workload(a.config)
    for s in a.variants:
        sh = hx.prepare_scheme(h, s)
        plan = get_plan(sh)
        hx.matvec(sh, x)
        i = plan.info()
        r = plan.bench(20, 200)
        gb = (i["stage1_bytes"] + i["stage2_bytes"] + 16 * mesh.n) / 1e9
        print(f"{s:9s} {r['ms']*1e3:7.1f} us ({gb / r['ms'] * 1e3 / 1e3:5.2f} TB/s)  "
              f"s1 {r['stage1_ms']*1e3:6.1f} us {i['stage1_bytes']/1e6:7.1f} MB seg {i['s1_segments']:6d} "
              f"grid {i['s1_grid']:6d}x{i['s1_block']:3d} tasks {i['s1_tasks']:5d} | "
              f"s2 {r['stage2_ms']*1e3:6.1f} us {i['stage2_bytes']/1e6:7.1f} MB seg {i['s2_segments']:6d} "
              f"runs {i['s2_runs']:7d} grid {i['s2_grid']:6d}x{i['s2_block']:3d} z {i['z_len']}",
              flush=True)


if __name__ == "__main__":
    main()
