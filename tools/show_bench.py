"""Print the per-variant table of a bench.py JSON line (default gpurun_out/qb.json)."""
import json
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/qb.json"
d = json.loads(open(path).read().splitlines()[-1])
for k, v in d["variants"].items():
    s = v.get("solve", {})
    print(f"{k:10s} {v['ms']:.4f} ms {v['GBps']:7.0f} GB/s {v['frac_of_peak']:.3f}  s1 {v['stage1_ms']:.4f} "
          f"({v['stage1_GBps'] or 0:5.0f})  s2 {v['stage2_ms']:.4f} ({v['stage2_GBps'] or 0:5.0f})  "
          f"{s.get('iterations', '')} {s.get('converged', '')}")
