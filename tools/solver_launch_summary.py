"""Summarise tools/profile_solver_launches.sh output into profiles/round1_solver_launches.json
(per-kernel device time of the second, timed solve; whole-graph durations)."""
import csv, collections, json, sys, re
out = {}
for c in (4, 2):
    rows = [r for r in csv.reader(l for l in open(f"gpurun_out/round1_solver_launches_config{c}.csv") if l.startswith('"'))]
    hdr = rows[0]; rows = rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    # the second (timed) solve: profile_solve runs two solves; split at the second init_kernel
    inits = [i for i, r in enumerate(rows) if r[ki].startswith("init_kernel")]
    start = inits[1] if len(inits) > 1 else 0
    # the preceding matvec of the second solve's r0 = b - A x0 starts 2 launches before init? keep from the perm/dot before
    sel = rows[start - 4:] if start >= 4 else rows[start:]
    agg = collections.OrderedDict()
    for r in sel:
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
        a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += float(r[vi].replace(",", "")) / 1e3
    tot = sum(v[1] for v in agg.values())
    out[f"config{c}"] = {"total_us": tot, "kernels": {k: {"launches": v[0], "us": round(v[1], 1), "share": round(v[1] / tot, 4)} for k, v in agg.items()}}
    g = [r for r in csv.reader(l for l in open(f"gpurun_out/round1_solver_graph_config{c}.csv") if l.startswith('"'))]
    out[f"config{c}"]["graph_profiles_us"] = [float(r[g[0].index("Metric Value")].replace(",", "")) / 1e3 for r in g[1:]]
    out[f"config{c}"]["plain_run"] = open(f"gpurun_out/ps_plain_{c}.log").read().strip()
print(json.dumps(out, indent=1))
json.dump(out, open("profiles/round1_solver_launches.json", "w"), indent=1)
