"""Summarise ncu captures (.ncu-rep) and launch lists into profiles/.

  python tools/ncu_summary.py <tag> <report.ncu-rep> [more.ncu-rep ...]
  python tools/ncu_summary.py --launches <tag> <launches.csv>
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

PROFILES = Path(__file__).resolve().parent.parent / "profiles"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__occupancy_limit_registers", "launch__shared_mem_per_block_static"]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1e3, "ms": 1e6, "ns": 1.0,
         "usecond": 1e3, "msecond": 1e6, "nsecond": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise(rep):
    hdr, units, rows = raw(rep)
    res = []
    for r in rows:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    val = float(v)
                    unit = units[i]
                    if unit in SCALE and ("bytes" in k or "duration" in k):
                        val *= SCALE[unit]
                        unit = "byte" if "bytes" in k else "ns"
                    d[k] = val
                except ValueError:
                    d[k] = v
        stalls = [(hdr[i].replace("smsp__average_warps_issue_stalled_", "")
                   .replace("_per_issue_active.ratio", ""), float(r[i]))
                  for i in range(len(hdr)) if hdr[i].startswith("smsp__average_warps_issue_stalled_")
                  and r[i].replace(".", "").isdigit()]
        d["top_stalls"] = sorted(stalls, key=lambda s: -s[1])[:6]
        d["dram_bytes_per_launch"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        res.append(d)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        agg[r[ik]].append(float(r[iv].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "total_ns": sum(v), "mean_ns": sum(v) / len(v),
             "share": sum(v) / tot} for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]


def main():
    PROFILES.mkdir(exist_ok=True)
    if sys.argv[1] == "--launches":
        tag, path = sys.argv[2], sys.argv[3]
        out = launches(path)
        (PROFILES / f"{tag}_launches.json").write_text(json.dumps(out, indent=1))
        for d in out:
            print(f"{d['kernel'][:70]:70s} n={d['launches']:4d} mean={d['mean_ns']/1e3:9.1f}us "
                  f"share={100*d['share']:5.1f}%")
        return
    tag = sys.argv[1]
    allres = {}
    for rep in sys.argv[2:]:
        allres[Path(rep).stem] = summarise(rep)
    (PROFILES / f"{tag}_ncu.json").write_text(json.dumps(allres, indent=1))
    for name, res in allres.items():
        for d in res:
            print(name, d["kernel"][:40], f"{d['gpu__time_duration.sum']/1e3:.1f}us",
                  f"dram={d['dram_bytes_per_launch']/1e9:.3f}GB",
                  f"dram%={d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')}",
                  d["top_stalls"][:3])


if __name__ == "__main__":
    main()
