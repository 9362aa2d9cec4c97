"""Source lines of one kernel in an ncu capture, by executed warp instructions.

  python tools/ncu_ins_lines.py <report.ncu-rep> <kernel substring> [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_fn = None
hdr = None
agg = collections.Counter()
src = {}
f = ""
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        f = row[1].split('/')[-1]
        continue
    if row[0] == "Function Name":
        cur_fn = row[1]
        hdr = None
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or pat not in cur_fn or row[0] == "":
        continue
    try:
        ln = int(row[0])
        ins = float(row[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    agg[(f, ln)] += ins
    src[(f, ln)] = row[1].strip()[:100]
tot = sum(agg.values())
print(f"{tot / 1e6:.1f}M warp instructions attributed")
for k, v in agg.most_common(top):
    print(f"{v / 1e6:7.2f}M {100 * v / tot:4.1f}% {k[0]}:{k[1]} {src[k]}")
