"""Hot source lines of one kernel in an ncu capture (source page, CUDA view).

  python tools/ncu_hot_lines.py <report.ncu-rep> <kernel substring> [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, pat = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    # the dump is a sequence of per-(kernel, file) tables
    cur_fn, cur_file, hdr = None, None, None
    agg = {}
    tot = {}
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1]
            continue
        if row[0] == "Function Name":
            cur_fn = row[1]
            hdr = None
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or cur_fn is None or pat not in cur_fn:
            continue
        if row[0] == "":
            continue  # SASS rows under a source line (already summed in the line's row)
        try:
            ln = int(row[0])
            smp = float(row[hdr.index("# Samples")] or 0)
            ins = float(row[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        key = (cur_fn[:60], cur_file.split("/")[-1], ln)
        a = agg.setdefault(key, [0.0, 0.0, row[1].strip()[:110], {}])
        a[0] += smp
        a[1] += ins
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and row[i]:
                try:
                    a[3][h] = a[3].get(h, 0.0) + float(row[i])
                except ValueError:
                    pass
        tot[cur_fn[:60]] = tot.get(cur_fn[:60], 0.0) + smp
    for fn, t in tot.items():
        print(f"== {fn}: {t:.0f} samples")
        rows = sorted(((k, v) for k, v in agg.items() if k[0] == fn), key=lambda kv: -kv[1][0])[:top]
        for (f, file, ln), (smp, ins, src, st) in rows:
            s3 = sorted(st.items(), key=lambda kv: -kv[1])[:2]
            print(f"{100 * smp / t:5.1f}% ins={ins / 1e6:7.2f}M {file}:{ln:<5d} {src}   "
                  + " ".join(f"{k[6:]}={v:.0f}" for k, v in s3))


if __name__ == "__main__":
    main()
