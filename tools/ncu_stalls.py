"""Per-source-line stall samples and instructions of one kernel in an ncu
report: python tools/ncu_stalls.py REP KERNEL_REGEX [top_n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
hdr, fname, agg = None, None, {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and fname:
        try:
            ln = int(r[0])
            v = float(r[hdr.index("Warp Stall Sampling (All Samples)")].replace(",", ""))
            n = float(r[hdr.index("Instructions Executed")].replace(",", ""))
        except ValueError:
            continue
        a = agg.setdefault((fname, ln, r[1][:90]), [0.0, 0.0])
        a[0] += v
        a[1] += n
tot = sum(v[0] for v in agg.values()) or 1.0
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}% stalls  {v[1]:12.0f} inst  {k[0]}:{k[1]}  {k[2]}")
