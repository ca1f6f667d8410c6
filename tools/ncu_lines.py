"""Per-source-line instruction counts and stall samples from an ncu report
(ncu -i REP --page source --csv --print-source cuda,sass).
Usage: python tools/ncu_lines.py REP [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
fname = None
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    i_ex = hdr.index("Instructions Executed")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        inst = float(r[i_ex]); samp = float(r[i_s])
    except ValueError:
        continue
    k = (fname, line)
    a = agg.setdefault(k, [0.0, 0.0, r[1][:90]])
    a[0] += inst
    a[1] += samp
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot_i:.0f}, stall samples {tot_s:.0f}")
for (f, l), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{f}:{l:4d} inst {100 * i / tot_i:5.1f}% samples {100 * s / tot_s:5.1f}%  {src}")
