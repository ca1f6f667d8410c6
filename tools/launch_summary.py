"""Per-kernel launch counts and mean durations from an ncu launch list
(ncu --metrics gpu__time_duration.sum --csv --log-file F).
Usage: python tools/launch_summary.py F [top_n]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hd = rows[h]
ki, vi = hd.index("Kernel Name"), hd.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    if len(r) > vi:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[r[ki][:70]][0] += 1
        agg[r[ki][:70]][1] += v
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{n:6d} {v / n / 1000:9.1f} us  {v / 1e6:8.2f} ms  {k}")
