"""Copy one tools/gpu_round.sh pass (gpurun_out/<tag>) into profiles/<dest>:
bench lines, the ncu launch-list summary (+ the gzipped list), and CSV
exports of the ncu --set full captures (the metrics the DESIGN tables cite).

    python tools/summarize_round.py r1b r1
"""
import collections
import csv
import gzip
import io
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "gpu__time_duration.sum",
           "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
           "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "sm__inst_executed.avg.pct_of_peak_sustained_elapsed",
           "l1tex__throughput.avg.pct_of_peak_sustained_active"]


def short(name: str) -> str:
    n = name.replace("void ", "").replace("<unnamed>::", "")
    if n.startswith("k_") or n.startswith("("):
        n = n.split("(")[0]
    return n[:60]


def launch_summary(src: str, dst: str, cmd: str) -> None:
    lines = open(src).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v
        k = short(r["Kernel Name"])
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + us)
    total = sum(t for _, t in agg.values())
    nl = sum(n for n, _ in agg.values())
    with open(dst, "w") as f:
        f.write(f"# {cmd}\n# cold-cache, serialised by ncu: the kernels' SHARES are what compares with the live step\n")
        f.write(f"# total {total / 1e3:.3f} ms over {nl} launches\n")
        f.write(f"{'kernel':60s} {'launches':>9s} {'total_us':>12s} {'avg_us':>9s} {'share':>6s}\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k:60s} {n:9d} {t:12.1f} {t / n:9.2f} {100 * t / total:5.1f}%\n")
    with open(src, "rb") as fi, gzip.open(dst.replace("_summary.txt", ".csv.gz"), "wb") as fo:
        shutil.copyfileobj(fi, fo)


def ncu_export(rep: str, dst: str, note: str) -> None:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    idx = [h.index("Kernel Name")] + [h.index(m) for m in METRICS if m in h]
    with open(dst, "w", newline="") as f:
        f.write(f"# {note}\n")
        w = csv.writer(f)
        for r in rows:
            w.writerow([short(r[idx[0]]) if r is not rows[0] and r is not rows[1] else r[idx[0]]]
                       + [r[i] for i in idx[1:]])


def main() -> None:
    tag, dest = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r1"
    src = os.path.join(ROOT, "gpurun_out", tag)
    out = os.path.join(ROOT, "profiles", dest)
    os.makedirs(out, exist_ok=True)
    for f in ("bench.json", "bench_ref.json", "mupdate.txt"):
        if os.path.exists(os.path.join(src, f)):
            shutil.copy(os.path.join(src, f), os.path.join(out, f))
    if os.path.exists(os.path.join(src, "launches.csv")):
        launch_summary(os.path.join(src, "launches.csv"), os.path.join(out, "launches_summary.txt"),
                       "ncu --metrics gpu__time_duration.sum --clock-control none -c 2600 "
                       "python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-micro")
    if os.path.exists(os.path.join(src, "eprop_c1.ncu-rep")):
        ncu_export(os.path.join(src, "eprop_c1.ncu-rep"), os.path.join(out, "eprop_c1_ncu_full.csv"),
                   "C1 blocked e-prop pass (tools/profile_eprop.py c1, EAGER=1), ncu --set full")
    if os.path.exists(os.path.join(src, "deepr.ncu-rep")):
        ncu_export(os.path.join(src, "deepr.ncu-rep"), os.path.join(out, "deepr_ncu_full.csv"),
                   "ROWS=262144 instance of the M-update recipe (tools/mupdate_breakdown.py), ncu --set full")
    if os.path.exists(os.path.join(src, "forward_c1.ncu-rep")):
        ncu_export(os.path.join(src, "forward_c1.ncu-rep"), os.path.join(out, "forward_c1_ncu_full.csv"),
                   "C1 grouped forward launch (8 timesteps, tools/profile_forward.py c1), ncu --set full")
    if os.path.exists(os.path.join(src, "prop_bucketed.ncu-rep")):
        ncu_export(os.path.join(src, "prop_bucketed.ncu-rep"), os.path.join(out, "prop_bucketed_ncu_full.csv"),
                   "M-prop q=10% on 2^20 rows through PropBuckets (tools/profile_prop.py), ncu --set full")
    print("wrote", sorted(os.listdir(out)))


if __name__ == "__main__":
    main()
