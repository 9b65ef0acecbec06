"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_*] --csv):
per kernel: launches, total/avg device time, share of the run, DRAM bytes per launch.
python tools/launch_summary.py launches.csv"""
import csv, sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
iK, iM, iV, iID = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = defaultdict(lambda: defaultdict(float))
launch = {}
for r in rows[1:]:
    name = r[iK].split("(")[0]
    name = "qk_pass_<hash> (specialized block pass)" if name.startswith("qk_pass_") else name
    launch[r[iID]] = name
    per[r[iID]][r[iM]] = float(r[iV].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for lid, m in per.items():
    a = agg[launch[lid]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values()) or 1
print(f"{'kernel':45s} {'launches':>8s} {'total ms':>10s} {'avg ms':>9s} {'share':>7s} {'DRAM GB/launch':>15s}")
for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:45s} {n:8d} {t / 1e6:10.3f} {t / n / 1e6:9.3f} {t / tot * 100:6.1f}% {b / n / 1e9:15.3f}")
