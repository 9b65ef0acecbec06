"""The last K launches of an ncu launch list, in launch order (steady state of
a bench run, after autotune): python tools/launch_tail.py launches.csv K"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
iK, iM, iV, iID = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
order, t = [], {}
for r in rows[1:]:
    if r[iM] != "gpu__time_duration.sum":
        continue
    if r[iID] not in t:
        order.append((r[iID], r[iK].split("(")[0]))
    t[r[iID]] = float(r[iV].replace(",", "")) / 1e6
k = int(sys.argv[2]) if len(sys.argv) > 2 else 12
for lid, name in order[-k:]:
    print(f"{lid:>6s}  {t[lid]:10.3f} ms  {name}")
