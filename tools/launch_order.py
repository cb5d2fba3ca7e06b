"""Print an ncu --csv launch list (gpu__time_duration.sum) in launch order."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = 0.0
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"]) / 1e3
            tot += v
            print(f"{d['ID']:>4} {v:9.1f} us  grid {d.get('Grid Size', ''):>16} {d['Kernel Name'].split('(')[0][:70]}")
print(f"total {tot:.1f} us")
