"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
idx = {k: i for i, k in enumerate(hdr)}
data = collections.OrderedDict()
for r in rows[start + 1:]:
    d = data.setdefault(r[idx["ID"]], {"name": r[idx["Kernel Name"]]})
    d[r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
tot = 0.0
for kid, d in data.items():
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    print(f"{kid:>4} {d['name'][:58]:58s} {t:9.1f} us  R {d.get('dram__bytes_read.sum', 0)/1e6:8.1f} MB"
          f"  W {d.get('dram__bytes_write.sum', 0)/1e6:8.1f} MB")
print(f"total {tot:.1f} us over {len(data)} launches")
