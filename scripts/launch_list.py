"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel name, launch count and mean duration (us)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
names = rows[hdr]
ik, iv, im = names.index("Kernel Name"), names.index("Metric Value"), names.index("Metric Name")
seq = []
for r in rows[hdr + 1:]:
    if len(r) == len(names) and r[im] == "gpu__time_duration.sum":
        v = float(r[iv].replace(",", ""))
        unit = r[names.index("Metric Unit")]
        us = v / 1e3 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1e3
        seq.append((r[ik].split("(")[0][:80], us))
agg = collections.OrderedDict()
for k, v in seq:
    agg.setdefault(k, []).append(v)
for k, v in agg.items():
    print(f"{len(v):5d} x {sum(v)/len(v):9.2f} us  {k}")
print("last 12 launches:")
for k, v in seq[-12:]:
    print(f"   {v:9.2f} us  {k}")
